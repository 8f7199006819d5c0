"""The frame server's step after the render: frames in its wire format.

The reference's frame loop (`FrameLoop.tick`, /root/reference/pkg/src/
raytracer/server.py:276-289) renders into a 0xAARRGGBB Framebuffer and then
re-packs every pixel on the host into the RAYF message — a 16-byte big-endian
header and R,G,B,A bytes (`encode_frame`, server.py:56-64).  `FrameEncoder`
renders straight into that message: the kernels pack R,G,B,A (option "rgba"
of the C ABI) into a page-locked buffer laid out header-then-payload, so a
frame needs no host-side pass at all.  `encode_frame` / `decode_frame_header`
restate the reference's functions for host framebuffers.
"""

from __future__ import annotations

import struct

import numpy as np

from . import _native
from .model import MAX_BOUNCE_LIMIT, camera_viewport_distance, pack_scene

FRAME_MAGIC = 0x52415946  # "RAYF" (server.py:46)
FORMAT_RGBA8 = 1          # server.py:47
HEADER = struct.Struct(">IIHHB3x")  # server.py:48


def encode_frame(frame_id: int, fb) -> bytes:
    """RAYF message of a 0xAARRGGBB framebuffer (server.py:56-64)."""
    header = HEADER.pack(FRAME_MAGIC, frame_id & 0xFFFFFFFF, fb.width, fb.height, FORMAT_RGBA8)
    bgra = np.ascontiguousarray(fb.pixels, dtype=np.uint32).view(np.uint8).reshape(-1, 4)
    return header + bgra[:, [2, 1, 0, 3]].tobytes()


def decode_frame_header(data: bytes):
    """(frame_id, width, height, fmt); raises ValueError on a bad magic (server.py:67-74)."""
    if len(data) < HEADER.size:
        raise ValueError("frame shorter than header")
    magic, frame_id, width, height, fmt = HEADER.unpack_from(data)
    if magic != FRAME_MAGIC:
        raise ValueError(f"bad frame magic 0x{magic:08X}")
    return frame_id, width, height, fmt


class FrameEncoder:
    """Render frames directly as RAYF messages on one GPU.

    `render(scene, cam, params, frame_id)` returns a memoryview of the
    message (header + R,G,B,A payload), valid until the next call."""

    def __init__(self, device: int = 0):
        self.ctx = _native.Context((int(device),))
        self.ctx.set_option("rgba", 1)
        self._buf = None
        self._dims = None

    def _buffer(self, width, height):
        if self._dims != (width, height):
            self._buf = np.zeros(HEADER.size + 4 * width * height, dtype=np.uint8)
            self._dims = (width, height)
            self.ctx.pin(self._buf)
        return self._buf

    def render(self, scene, cam, params, frame_id: int, workers=None, *, precision=None) -> memoryview:
        if params.bounce_limit > MAX_BOUNCE_LIMIT:
            raise ValueError(f"bounce limit capped at {MAX_BOUNCE_LIMIT}")
        from .renderer import _prec, _scene_argv

        prec = _prec(precision)
        w, h = int(params.width), int(params.height)
        buf = self._buffer(w, h)
        HEADER.pack_into(buf, 0, FRAME_MAGIC, frame_id & 0xFFFFFFFF, w, h, FORMAT_RGBA8)
        ps = pack_scene(scene)
        cam_pos = np.array(cam.position, dtype=np.float64)
        n_parts = 1 if workers is None else int(workers)
        rc = _native.load().rt_render_v1(
            self.ctx.handle, _native.ptr(buf.ctypes.data + HEADER.size), None, w, h, _native.ptr(cam_pos),
            float(cam.yaw), float(cam.pitch), camera_viewport_distance(cam.fov), *_scene_argv(ps),
            int(params.shadow_samples), int(params.bounce_limit), n_parts, prec,
        )
        _native.check(rc, "rt_render_v1")
        return memoryview(buf)

    def close(self):
        self.ctx.close()


class PipelinedFrameEncoder:
    """`FrameEncoder` for the frame loop (FrameLoop.tick, server.py:276-289):
    up to `depth` RAYF messages in flight, each frame's device-to-host copy
    overlapping the next frame's kernels (rt_render_async_v1).

    `submit(...)` returns a ticket; `wait(ticket)` returns that frame's
    message, valid until `depth` more frames have been submitted."""

    def __init__(self, depth: int = 3, device: int = 0):
        if not 1 <= int(depth) <= 4:
            raise ValueError("depth must be 1-4")
        self.depth = int(depth)
        self.ctx = _native.Context((int(device),))
        self.ctx.set_option("rgba", 1)
        self._bufs = [None] * self.depth
        self._dims = None
        self._next = 0
        self._pending = set()

    def submit(self, scene, cam, params, frame_id: int, *, precision=None) -> int:
        if params.bounce_limit > MAX_BOUNCE_LIMIT:
            raise ValueError(f"bounce limit capped at {MAX_BOUNCE_LIMIT}")
        from .renderer import _prec, _scene_argv

        prec = _prec(precision)
        w, h = int(params.width), int(params.height)
        ticket = self._next
        slot = ticket % self.depth
        if ticket - self.depth in self._pending:
            self.wait(ticket - self.depth)
        if self._dims != (w, h):
            self.drain()
            for i in range(self.depth):
                if self._bufs[i] is not None:
                    _native._PINS.release(self._bufs[i])
                    self.ctx.unpin(self._bufs[i])
                self._bufs[i] = np.zeros(HEADER.size + 4 * w * h, dtype=np.uint8)
                self.ctx.pin(self._bufs[i], max_pinned=self.depth + 1)
                _native._PINS.hold(self._bufs[i])  # copies land here while frames are in flight
            self._dims = (w, h)
        buf = self._bufs[slot]
        HEADER.pack_into(buf, 0, FRAME_MAGIC, frame_id & 0xFFFFFFFF, w, h, FORMAT_RGBA8)
        ps = pack_scene(scene)
        cam_pos = np.array(cam.position, dtype=np.float64)
        rc = _native.load().rt_render_async_v1(
            self.ctx.handle, slot, _native.ptr(buf.ctypes.data + HEADER.size), w, h, _native.ptr(cam_pos),
            float(cam.yaw), float(cam.pitch), camera_viewport_distance(cam.fov), *_scene_argv(ps),
            int(params.shadow_samples), int(params.bounce_limit), prec,
        )
        _native.check(rc, "rt_render_async_v1")
        self._pending.add(ticket)
        self._next += 1
        return ticket

    def wait(self, ticket: int) -> memoryview:
        slot = ticket % self.depth
        if ticket in self._pending:
            _native.check(_native.load().rt_frame_wait_v1(self.ctx.handle, slot), "rt_frame_wait_v1")
            self._pending.discard(ticket)
        return memoryview(self._bufs[slot])

    def drain(self):
        for t in sorted(self._pending):
            self.wait(t)

    def close(self):
        self.drain()
        for b in self._bufs:
            if b is not None:
                _native._PINS.release(b)
        self.ctx.close()
