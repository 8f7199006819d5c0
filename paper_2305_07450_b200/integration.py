"""Swap the reference renderer for the B200 one inside an existing program.

The reference's callers import `render_frame` by name at import time —
`raytracer.bench` (bench.py:15), `raytracer.cli` (cli.py:17) and
`raytracer.server` (server.py:43) — so rebinding `raytracer.renderer`
alone would leave them on the numba path.  `install()` rebinds every one.

It also replaces the frame server's step, `FrameLoop.tick`
(server.py:276-289): the reference renders into the loop's 0xAARRGGBB
framebuffer and then re-packs every pixel on the host into the RAYF
message (`encode_frame`, server.py:56-64).  The B200 tick renders the
message itself — the kernels pack R,G,B,A into a page-locked buffer laid out
header-then-payload (stream.FrameEncoder) — and hands the same bytes to every
`FrameSink`; there is no host-side encode pass.  `loop.fb` stays readable:
it is filled from the last message on first access after a tick (lazily, so
a loop nobody inspects never pays for it).
"""

from __future__ import annotations

import functools
import importlib
import os
import sys

from . import _native
from . import renderer as _b200

_TARGETS = ("raytracer.renderer", "raytracer.bench", "raytracer.cli", "raytracer.server")
_saved = {}
_MISSING = object()


def _b200_tick(precision):
    """FrameLoop.tick (server.py:276-289) with the render and the encode on
    the GPU: apply controls, physics step, RAYF message, broadcast."""

    def tick(self):
        self._drain_mailbox()
        if self.paused:
            return None
        server = sys.modules[type(self).__module__]
        if self.physics is not None:
            server.verlet_step(self.physics, self.scene.bodies, self.floor_height, server.FIXED_DT)
        enc = self.__dict__.get("_b200_encoder")
        if enc is None:
            from .stream import FrameEncoder

            dev = int(os.environ.get("LOCAL_RANK", "0")) % max(1, _native.device_count())
            enc = self.__dict__["_b200_encoder"] = FrameEncoder(dev)
        self.frame_id += 1
        payload = bytes(enc.render(self.scene, self.camera, self.params, self.frame_id, workers=self.workers,
                                   precision=precision))
        self.__dict__["_b200_payload"] = payload  # loop.fb is derived from it on demand
        with self._sinks_lock:
            for sink in self._sinks:
                sink.offer(payload)
        return payload

    return tick


def _fb_get(self):
    fb = self.__dict__["_b200_fb"]
    payload = self.__dict__.pop("_b200_payload", None)
    if payload is not None and len(payload) == 16 + 4 * fb.pixels.size:
        from .stream import HEADER
        import numpy as np

        rgba = np.frombuffer(payload, dtype=np.uint8, offset=HEADER.size).reshape(-1, 4)
        fb.pixels.view(np.uint8).reshape(-1, 4)[:] = rgba[:, [2, 1, 0, 3]]
    return fb


def _fb_set(self, fb):
    self.__dict__["_b200_fb"] = fb
    self.__dict__.pop("_b200_payload", None)


def install(precision=None, package: str = "raytracer", frame_loop: bool = True):
    """Point the reference package's render entry points at libb200rt, and
    (frame_loop) its FrameLoop.tick at the GPU-encoding tick.

    Returns the list of modules patched.  `uninstall()` restores them."""
    if precision is None:
        fn, ray = _b200.render_frame, _b200.ray_trace_iterative
    else:
        fn = functools.partial(_b200.render_frame, precision=precision)
        ray = functools.partial(_b200.ray_trace_iterative, precision=precision)
    patched = []
    for name in _TARGETS:
        name = name.replace("raytracer", package, 1)
        try:
            mod = sys.modules.get(name) or importlib.import_module(name)
        except ImportError:
            continue
        for attr, new in (("render_frame", fn), ("ray_trace_iterative", ray)):
            if hasattr(mod, attr):
                _saved.setdefault((name, attr), getattr(mod, attr))
                setattr(mod, attr, new)
        loop_cls = getattr(mod, "FrameLoop", None)
        if frame_loop and isinstance(loop_cls, type) and hasattr(loop_cls, "tick"):
            for attr, new in (("tick", _b200_tick(precision)), ("fb", property(_fb_get, _fb_set))):
                _saved.setdefault((name, "FrameLoop." + attr), loop_cls.__dict__.get(attr, _MISSING))
                setattr(loop_cls, attr, new)
        patched.append(name)
    return patched


def uninstall():
    for (name, attr), old in list(_saved.items()):
        mod = sys.modules.get(name)
        if mod is None:
            continue
        obj = mod
        if attr.startswith("FrameLoop."):
            obj, attr = mod.FrameLoop, attr.split(".", 1)[1]
        if old is _MISSING:
            delattr(obj, attr)
        else:
            setattr(obj, attr, old)
    _saved.clear()
