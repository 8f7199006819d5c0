"""The reference's renderer API, executed by the sm_100a kernels of libb200rt.

Drop-in for /root/reference/pkg/src/raytracer/renderer.py: same names,
signatures, argument meaning and errors —

    render_frame(scene, cam, params, out, workers=None)     renderer.py:316-349
    ray_trace_iterative(ray, scene, params) -> (r, g, b)    renderer.py:303-313
    skybox_sample(direction, sky) -> (r, g, b)              renderer.py:77-79
    pack_color(c) -> int                                    renderer.py:53-57
    MAX_BOUNCE_LIMIT, REFLECT_EPS                           renderer.py:33-36

plus the batched `trace_rays` that backs `ray_trace_iterative`.  Inputs are
duck-typed, so the reference's own Scene/Camera/RenderParams/Framebuffer
objects work unchanged.

`workers` keeps its meaning — how many parallel workers split the frame —
and becomes the number of row-block partitions, spread over up to that many
GPUs; as in the reference the pixels do not depend on it.

`precision` (keyword, default "fp32", or $B200RT_PRECISION as the first frame finds it) picks the FP32
product kernel or the FP64 validation kernel that reproduces the reference
bit for bit.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native
from .model import MAX_BOUNCE_LIMIT, REFLECT_EPS, camera_viewport_distance, pack_scene, scene_argv

__all__ = [
    "MAX_BOUNCE_LIMIT",
    "REFLECT_EPS",
    "render_frame",
    "ray_trace_iterative",
    "trace_rays",
    "skybox_sample",
    "pack_color",
    "default_precision",
    "FramePipeline",
]

_PIN_MIN_BYTES = 1 << 18  # page-lock framebuffers of >= 256 KiB


_FAST = []  # [module or None]: the CPython fast path (csrc/pyfast.c), loaded once


def _fast():
    """The CPython fast path (scene packing + the C-ABI call without ctypes
    marshalling), or None when it is not built: the ctypes path serves."""
    if not _FAST:
        try:
            from . import _pyfast
        except ImportError:
            _FAST.append(None)
        else:
            lib = _native.load()
            _pyfast.set_entry_points(ctypes.cast(lib.rt_render_v1, ctypes.c_void_p).value,
                                     ctypes.cast(lib.rt_render_async_v1, ctypes.c_void_p).value)
            _FAST.append(_pyfast)
    return _FAST[0]


def default_precision() -> str:
    return os.environ.get("B200RT_PRECISION", "fp32")


_DEFAULT_PREC = []  # $B200RT_PRECISION, read on the first frame (an environ lookup costs ~1 us)


def _prec(precision) -> int:
    if precision is None:
        if not _DEFAULT_PREC:
            _DEFAULT_PREC.append(_prec(default_precision()))
        return _DEFAULT_PREC[0]
    if precision not in _native.PRECISIONS:
        raise ValueError(f"precision must be one of {sorted(_native.PRECISIONS)}, got {precision!r}")
    return _native.PRECISIONS[precision]


def _scene_argv(ps):
    argv = getattr(ps, "argv", None)
    if argv is not None:  # pack_scene's precomputed addresses
        return argv
    P = _native.ptr
    return [
        ps.n_bodies, P(ps.kinds), P(ps.positions), P(ps.sizes), P(ps.colors), P(ps.refls), P(ps.light_pos),
        ps.light_radius, P(ps.light_color), ps.ambient, ps.max_refl, P(ps.sky), ps.sky_w, ps.sky_h,
        int(ps.has_sky),
    ]


def pack_color(c) -> int:
    """Pack a [0,1] RGB triple into 0xAARRGGBB, alpha opaque (renderer.py:45-57)."""
    if not all(0.0 <= ch <= 1.0 for ch in c):
        raise ValueError(f"channels must be in [0, 1], got {c}")
    r = int(c[0] * 255.0 + 0.5)
    g = int(c[1] * 255.0 + 0.5)
    b = int(c[2] * 255.0 + 0.5)
    return 0xFF000000 | (r << 16) | (g << 8) | b


def render_frame(scene, cam, params, out, workers=None, *, precision=None, radiance=None):
    """Render one frame into `out`; pixel (x, y) lands at index x + y * width.

    `workers` picks the number of row-block partitions (and GPUs, up to the
    number visible); the result does not depend on it.  `radiance`, when
    given, is filled with the pre-quantisation colours: float32[w*h, 3] for
    precision "fp32", float64[w*h, 3] for "fp64".
    """
    if (out.width, out.height) != (params.width, params.height):
        raise ValueError(
            f"framebuffer {out.width}x{out.height} does not match params {params.width}x{params.height}"
        )
    if params.bounce_limit > MAX_BOUNCE_LIMIT:
        raise ValueError(f"bounce limit capped at {MAX_BOUNCE_LIMIT}")
    prec = _prec(precision)
    pixels = out.pixels
    if pixels.dtype != np.uint32 or not pixels.flags.c_contiguous or pixels.size != params.width * params.height:
        raise ValueError("framebuffer pixels must be a contiguous uint32 array of width * height")
    if radiance is not None:
        want = np.float64 if prec == _native.RT_PREC_FP64 else np.float32
        if radiance.dtype != want or not radiance.flags.c_contiguous or radiance.size != 3 * pixels.size:
            raise ValueError(f"radiance must be a contiguous {np.dtype(want).name}[w*h, 3] array")
    n_parts = 1 if workers is None else int(workers)
    if n_parts < 1:
        raise ValueError("workers must be >= 1")
    ctx = _native.context(n_parts)
    if pixels.nbytes >= _PIN_MIN_BYTES:
        ctx.pin(pixels)
    fast = _fast()
    rc = None
    if fast is not None:
        rc = fast.render(ctx.handle.value, ctx.address(pixels), 0 if radiance is None else _native.ptr(radiance).value,
                         int(params.width), int(params.height), cam.position, float(cam.yaw), float(cam.pitch),
                         camera_viewport_distance(cam.fov), scene, int(params.shadow_samples),
                         int(params.bounce_limit), n_parts, prec)
    if rc is None:  # no fast path, or a scene it does not take: the ctypes path (and its errors)
        argv, keep = scene_argv(scene)
        cp = cam.position
        cam_pos = (ctypes.c_double * 3)(cp[0], cp[1], cp[2])
        rc = _native.load().rt_render_v1(
            ctx.handle, ctx.address(pixels), _native.ptr(radiance), int(params.width), int(params.height),
            cam_pos, float(cam.yaw), float(cam.pitch), camera_viewport_distance(cam.fov),
            *argv, int(params.shadow_samples), int(params.bounce_limit), n_parts, prec,
        )
        del keep
    _native.check(rc, "rt_render_v1")


class FramePipeline:
    """Frames rendered back to back, each frame's device-to-host copy
    overlapping the next frame's kernels — the frame server's loop
    (`FrameLoop.tick`, server.py:276-289) without the idle PCIe time.

    `submit(scene, cam, params, out)` validates like `render_frame`, enqueues
    the frame and returns a ticket; `wait(ticket)` returns `out` once its
    pixels are in (bit for bit what `render_frame` gives).  At most `depth`
    (2-4) frames are in flight; submitting more waits for the oldest.  `out`
    must not be touched between submit and wait."""

    def __init__(self, depth: int = 2, *, precision=None):
        if not 1 <= int(depth) <= 4:
            raise ValueError("depth must be 1-4")
        self.depth = int(depth)
        self.precision = precision
        if _native.device_count() < 1:
            raise _native.NativeError("no CUDA device visible: the b200rt frame render has no CPU path")
        # its own context (streams, frame slots); its framebuffers are held in
        # the pin registry while their copies are in flight, so no other
        # caller's pinning evicts them (_native._Pins)
        dev = int(os.environ.get("LOCAL_RANK", "0")) % _native.device_count()
        self.ctx = _native.Context((dev,))
        for k, v in _native.get_options().items():
            self.ctx.set_option(k, v)
        self._next = 0
        self._pending = {}  # ticket -> framebuffer

    def submit(self, scene, cam, params, out) -> int:
        if (out.width, out.height) != (params.width, params.height):
            raise ValueError(
                f"framebuffer {out.width}x{out.height} does not match params {params.width}x{params.height}"
            )
        if params.bounce_limit > MAX_BOUNCE_LIMIT:
            raise ValueError(f"bounce limit capped at {MAX_BOUNCE_LIMIT}")
        pixels = out.pixels
        if pixels.dtype != np.uint32 or not pixels.flags.c_contiguous or pixels.size != params.width * params.height:
            raise ValueError("framebuffer pixels must be a contiguous uint32 array of width * height")
        prec = _prec(self.precision)
        ticket = self._next
        oldest = ticket - self.depth
        if oldest in self._pending:
            self.wait(oldest)
        self.ctx.pin(pixels, max_pinned=2 * self.depth + 2)
        fast = _fast()
        rc = None
        if fast is not None:
            rc = fast.render_async(self.ctx.handle.value, ticket % self.depth, self.ctx.address(pixels),
                                   int(params.width), int(params.height), cam.position, float(cam.yaw),
                                   float(cam.pitch), camera_viewport_distance(cam.fov), scene,
                                   int(params.shadow_samples), int(params.bounce_limit), prec)
        if rc is None:
            argv, keep = scene_argv(scene)
            cp = cam.position
            cam_pos = (ctypes.c_double * 3)(cp[0], cp[1], cp[2])
            rc = _native.load().rt_render_async_v1(
                self.ctx.handle, ticket % self.depth, self.ctx.address(pixels), int(params.width),
                int(params.height), cam_pos, float(cam.yaw), float(cam.pitch), camera_viewport_distance(cam.fov),
                *argv, int(params.shadow_samples), int(params.bounce_limit), prec,
            )
            del keep
        _native.check(rc, "rt_render_async_v1")
        _native._PINS.hold(pixels)
        self._pending[ticket] = out
        self._next += 1
        return ticket

    def wait(self, ticket: int):
        out = self._pending.pop(ticket)
        try:
            _native.check(_native.load().rt_frame_wait_v1(self.ctx.handle, ticket % self.depth), "rt_frame_wait_v1")
        finally:
            _native._PINS.release(out.pixels)
        return out

    def drain(self):
        for t in sorted(self._pending):
            self.wait(t)

    def close(self):
        self.drain()
        self.ctx.close()


def trace_rays(origins, directions, scene, params, *, precision=None) -> np.ndarray:
    """Batched `ray_trace_iterative`: colours of rays (origins[i], directions[i]).

    Returns float32[n, 3] ("fp32") or float64[n, 3] ("fp64")."""
    if params.bounce_limit > MAX_BOUNCE_LIMIT:
        raise ValueError(f"bounce limit capped at {MAX_BOUNCE_LIMIT}")
    prec = _prec(precision)
    o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    d = np.ascontiguousarray(directions, dtype=np.float64).reshape(-1, 3)
    if o.shape != d.shape:
        raise ValueError("origins and directions must have the same shape")
    out = np.zeros(o.shape, dtype=np.float64 if prec == _native.RT_PREC_FP64 else np.float32)
    ctx = _native.context(1)
    ps = pack_scene(scene)
    rc = _native.load().rt_trace_rays_v1(
        ctx.handle, _native.ptr(o), _native.ptr(d), o.shape[0], _native.ptr(out), *_scene_argv(ps),
        int(params.shadow_samples), int(params.bounce_limit), prec,
    )
    _native.check(rc, "rt_trace_rays_v1")
    return out


def ray_trace_iterative(ray, scene, params, *, precision=None):
    """Colour gathered by one ray under the scene's light and bounce budget
    (renderer.py:303-313); a tuple of Python floats."""
    if params.bounce_limit > MAX_BOUNCE_LIMIT:
        raise ValueError(f"bounce limit capped at {MAX_BOUNCE_LIMIT}")
    c = trace_rays([ray.origin], [ray.direction], scene, params, precision=precision)[0]
    return (float(c[0]), float(c[1]), float(c[2]))


def skybox_sample(direction, sky):
    """Equirectangular nearest-texel lookup, clamped to [0, 1] (renderer.py:60-79).
    Evaluated on the GPU in float64, bit-identical to the reference."""
    d = np.ascontiguousarray(direction, dtype=np.float64).reshape(-1, 3)
    texels = np.ascontiguousarray(sky.texels, dtype=np.float32)
    out = np.zeros(d.shape, dtype=np.float64)
    ctx = _native.context(1)
    rc = _native.load().rt_sky_sample_v1(ctx.handle, _native.ptr(d), d.shape[0], _native.ptr(out),
                                         _native.ptr(texels), int(sky.width), int(sky.height))
    _native.check(rc, "rt_sky_sample_v1")
    if np.ndim(direction) == 1 or (len(direction) == 3 and np.ndim(direction[0]) == 0):
        return (float(out[0, 0]), float(out[0, 1]), float(out[0, 2]))
    return out


def last_kernel_ms(workers=None) -> float:
    """Device time of the render kernels of the last call (CUDA events)."""
    return _native.context(1 if workers is None else int(workers)).last_kernel_ms()
