"""TEST INFRASTRUCTURE ONLY — ctypes front end of the CPU float64 oracle.

The oracle (``oracle/rt_oracle.c``) restates the reference frame render
(/root/reference/pkg/src/raytracer/renderer.py:45-279 and the @njit helpers
in vecmath.py, camera.py, geometry.py, shading.py) in plain C, float64,
no FMA contraction.  It is pinned bit-exactly against the reference's golden
sha256 (pkg/tests/test_acceptance.py:31) and against fixtures produced by the
reference itself (tests/golden/make_golden.py, tests/test_oracle.py).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module; the product package never does.

All functions take a *packed scene*: a mapping with the reference's
structure-of-arrays layout (geometry.py:162-176, scene.py:100-104):
``kinds`` int32[n], ``positions`` f64[n,3], ``sizes`` f64[n], ``colors``
f64[n,3], ``refls`` f64[n], ``light_pos`` f64[3], ``light_radius``,
``light_color`` f64[3], ``ambient``, ``max_refl``, ``sky`` f32[H,W,3],
``sky_w``, ``sky_h``, ``has_sky``.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "librt_oracle.so")
_lib = None

_d = ctypes.c_double
_i = ctypes.c_int
_p = ctypes.c_void_p


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "rt_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.rto_render.restype = _i
        L.rto_render.argtypes = [_p, _p, _i, _i, _p, _d, _d, _d, _i, _p, _p, _p, _p, _p, _p, _d, _p, _d, _d,
                                 _p, _i, _i, _i, _i, _i, _i, _i, _i]
        L.rto_trace_rays.restype = _i
        L.rto_trace_rays.argtypes = [_p, _p, ctypes.c_long, _p, _i, _p, _p, _p, _p, _p, _p, _d, _p, _d, _d,
                                     _p, _i, _i, _i, _i, _i, _i]
        L.rto_primary_directions.restype = None
        L.rto_primary_directions.argtypes = [_p, _p, ctypes.c_long, _i, _i, _d, _d, _d, _p]
        L.rto_sky_samples.restype = None
        L.rto_sky_samples.argtypes = [_p, ctypes.c_long, _p, _i, _i, _p]
        L.rto_disc_table.restype = None
        L.rto_disc_table.argtypes = [_i, _d, _p]
        L.rto_max_threads.restype = _i
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _scene_arrays(ps):
    kinds = np.ascontiguousarray(ps["kinds"], dtype=np.int32)
    n = kinds.shape[0]
    positions = np.ascontiguousarray(ps["positions"], dtype=np.float64).reshape(n, 3)
    sizes = np.ascontiguousarray(ps["sizes"], dtype=np.float64).reshape(n)
    colors = np.ascontiguousarray(ps["colors"], dtype=np.float64).reshape(n, 3)
    refls = np.ascontiguousarray(ps["refls"], dtype=np.float64).reshape(n)
    light_pos = np.ascontiguousarray(ps["light_pos"], dtype=np.float64)
    light_color = np.ascontiguousarray(ps["light_color"], dtype=np.float64)
    sky = np.ascontiguousarray(ps["sky"], dtype=np.float32)
    # keep-alive tuple, then the argument tail shared by render/trace
    keep = (kinds, positions, sizes, colors, refls, light_pos, light_color, sky)
    args = [n, _ptr(kinds), _ptr(positions), _ptr(sizes), _ptr(colors), _ptr(refls), _ptr(light_pos),
            float(ps["light_radius"]), _ptr(light_color), float(ps["ambient"]), float(ps["max_refl"]),
            _ptr(sky), int(ps["sky_w"]), int(ps["sky_h"]), int(bool(ps["has_sky"]))]
    return keep, args


def viewport_distance(fov_degrees: float) -> float:
    """camera.py:64-67 (host-side, Python math like the reference)."""
    return 1.0 / math.tan(math.radians(fov_degrees) / 2.0)


def render(ps, cam_pos, yaw, pitch, fov, width, height, samples, bounces, *, radiance=False, row0=0,
           row_step=1, threads=0):
    """Reference `render_frame` restated: returns uint32[w*h] (and float64[w*h,3])."""
    L = lib()
    pixels = np.zeros(width * height, dtype=np.uint32)
    rad = np.zeros((width * height, 3), dtype=np.float64) if radiance else None
    cam = np.ascontiguousarray(cam_pos, dtype=np.float64)
    keep, sargs = _scene_arrays(ps)
    rc = L.rto_render(_ptr(pixels), _ptr(rad), width, height, _ptr(cam), float(yaw), float(pitch),
                      viewport_distance(fov), *sargs, int(samples), int(bounces), int(row0), int(row_step),
                      int(threads))
    del keep
    if rc != 0:
        raise ValueError("oracle rejected the render parameters")
    return (pixels, rad) if radiance else pixels


def trace_rays(ps, origins, dirs, samples, bounces, threads=0):
    """Reference `ray_trace_iterative` restated for a batch: float64[n,3]."""
    L = lib()
    o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    d = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
    out = np.zeros_like(o)
    keep, sargs = _scene_arrays(ps)
    rc = L.rto_trace_rays(_ptr(o), _ptr(d), o.shape[0], _ptr(out), *sargs, int(samples), int(bounces),
                          int(threads))
    del keep
    if rc != 0:
        raise ValueError("oracle rejected the trace parameters")
    return out


def primary_directions(xs, ys, width, height, yaw, pitch, fov):
    L = lib()
    xs = np.ascontiguousarray(xs, dtype=np.int32)
    ys = np.ascontiguousarray(ys, dtype=np.int32)
    out = np.zeros((xs.shape[0], 3), dtype=np.float64)
    L.rto_primary_directions(_ptr(xs), _ptr(ys), xs.shape[0], width, height, float(yaw), float(pitch),
                             viewport_distance(fov), _ptr(out))
    return out


def sky_samples(dirs, texels):
    L = lib()
    d = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(texels, dtype=np.float32)
    out = np.zeros_like(d)
    L.rto_sky_samples(_ptr(d), d.shape[0], _ptr(t), t.shape[1], t.shape[0], _ptr(out))
    return out


def disc_table(n, radius):
    out = np.zeros((n, 2), dtype=np.float64)
    lib().rto_disc_table(int(n), float(radius), _ptr(out))
    return out


def max_threads():
    return lib().rto_max_threads()
