"""ctypes binding of libb200rt.so (the C ABI declared in include/b200rt.h).

There is no CPU fallback: if the library is missing, or no CUDA device is
visible, every compute call raises.  ctypes.CDLL releases the GIL for the
duration of each call, like the reference's nogil=True kernel
(/root/reference/pkg/src/raytracer/renderer.py:227).
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("B200RT_LIB") or os.path.join(_PKG, "libb200rt.so")

RT_OK = 0
RT_ERR_INVALID = -1
RT_ERR_CUDA = -2
RT_ERR_NO_DEVICE = -3
RT_ERR_NOMEM = -4
RT_ERR_LIMIT = -5
RT_ALREADY_REGISTERED = 1
RT_PREC_FP32 = 0
RT_PREC_FP64 = 1
PRECISIONS = {"fp32": RT_PREC_FP32, "fp64": RT_PREC_FP64}

_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_d = ctypes.c_double
_p = ctypes.c_void_p

# name -> (restype, argtypes); the exact export list of include/b200rt.h
SIGNATURES = {
    "rt_version": (ctypes.c_int, []),
    "rt_last_error": (ctypes.c_char_p, []),
    "rt_device_count": (ctypes.c_int, [_p]),
    "rt_ctx_create": (ctypes.c_int, [_p, _p, _i32]),
    "rt_ctx_destroy": (ctypes.c_int, [_p]),
    "rt_set_scene_v1": (ctypes.c_int, [_p, _i32, _p, _p, _p, _p, _p, _p, _d, _p, _d, _d, _p, _i32, _i32, _i32]),
    "rt_render_v1": (ctypes.c_int, [_p, _p, _p, _i32, _i32, _p, _d, _d, _d, _i32, _p, _p, _p, _p, _p, _p, _d, _p,
                                    _d, _d, _p, _i32, _i32, _i32, _i32, _i32, _i32, _i32]),
    "rt_render_device_v1": (ctypes.c_int, [_p, _i32, _p, _i64, _p, _i32, _i32, _p, _d, _d, _d, _i32, _i32, _i32,
                                           _i32, _i32, _i32, _p]),
    "rt_render_async_v1": (ctypes.c_int, [_p, _i32, _p, _i32, _i32, _p, _d, _d, _d, _i32, _p, _p, _p, _p, _p, _p, _d,
                                          _p, _d, _d, _p, _i32, _i32, _i32, _i32, _i32, _i32]),
    "rt_frame_wait_v1": (ctypes.c_int, [_p, _i32]),
    "rt_trace_rays_v1": (ctypes.c_int, [_p, _p, _p, _i64, _p, _i32, _p, _p, _p, _p, _p, _p, _d, _p, _d, _d, _p,
                                        _i32, _i32, _i32, _i32, _i32, _i32]),
    "rt_sky_sample_v1": (ctypes.c_int, [_p, _p, _i64, _p, _p, _i32, _i32]),
    "rt_host_register": (ctypes.c_int, [_p, _p, ctypes.c_size_t]),
    "rt_host_unregister": (ctypes.c_int, [_p, _p]),
    "rt_set_option": (ctypes.c_int, [_p, ctypes.c_char_p, _i32]),
    "rt_work_counts": (ctypes.c_int, [_p, _p, _i32, _i32]),
    "rt_last_kernel_ms": (ctypes.c_int, [_p, _p]),
    "rt_last_d2h_bytes": (ctypes.c_int, [_p, _p]),
    "rt_frame_expand_v1": (ctypes.c_int, [_p, _i32, _i32, _p, ctypes.c_int64, _i32, _p]),
    "rt_phase_ms": (ctypes.c_int, [_p, _p, _i32]),
    "rt_band_times_ms": (ctypes.c_int, [_p, _p, _i32]),
    "rt_launch_count": (ctypes.c_int, [_p, _p]),
    "rt_ipc_get_handle": (ctypes.c_int, [_p, _p]),
    "rt_ipc_open": (ctypes.c_int, [_p, _p]),
    "rt_ipc_close": (ctypes.c_int, [_p]),
    "rt_copy_to_host": (ctypes.c_int, [_p, _i32, _p, _p, ctypes.c_size_t, _p]),
    "rt_copy_partition_to_host": (ctypes.c_int, [_p, _i32, _p, _p, _i32, _i32, _i32, _i32, _i32, _p]),
    "rt_device_malloc": (ctypes.c_int, [_i32, ctypes.c_size_t, _p]),
    "rt_device_free": (ctypes.c_int, [_p]),
    "rt_fp32_peak_tflops": (ctypes.c_int, [_i32, _p]),
}

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    """A CUDA-side failure reported by libb200rt."""


def load():
    """Load libb200rt.so (in-tree); raise if it is not built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is not built: run `python -m paper_2305_07450_b200.build` "
                    "(there is no CPU fallback for the frame render)"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    return (load().rt_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str):
    if rc == RT_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc in (RT_ERR_INVALID, RT_ERR_LIMIT):
        raise ValueError(msg)
    raise NativeError(msg)


def ptr(a) -> ctypes.c_void_p | None:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return ctypes.c_void_p(a.ctypes.data)
    return ctypes.c_void_p(int(a))


def device_count() -> int:
    n = _i32(0)
    check(load().rt_device_count(ctypes.byref(n)), "rt_device_count")
    return n.value


class Context:
    """One rt_ctx: a stream, scene cache and staging framebuffer per device."""

    def __init__(self, devices=(0,)):
        self.devices = tuple(int(d) for d in devices)
        lib = load()
        h = ctypes.c_void_p()
        arr = (_i32 * len(self.devices))(*self.devices)
        check(lib.rt_ctx_create(ctypes.byref(h), arr, len(self.devices)), "rt_ctx_create")
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            load().rt_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- pinned host framebuffers (the process-wide registry, _PINS) ------------
    def pin(self, arr: np.ndarray, max_pinned: int = 4) -> bool:
        """Page-lock `arr` so the frame copy runs at PCIe speed (see _Pins)."""
        return _PINS.pin(arr, max_pinned)

    def address(self, arr: np.ndarray) -> int:
        """Device-visible host address of `arr` (mapped: the host address)."""
        return arr.__array_interface__["data"][0]

    def unpin(self, arr: np.ndarray) -> None:
        """Release a buffer page-locked by pin()."""
        _PINS.unpin(arr)

    def set_option(self, name: str, value) -> None:
        check(load().rt_set_option(self.handle, name.encode(), int(value)), "rt_set_option")

    def work_counts(self, reset: bool = True) -> dict:
        keys = ("hits", "cull_tests", "sampled_hits", "shadow_rays", "sphere_tests", "plane_tests", "trace_rays",
                "trace_tests", "trace_unculled_warps", "conic_hits", "conic_tests", "lane_hits", "conic_z_tests")
        arr = (ctypes.c_uint64 * len(keys))()
        check(load().rt_work_counts(self.handle, arr, len(keys), int(reset)), "rt_work_counts")
        return dict(zip(keys, (int(v) for v in arr)))

    def last_kernel_ms(self) -> float:
        v = ctypes.c_float(0)
        check(load().rt_last_kernel_ms(self.handle, ctypes.byref(v)), "rt_last_kernel_ms")
        return float(v.value)

    def last_d2h_bytes(self) -> int:
        v = ctypes.c_int64(0)
        check(load().rt_last_d2h_bytes(self.handle, ctypes.byref(v)), "rt_last_d2h_bytes")
        return int(v.value)

    def phase_ms(self) -> dict:
        arr = (ctypes.c_float * 4)()
        check(load().rt_phase_ms(self.handle, arr, 4), "rt_phase_ms")
        return dict(zip(("trace", "classify", "shadow", "shade"), (float(v) for v in arr)))

    def band_times_ms(self) -> list:
        """[(kernels_end_ms, copy_end_ms)] per row band of the last frame (option "band_times")."""
        arr = (ctypes.c_float * 16)()
        n = load().rt_band_times_ms(self.handle, arr, 16)
        check(min(n, 0), "rt_band_times_ms")
        return [(float(arr[2 * k]), float(arr[2 * k + 1])) for k in range(n)]

    def launch_count(self) -> int:
        v = _i64(0)
        check(load().rt_launch_count(self.handle, ctypes.byref(v)), "rt_launch_count")
        return int(v.value)


class _Pins:
    """Process-wide registry of page-locked host framebuffers.

    A registration (cudaHostRegister, portable + mapped) belongs to the
    process, not to a context, so one registry serves render_frame,
    FramePipeline and the frame encoders alike:

    * it holds only a weak reference: when the caller drops a framebuffer its
      pages are unlocked (weakref callback, before numpy frees the memory) —
      nothing is retained;
    * at most `max_pinned` live buffers stay locked, least recently used
      first out — but never one that is `hold()`-ed (a device-to-host copy
      into it is in flight: FramePipeline / PipelinedFrameEncoder);
    * a range some other code already page-locked (RT_ALREADY_REGISTERED) is
      used as is and never unregistered here.
    """

    def __init__(self):
        self._lock = threading.RLock()
        self._entries = {}  # address -> [weakref, nbytes, holds, owned]
        self._order = []    # addresses, least recently used first
        self._last = None   # weakref of the array pinned or hit last (lock-free fast path)

    def _drop(self, addr):
        e = self._entries.pop(addr, None)
        if e is not None and self._last is e[0]:
            self._last = None
        if addr in self._order:
            self._order.remove(addr)
        if e is not None and e[3]:
            if load is None or ctypes is None:  # interpreter shutdown: the process releases the pages
                return
            load().rt_host_unregister(None, ctypes.c_void_p(addr))

    def _finalize(self, addr, ref):
        with self._lock:
            e = self._entries.get(addr)
            if e is not None and e[0] is ref:
                self._drop(addr)

    def pin(self, arr: np.ndarray, max_pinned: int = 4) -> bool:
        last = self._last
        if last is not None and last() is arr:  # the same framebuffer as the last frame's
            return True
        addr = arr.__array_interface__["data"][0]
        with self._lock:
            e = self._entries.get(addr)
            if e is not None:
                if e[0]() is arr and e[1] >= arr.nbytes:
                    self._order.remove(addr)
                    self._order.append(addr)
                    self._last = e[0]
                    return True
                if e[2] == 0:
                    self._drop(addr)  # a different or larger array now lives here
                else:
                    return False
            rc = load().rt_host_register(None, ptr(arr), arr.nbytes)
            if rc < 0:
                return False
            ref = weakref.ref(arr, lambda r, a=addr: self._finalize(a, r))
            self._entries[addr] = [ref, arr.nbytes, 0, rc == RT_OK]
            self._order.append(addr)
            self._last = ref
            for old in list(self._order):
                if len(self._order) <= max_pinned:
                    break
                if old != addr and self._entries[old][2] == 0:
                    self._drop(old)
            return True

    def unpin(self, arr: np.ndarray) -> None:
        addr = arr.__array_interface__["data"][0]
        with self._lock:
            e = self._entries.get(addr)
            if e is not None and e[0]() is arr:
                if e[2] > 0:
                    raise RuntimeError("framebuffer has a copy in flight: wait for it before unpinning")
                self._drop(addr)

    def hold(self, arr: np.ndarray) -> None:
        """Mark a copy into `arr` in flight: it is not evicted until release()."""
        with self._lock:
            e = self._entries.get(arr.__array_interface__["data"][0])
            if e is not None:
                e[2] += 1

    def release(self, arr: np.ndarray) -> None:
        with self._lock:
            e = self._entries.get(arr.__array_interface__["data"][0])
            if e is not None and e[2] > 0:
                e[2] -= 1

    def pinned(self, arr: np.ndarray) -> bool:
        with self._lock:
            e = self._entries.get(arr.__array_interface__["data"][0])
            return e is not None and e[0]() is arr

    def count(self) -> int:
        with self._lock:
            return len(self._entries)


_PINS = _Pins()

_contexts = {}
_ctx_lock = threading.Lock()
_options = {}  # execution options applied to every context (rt_set_option)


def set_options(**opts) -> None:
    """Execution options for every context, present and future:
    wave (bool), cull (bool), conic (bool), count_work (bool), bands (0-8) — see
    include/b200rt.h (rt_set_option)."""
    with _ctx_lock:
        _options.update({k: int(v) for k, v in opts.items()})
        for ctx in _contexts.values():
            for k, v in opts.items():
                ctx.set_option(k, v)


def get_options() -> dict:
    return dict(_options)


_ctx_fast = {}  # requested device count -> its context (a render's first lookup)


def context(n_devices: int = 1) -> Context:
    """Process-wide context over n visible devices (clamped), starting at this
    process's local rank ($LOCAL_RANK, as set by torchrun) so that one process
    per GPU renders on its own GPU."""
    ctx = _ctx_fast.get(n_devices)
    if ctx is not None:
        return ctx
    n_vis = device_count()
    if n_vis < 1:
        raise NativeError("no CUDA device visible: the b200rt frame render has no CPU path")
    n = max(1, min(int(n_devices), n_vis))
    first = int(os.environ.get("LOCAL_RANK", "0")) % n_vis
    with _ctx_lock:
        ctx = _contexts.get(n)
        if ctx is None:
            ctx = Context(tuple((first + i) % n_vis for i in range(n)))
            for k, v in _options.items():
                ctx.set_option(k, v)
            _contexts[n] = ctx
        _ctx_fast[n_devices] = ctx
        return ctx


def fp32_peak_tflops(device: int = 0) -> float:
    v = _d(0)
    check(load().rt_fp32_peak_tflops(int(device), ctypes.byref(v)), "rt_fp32_peak_tflops")
    return float(v.value)
