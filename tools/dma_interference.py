"""Does a device-to-host copy running beside a frame slow the frame's kernels?
Device time (CUDA events on the kernels' stream) of one frame
(rt_render_device_v1), of a pure FFMA stream and of an L2 pointer chase —
alone, beside a 64 MB D2H copy (copy engine, into pinned memory) and beside
a device-to-device copy.  Measured on B200: every kernel runs
17-44% slower while a D2H DMA is in flight (the FFMA stream 38%), though
nvml reports 1965 MHz and no throttle reason; a D2D copy costs ~3%."""
import ctypes
import os
import statistics
import time
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2305_07450_b200 as rt  # noqa: E402
from paper_2305_07450_b200 import _native  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "C2"
c = rt.CONFIGS[key]
lib = _native.load()
ctx = _native.Context((0,))
ps = rt.pack_scene(c.scene())
P = _native.ptr
_native.check(lib.rt_set_scene_v1(ctx.handle, ps.n_bodies, P(ps.kinds), P(ps.positions), P(ps.sizes), P(ps.colors),
                                  P(ps.refls), P(ps.light_pos), ps.light_radius, P(ps.light_color), ps.ambient,
                                  ps.max_refl, P(ps.sky), ps.sky_w, ps.sky_h, int(ps.has_sky)), "set_scene")
dev = torch.device("cuda:0")
main = torch.cuda.Stream(dev)
side = torch.cuda.Stream(dev, priority=-5)
out = torch.empty(c.width * c.height, dtype=torch.int32, device=dev)
src = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
dst = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True)
cam = c.camera()
cp = np.array(cam.position, dtype=np.float64)


def frame():
    rc = lib.rt_render_device_v1(ctx.handle, 0, ctypes.c_void_p(out.data_ptr()), c.width, None, c.width, c.height,
                                 P(cp), float(cam.yaw), float(cam.pitch), rt.camera_viewport_distance(cam.fov),
                                 c.samples, c.bounces, 0, 1, 8, 0, ctypes.c_void_p(main.cuda_stream))
    _native.check(rc, "render")


def measure(side_work, n=30):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            side_work()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        frame()
        e1.record(main)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


for _ in range(10):
    frame()
torch.cuda.synchronize()
print(f"{key} frame alone:               {measure(lambda: None):7.1f} us")
print(f"{key} frame beside a D2H DMA:    {measure(lambda: dst.copy_(src, non_blocking=True)):7.1f} us")
print(f"{key} frame beside a D2D copy:    {measure(lambda: src[: 32 << 20].copy_(src[32 << 20:], non_blocking=True)):7.1f} us")

# what kind of work the copy slows: a pure FFMA stream and an L2 pointer chase
from torch.utils.cpp_extension import load_inline  # noqa: E402

src_cu = r"""
#include <cuda_runtime.h>
__global__ void ffma(float *o, int it) { float a = threadIdx.x, b = 1.0001f; for (int i = 0; i < it; i++) { a = fmaf(a, b, 0.5f); a = fmaf(a, b, 0.25f); } if (a == 1.234f) o[0] = a; }
__global__ void chase(const int *n, int *o, int it) { int p = (blockIdx.x * 977 + threadIdx.x * 131) & ((1 << 20) - 1); for (int i = 0; i < it; i++) p = __ldcg(n + p); if (p == -7) o[0] = p; }
void run_ffma(long o, int it, long st) { ffma<<<148 * 8, 256, 0, (cudaStream_t)st>>>((float *)o, it); }
void run_chase(long n, long o, int it, long st) { chase<<<148 * 8, 256, 0, (cudaStream_t)st>>>((const int *)n, (int *)o, it); }
"""
mod = load_inline("interf", cpp_sources="void run_ffma(long o, int it, long st); void run_chase(long n, long o, int it, long st);",
                  cuda_sources=src_cu, functions=["run_ffma", "run_chase"], extra_cuda_cflags=["-O3", "-gencode", "arch=compute_100a,code=sm_100a"], verbose=False)
nxt = torch.randint(0, 1 << 20, (1 << 20,), dtype=torch.int32, device=dev)
o = torch.zeros(4, dtype=torch.int32, device=dev)


def timed(fn, side_work, n=20, delay=0.0):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            side_work()
        if delay:
            t = time.perf_counter()
            while time.perf_counter() - t < delay:
                pass
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        fn()
        e1.record(main)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)


ff = lambda: mod.run_ffma(o.data_ptr(), 4000, main.cuda_stream)  # noqa: E731
ch = lambda: mod.run_chase(nxt.data_ptr(), o.data_ptr(), 200, main.cuda_stream)  # noqa: E731
dma = lambda: dst.copy_(src, non_blocking=True)  # noqa: E731
for name, fn in (("FFMA stream", ff), ("L2 pointer chase", ch)):
    fn()
    print(f"{name:18s} alone {timed(fn, lambda: None):7.1f} us, beside D2H DMA {timed(fn, dma):7.1f} us, "
          f"DMA started 200 us before {timed(fn, dma, delay=2e-4):7.1f} us")
print(f"{key} frame, DMA started 200 us before: {timed(frame, dma, delay=2e-4):7.1f} us")
