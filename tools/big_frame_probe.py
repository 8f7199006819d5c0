"""Frames far larger than the benchmark ones (8K; 8192^2 with 31 bounces, whose
hit slots exceed 31 bits and take the megakernel): they render, and how fast."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_2305_07450_b200 as rt
scene, cam = rt.build_benchmark_scene(), rt.benchmark_camera()
for (w, h, s, b) in ((7680, 4320, 16, 3), (8192, 8192, 8, 31)):
    fb = rt.Framebuffer.create(w, h)
    rt.render_frame(scene, cam, rt.RenderParams(s, b, w, h), fb)  # first call: allocations, pinning
    t = time.perf_counter()
    rt.render_frame(scene, cam, rt.RenderParams(s, b, w, h), fb)
    print(w, h, s, b, "ok", round((time.perf_counter() - t) * 1e3, 1), "ms", "kernel", round(rt.last_kernel_ms(), 2), "ms", hex(int(fb.pixels[w * (h // 2) + w // 2])), flush=True)
