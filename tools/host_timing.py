"""Host-side breakdown of synchronous render_frame calls ($B200RT_HOST_TIMING:
rt_render_v1 prints setup / enqueue / wait / device times to stderr).

    B200RT_HOST_TIMING=1 python tools/host_timing.py C2 C1 P720
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("B200RT_HOST_TIMING", "1")
import paper_2305_07450_b200 as rt  # noqa: E402

for key in sys.argv[1:] or ["C2"]:
    cfg = rt.CONFIGS[key]
    scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
    fb = rt.Framebuffer.create(cfg.width, cfg.height)
    for _ in range(20):
        rt.render_frame(scene, cam, params, fb)
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        rt.render_frame(scene, cam, params, fb)
        ts.append(time.perf_counter() - t)
    print(f"{key}: render_frame median {1e6 * statistics.median(ts):.1f} us", file=sys.stderr, flush=True)
