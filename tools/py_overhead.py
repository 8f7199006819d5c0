"""Where render_frame's host time goes outside the C call (C2)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_07450_b200 as rt  # noqa: E402
from paper_2305_07450_b200 import _native, renderer  # noqa: E402
from paper_2305_07450_b200.model import camera_viewport_distance  # noqa: E402

cfg = rt.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
fb = rt.Framebuffer.create(cfg.width, cfg.height)
ctx = _native.context(1)
for _ in range(20):
    rt.render_frame(scene, cam, params, fb)


def t(fn, n=200):
    ts = []
    for _ in range(n):
        a = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - a)
    return 1e6 * statistics.median(ts)


fast = renderer._fast()
args = lambda: (ctx.handle.value, ctx.address(fb.pixels), 0, int(params.width), int(params.height), cam.position,  # noqa: E731
                float(cam.yaw), float(cam.pitch), camera_viewport_distance(cam.fov), scene,
                int(params.shadow_samples), int(params.bounce_limit), 1, 0)
print(f"render_frame          {t(lambda: rt.render_frame(scene, cam, params, fb)):8.1f} us")
print(f"fast.render (C call)  {t(lambda: fast.render(*args())):8.1f} us")
print(f"ctx.pin               {t(lambda: ctx.pin(fb.pixels)):8.2f} us")
print(f"_native.context(1)    {t(lambda: _native.context(1)):8.2f} us")
print(f"_prec(None)           {t(lambda: renderer._prec(None)):8.2f} us")
print(f"viewport distance     {t(lambda: camera_viewport_distance(cam.fov)):8.2f} us")
