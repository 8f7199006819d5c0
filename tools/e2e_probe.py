"""Where an end-to-end frame goes: the Python entry (render_frame), the bare
C ABI call with pre-packed arguments, and the device time of the launch
sequence (rt_last_kernel_ms), per row-band count."""

import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


import paper_2305_07450_b200 as rt  # noqa: E402
from paper_2305_07450_b200 import _native, renderer  # noqa: E402


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "C2"
    cfg = rt.CONFIGS[key]
    scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
    fb = rt.Framebuffer.create(cfg.width, cfg.height)
    ctx = _native.context(1)
    ctx.pin(fb.pixels)
    lib = _native.load()
    ps = rt.pack_scene(scene)
    cp = (ctypes.c_double * 3)(*cam.position)
    vd = rt.camera_viewport_distance(cam.fov)
    argv = renderer._scene_argv(ps)
    px = ctx.address(fb.pixels)

    def bare():
        rc = lib.rt_render_v1(ctx.handle, px, None, cfg.width, cfg.height, cp, float(cam.yaw), float(cam.pitch), vd,
                              *argv, params.shadow_samples, params.bounce_limit, 1, 0)
        assert rc == 0

    for bands in [int(b) for b in os.environ.get("BANDS", "1,2,3,4").split(",")]:
        ctx.set_option("bands", bands)
        for _ in range(20):
            bare()
        tb, tp, dev = [], [], []
        for _ in range(200):
            t = time.perf_counter()
            bare()
            tb.append(time.perf_counter() - t)
            dev.append(ctx.last_kernel_ms())
        for _ in range(200):
            t = time.perf_counter()
            rt.render_frame(scene, cam, params, fb)
            tp.append(time.perf_counter() - t)
        m = lambda v: 1e6 * statistics.median(v)  # noqa: E731
        print(f"{key} bands={bands}: render_frame {m(tp):.1f} us | bare C call {m(tb):.1f} us | "
              f"device launch->last kernel {1e3 * statistics.median(dev):.1f} us", flush=True)
    ctx.set_option("bands", 0)


if __name__ == "__main__":
    main()
