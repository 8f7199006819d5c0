"""Row-band timeline of one synchronous end-to-end frame: for each band count
and first-band share, the bare C call's wall time and, per band, when its
kernels and its device-to-host copy end (option "band_times")."""

import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


import paper_2305_07450_b200 as rt  # noqa: E402
from paper_2305_07450_b200 import _native, renderer  # noqa: E402


def main():
    keys = sys.argv[1:] or ["C2"]
    ctx = _native.context(1)
    lib = _native.load()
    for key in keys:
        cfg = rt.CONFIGS[key]
        scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
        fb = rt.Framebuffer.create(cfg.width, cfg.height)
        ctx.pin(fb.pixels)
        ps = rt.pack_scene(scene)
        cp = (ctypes.c_double * 3)(*cam.position)
        vd = rt.camera_viewport_distance(cam.fov)
        argv = renderer._scene_argv(ps)
        px = ctx.address(fb.pixels)

        def bare():
            rc = lib.rt_render_v1(ctx.handle, px, None, cfg.width, cfg.height, cp, float(cam.yaw), float(cam.pitch),
                                  vd, *argv, params.shadow_samples, params.bounce_limit, 1, 0)
            assert rc == 0

        ref = None
        specs = os.environ.get("SPLITS", "1:0,2:0,2:550,3:0,4:0,4:450,6:0")
        for spec in specs.split(","):
            bands, first = (int(v) for v in spec.split(":"))
            ctx.set_option("bands", bands)
            ctx.set_option("band_first", first)
            for _ in range(30):
                bare()
            frame = bytes(fb.pixels)
            if ref is None:
                ref = frame
            assert frame == ref, "band split changed the frame"
            tb = []
            for _ in range(300):
                t = time.perf_counter()
                bare()
                tb.append(time.perf_counter() - t)
            ctx.set_option("band_times", 1)
            tl = []
            for _ in range(50):
                bare()
                tl.append(ctx.band_times_ms())
            ctx.set_option("band_times", 0)
            med = [tuple(1e3 * statistics.median(f[k][j] for f in tl) for j in range(2)) for k in range(len(tl[0]))]
            line = " ".join(f"[{a:.0f}|{b:.0f}]" for a, b in med)
            print(f"{key} bands={bands} first={first}: bare call {1e6 * statistics.median(tb):.1f} us "
                  f"(p10 {1e6 * sorted(tb)[len(tb) // 10]:.1f}) | per band [kernels end|copy end] us {line}",
                  flush=True)
        ctx.set_option("bands", 0)
        ctx.set_option("band_first", 0)
        ctx.unpin(fb.pixels)


if __name__ == "__main__":
    main()
