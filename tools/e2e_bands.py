"""End-to-end render_frame time against the number of copy-overlapped row bands."""

import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2305_07450_b200 as rt  # noqa: E402
from paper_2305_07450_b200 import _native  # noqa: E402


def main():
    keys = sys.argv[1:] or ["C2", "P720", "C3"]
    ctx = _native.context(1)
    for key in keys:
        cfg = rt.CONFIGS[key]
        scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
        fb = rt.Framebuffer.create(cfg.width, cfg.height)
        ref = None
        for bands in (1, 2, 3, 4):
            ctx.set_option("bands", bands)
            for _ in range(10):
                rt.render_frame(scene, cam, params, fb)
            if ref is None:
                ref = fb.pixels.copy()
            assert (fb.pixels == ref).all()
            ts, ks = [], []
            for _ in range(200):
                t = time.perf_counter()
                rt.render_frame(scene, cam, params, fb)
                ts.append(time.perf_counter() - t)
                ks.append(ctx.last_kernel_ms())
            print(f"{key} bands={bands}: e2e median {1e6 * statistics.median(ts):.1f} us  mean {1e6 * statistics.mean(ts):.1f} us"
                  f"  device {1e3 * statistics.median(ks):.1f} us", flush=True)
        ctx.set_option("bands", 0)


if __name__ == "__main__":
    main()
