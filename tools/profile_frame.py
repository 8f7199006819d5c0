"""Render a few frames of one configuration through render_frame — the short
command the ncu captures profile (profiles/).

    python tools/profile_frame.py --config C2 --frames 3 [--precision fp32]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2305_07450_b200 as rt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--frames", type=int, default=3)
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--workers", type=int, default=None)
    ap.add_argument("--bands", type=int, default=1, help="rt_render_v1 row bands (0 = by frame size)")
    a = ap.parse_args()
    cfg = rt.CONFIGS[a.config]
    from paper_2305_07450_b200 import _native

    _native.set_options(bands=a.bands)
    scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
    fb = rt.Framebuffer.create(cfg.width, cfg.height)
    for i in range(a.frames):
        rt.render_frame(scene, cam, params, fb, workers=a.workers, precision=a.precision)
        print(f"frame {i}: kernel {rt.last_kernel_ms(a.workers):.3f} ms", flush=True)


if __name__ == "__main__":
    main()
