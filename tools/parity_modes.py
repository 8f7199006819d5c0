"""Literal-gate failure fractions per FP32 execution path, on the GPU box:
for each configuration, the oracle's radiance once, then every mode's frame.

    B200RT_LIB=... python tools/parity_modes.py C5@384x216 C2 ...
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import parity  # noqa: E402
import paper_2305_07450_b200 as rt  # noqa: E402
from paper_2305_07450_b200 import _native  # noqa: E402
from parity_dump import config  # noqa: E402

MODES = {"cull": dict(wave=True, cull=True, conic=True), "ray": dict(wave=True, cull=True, conic=False),
         "wave": dict(wave=True, cull=False), "mega": dict(wave=False, cull=False)}


def main():
    modes = os.environ.get("MODES", "cull,ray,wave,mega").split(",")
    for key in sys.argv[1:]:
        cfg, w, h = config(key)
        scene, cam = cfg.scene(), cfg.camera()
        t = time.time()
        want_px, want = oracle.render(vars(rt.pack_scene(scene)), cam.position, cam.yaw, cam.pitch, cam.fov, w, h,
                                      cfg.samples, cfg.bounces, radiance=True)
        ot = time.time() - t
        for m in modes:
            _native.set_options(**MODES[m])
            fb = rt.Framebuffer.create(w, h)
            rad = np.zeros((w * h, 3), np.float32)
            rt.render_frame(scene, cam, rt.RenderParams(cfg.samples, cfg.bounces, w, h), fb, radiance=rad)
            bf, bw = parity.byte_gate(fb.pixels, want_px)
            rf, rw = parity.relative_gate(rad, want)
            af, _ = parity.radiance_gate(rad, want)
            print(f"{key:12s} {m:5s} byte {bf:.6%} (max {bw:3d})  rel-fail {1 - rf:.4%}  abs-fail {1 - af:.4%}"
                  f"  (oracle {ot:.1f}s)", flush=True)


if __name__ == "__main__":
    main()
