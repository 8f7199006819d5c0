"""Render configurations on the GPU (FP32, radiance on) and save the frames
to gpurun_out/parity_<key>.npz for offline analysis against the oracle
(tools/parity_analyse.py, run in the build container).

    python tools/parity_dump.py C5@384x216 C2 ...
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2305_07450_b200 as rt  # noqa: E402


def config(key):
    if "@" in key:
        base, size = key.split("@")
        w, h = (int(v) for v in size.split("x"))
        return rt.CONFIGS[base], w, h
    c = rt.CONFIGS[key]
    return c, c.width, c.height


def main():
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    for key in sys.argv[1:]:
        cfg, w, h = config(key)
        scene, cam = cfg.scene(), cfg.camera()
        fb = rt.Framebuffer.create(w, h)
        rad = np.zeros((w * h, 3), np.float32)
        rt.render_frame(scene, cam, rt.RenderParams(cfg.samples, cfg.bounces, w, h), fb, radiance=rad)
        np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"parity_{key.replace('@', '_')}.npz"), px=fb.pixels,
                            rad=rad)
        print(key, "saved")


if __name__ == "__main__":
    main()
