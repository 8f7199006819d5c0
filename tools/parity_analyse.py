"""Offline analysis of GPU frames saved by tools/parity_dump.py against the
oracle: where do pixels fail the pure-relative 1e-4 radiance gate?

    python tools/parity_analyse.py C5@384x216 [...]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import paper_2305_07450_b200 as rt  # noqa: E402
from parity_dump import config  # noqa: E402


def main():
    for key in sys.argv[1:]:
        cfg, w, h = config(key)
        d = np.load(os.path.join(ROOT, "gpurun_out", f"parity_{key.replace('@', '_')}.npz"))
        scene, cam = cfg.scene(), cfg.camera()
        cache = os.path.join(ROOT, "gpurun_out", f"oracle_{key.replace('@', '_')}.npz")
        if os.path.exists(cache):
            o = np.load(cache)
            want_px, want = o["px"], o["rad"]
        else:
            want_px, want = oracle.render(vars(rt.pack_scene(scene)), cam.position, cam.yaw, cam.pitch, cam.fov, w, h,
                                          cfg.samples, cfg.bounces, radiance=True)
            np.savez_compressed(cache, px=want_px, rad=want)
        got = d["rad"].astype(np.float64)
        err = np.abs(got - want)
        rel = err / np.maximum(np.abs(want), 1e-30)
        bad = (rel > 1e-4).any(-1)
        print(f"{key}: {bad.sum()} of {bad.size} pixels fail ({bad.mean():.4%})")
        relmax = rel.max(-1)[bad]
        errmax = err.max(-1)[bad]
        for lo, hi in ((1e-4, 3e-4), (3e-4, 1e-3), (1e-3, 1e-2), (1e-2, 1e9)):
            m = (relmax > lo) & (relmax <= hi)
            print(f"  rel in ({lo:g}, {hi:g}]: {m.sum()}  (abs err median {np.median(errmax[m]) if m.any() else 0:.2e})")
        # abs error as multiples of 1/samples (a flipped shadow sample moves the
        # coefficient by 1/n; the pixel moves by ~base*(1-amb)*d/n)
        ys, xs = np.nonzero(bad.reshape(h, w))
        print("  rows of failures (hist):", np.histogram(ys, bins=8, range=(0, h))[0].tolist())
        np.save(os.path.join(ROOT, "gpurun_out", f"bad_{key.replace('@', '_')}.npy"), np.stack([xs, ys], -1))


if __name__ == "__main__":
    main()
