"""How sensitive is a frame to float32 rounding of each intermediate?  Builds
the oracle with -DRTO_ROUND=mask (oracle/rt_oracle.c: 1 primary direction,
2 hit point + normal, 4 shadow origin + sample directions, 8 reflected ray)
and reports, per mask, the share of pixels outside the pure-relative 1e-4
radiance gate against the exact oracle.  Runs on the CPU.

    python tools/precision_probe.py C5@384x216 [masks...]
"""
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import oracle  # noqa: E402
import parity  # noqa: E402
import paper_2305_07450_b200 as rt  # noqa: E402
from parity_dump import config  # noqa: E402


def build(mask):
    out = f"/tmp/librt_oracle_round{mask}.so"
    subprocess.run(["gcc", "-O2", "-fPIC", "-std=c11", "-D_GNU_SOURCE", "-ffp-contract=off", "-fno-fast-math",
                    "-fopenmp", f"-DRTO_ROUND={mask}", "-shared", "-o", out, os.path.join(ROOT, "oracle", "rt_oracle.c"),
                    "-lm"], check=True)
    return out


def render_with(lib_path, cfg, w, h):
    saved = oracle._lib
    oracle._lib = None
    real = oracle._LIB_PATH
    oracle._LIB_PATH = lib_path
    try:
        L = ctypes.CDLL(lib_path)
        oracle._lib = None
        # reuse the signature setup of oracle.lib()
        orig_cdll = ctypes.CDLL
        ctypes.CDLL = lambda p: L
        try:
            scene, cam = cfg.scene(), cfg.camera()
            return oracle.render(vars(rt.pack_scene(scene)), cam.position, cam.yaw, cam.pitch, cam.fov, w, h,
                                 cfg.samples, cfg.bounces, radiance=True)
        finally:
            ctypes.CDLL = orig_cdll
    finally:
        oracle._lib = saved
        oracle._LIB_PATH = real


def main():
    key = sys.argv[1]
    masks = [int(m) for m in sys.argv[2:]] or [1, 2, 4, 8, 15, 14]
    cfg, w, h = config(key)
    scene, cam = cfg.scene(), cfg.camera()
    want_px, want = oracle.render(vars(rt.pack_scene(scene)), cam.position, cam.yaw, cam.pitch, cam.fov, w, h,
                                  cfg.samples, cfg.bounces, radiance=True)
    for m in masks:
        px, rad = render_with(build(m), cfg, w, h)
        rf, _ = parity.relative_gate(rad, want)
        bf, bw = parity.byte_gate(px, want_px)
        print(f"{key} round mask {m:2d}: relative-gate failures {1 - rf:.4%}, byte gate {bf:.5%} (max {bw})",
              flush=True)


if __name__ == "__main__":
    main()
