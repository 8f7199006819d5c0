"""Median device time of the render kernel per configuration (A/B runs:
select the library with $B200RT_LIB).

    python tools/ab_kernel.py C2 C4 P720 [--frames 20] [--precision fp32]
"""

import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2305_07450_b200 as rt  # noqa: E402
from paper_2305_07450_b200 import _native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C2", "C4"])
    ap.add_argument("--frames", type=int, default=20)
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--mode", default=None, help="cull | ray | wave | mega")
    ap.add_argument("--bands", type=int, default=1, help="row bands of rt_render_v1 (0 = by frame size)")
    ap.add_argument("--opt", action="append", default=[], help="extra rt_set_option name=value (repeatable)")
    a = ap.parse_args()
    tag = os.path.basename(_native.LIB_PATH)
    _native.set_options(bands=a.bands, phases=1)
    if a.mode:
        _native.set_options(**{"cull": dict(wave=1, cull=1, conic=1), "ray": dict(wave=1, cull=1, conic=0),
                               "wave": dict(wave=1, cull=0), "mega": dict(wave=0, cull=0)}[a.mode])
        tag += f"[{a.mode}]"
    for o in a.opt:
        name, value = o.split("=")
        _native.set_options(**{name: int(value)})
        tag += f"[{o}]"
    for key in a.configs:
        cfg = rt.CONFIGS[key]
        scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
        fb = rt.Framebuffer.create(cfg.width, cfg.height)
        ms = []
        for i in range(a.frames + 3):
            rt.render_frame(scene, cam, params, fb, precision=a.precision)
            if i >= 3:
                ms.append(rt.last_kernel_ms())
        ph = _native.context(1).phase_ms()
        phs = " ".join(f"{k} {v:.4f}" for k, v in ph.items()) if sum(ph.values()) else "single kernel"
        print(f"{tag:>14} {key:>6} {a.precision} median {statistics.median(ms):8.4f} ms  min {min(ms):8.4f} ms"
              f"  [{phs}]", flush=True)


if __name__ == "__main__":
    main()
