"""Executed-work tallies of the culled shadow pass per configuration.

    python tools/work_stats.py C2 C4 ...
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2305_07450_b200 as rt  # noqa: E402
from paper_2305_07450_b200 import _native  # noqa: E402


def main():
    keys = sys.argv[1:] or ["C2"]
    _native.set_options(count_work=True)
    ctx = _native.context(1)
    out = {}
    for key in keys:
        cfg = rt.CONFIGS[key]
        fb = rt.Framebuffer.create(cfg.width, cfg.height)
        ctx.work_counts(reset=True)
        rt.render_frame(cfg.scene(), cfg.camera(), cfg.params(), fb)
        out[key] = ctx.work_counts(reset=True)
        print(key, json.dumps(out[key]), flush=True)


if __name__ == "__main__":
    main()
