"""The reference's command line with the render backend selectable.

    python -m paper_2305_07450_b200.cli [--backend b200|reference] [--precision fp32|fp64] \\
        render --width 1280 --height 720 --samples 200 --bounces 3 --out frame.ppm
    python -m paper_2305_07450_b200.cli bench --resolution 720p --samples 1 --bounces 1

Everything after the backend options is the reference CLI's own argument list
(`raytracer render | bench | serve`, /root/reference/pkg/src/raytracer/cli.py:101-142),
handed unchanged to the reference's `raytracer.cli.main`.  With `--backend b200`
(the default) `install()` first rebinds the reference's `render_frame` in
`raytracer.renderer`, `raytracer.cli` (cli.py:17, called by `cmd_render`,
cli.py:59-66), `raytracer.bench` (`run_benchmark`, bench.py:15 / cli.py:69-83)
and `raytracer.server` (`FrameLoop.tick`, used by `serve`) to libb200rt, so
`render` writes its PPM through the reference's own `write_ppm`
(sceneio.py:170-179) from a frame rendered on the B200, and `bench` reports
the reference harness's frames/s for the B200 renderer.  `--backend reference`
runs the stock numba path (no rebinding), for side-by-side runs.

The reference package must be importable (`pip install /root/reference/pkg`,
or tools/install_reference.sh into baseline/_ref, which this module adds to
sys.path when present).
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def _import_reference_cli():
    try:
        import raytracer.cli as cli
    except ImportError:
        if os.path.isdir(REF) and REF not in sys.path:
            sys.path.insert(0, REF)
        import raytracer.cli as cli
    return cli


def main(argv=None) -> int:
    pre = argparse.ArgumentParser(prog="paper_2305_07450_b200.cli", add_help=False)
    pre.add_argument("--backend", choices=["b200", "reference"], default="b200")
    pre.add_argument("--precision", choices=["fp32", "fp64"], default=None,
                     help="B200 kernels: fp32 (product) or fp64 (bit-identical to the reference)")
    opts, rest = pre.parse_known_args(sys.argv[1:] if argv is None else argv)
    cli = _import_reference_cli()
    if opts.backend == "b200":
        from .integration import install

        install(precision=opts.precision)
    return cli.main(rest)


if __name__ == "__main__":
    sys.exit(main())
