"""pytest plugin: run the REFERENCE's own test suite with its render entry
points rebound to libb200rt (paper_2305_07450_b200.install()).

    B200RT_REF_PRECISION=fp64 python -m pytest -p ref_suite_plugin \\
        baseline/_ref/ref_tests            (PYTHONPATH=tests:.)

The reference package is the unmodified one pip-installed into baseline/_ref
(tools/install_reference.sh).  install() runs in pytest_configure, before the
reference's test modules are imported, so their `from raytracer.renderer
import render_frame` (and raytracer.bench / cli / server's own imports)
resolve to the B200 renderer.  Used by tests/test_gpu_reference_suite.py.
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def pytest_configure(config):
    for p in (REF, ROOT):
        if p not in sys.path:
            sys.path.insert(0, p)
    import raytracer

    if not os.path.abspath(raytracer.__file__).startswith(REF):
        raise RuntimeError(f"raytracer imported from {raytracer.__file__}, not baseline/_ref")
    import paper_2305_07450_b200 as rt

    precision = os.environ.get("B200RT_REF_PRECISION", "fp64")
    patched = rt.install(precision=precision)
    config._b200_patched = patched


def pytest_unconfigure(config):
    """$B200RT_REF_MARKER: a JSON record that install() ran and the GPU library served the suite."""
    path = os.environ.get("B200RT_REF_MARKER")
    if not path:
        return
    from paper_2305_07450_b200 import _native

    _native.load()
    with open(path, "w") as f:
        json.dump({"patched": getattr(config, "_b200_patched", []), "lib": _native.LIB_PATH,
                   "contexts": len(_native._contexts)}, f)
