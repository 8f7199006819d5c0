"""Swap the reference renderer for the B200 one inside an existing program.

The reference's callers import `render_frame` by name at import time —
`raytracer.bench` (bench.py:15), `raytracer.cli` (cli.py:17) and
`raytracer.server` (server.py:43) — so rebinding `raytracer.renderer`
alone would leave them on the numba path.  `install()` rebinds every one.
"""

from __future__ import annotations

import functools
import importlib
import sys

from . import renderer as _b200

_TARGETS = ("raytracer.renderer", "raytracer.bench", "raytracer.cli", "raytracer.server")
_saved = {}


def install(precision=None, package: str = "raytracer"):
    """Point the reference package's render entry points at libb200rt.

    Returns the list of modules patched.  `uninstall()` restores them."""
    fn = _b200.render_frame if precision is None else functools.partial(_b200.render_frame, precision=precision)
    patched = []
    for name in _TARGETS:
        name = name.replace("raytracer", package, 1)
        try:
            mod = sys.modules.get(name) or importlib.import_module(name)
        except ImportError:
            continue
        for attr, new in (("render_frame", fn), ("ray_trace_iterative", _b200.ray_trace_iterative)):
            if hasattr(mod, attr):
                _saved.setdefault((name, attr), getattr(mod, attr))
                setattr(mod, attr, new)
        patched.append(name)
    return patched


def uninstall():
    for (name, attr), old in list(_saved.items()):
        mod = sys.modules.get(name)
        if mod is not None:
            setattr(mod, attr, old)
    _saved.clear()
