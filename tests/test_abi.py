"""The C-ABI library loads and exports exactly what include/b200rt.h declares
(no compute calls: these run on the GPU-less build host)."""

import os
import re
import subprocess

import pytest

from paper_2305_07450_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "b200rt.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^(?:const\s+)?\w+\s*\*?\s*(rt_\w+)\s*\(", src, flags=re.M)))


def test_header_parses():
    names = declared()
    assert "rt_render_v1" in names and "rt_last_error" in names and len(names) >= 20


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    for name in declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (rt_\w+)", out))
    assert set(declared()) <= exported


def test_binding_table_matches_header():
    assert sorted(_native.SIGNATURES) == declared()


def test_library_is_sm_100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_version_and_device_count_are_safe_without_gpu():
    lib = _native.load()
    assert lib.rt_version() == 1
    assert _native.device_count() >= 0
