"""pow_cr (csrc/rt_pow.cuh, the FP64 kernels' Blinn pow) against the C
library's pow — the function numba's `d**reflectivity` calls in the
reference (shading.py:73).  The same source is compiled for the host with
g++ (contraction off, as the FP64 kernels' -fmad=false) and run on random
arguments of the Blinn domain.  pow_cr is correctly rounded to ~2^-90; glibc's
pow misrounds when the exact value lies within ~0.0005 ulp of a midpoint, so
the two agree except on that small fraction, and never by more than 1 ulp."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_pow_cr_matches_libm(tmp_path):
    exe = tmp_path / "pow_check"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-I", os.path.join(ROOT, "paper_2305_07450_b200", "csrc"),
                    os.path.join(ROOT, "tests", "native", "pow_check.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "2000000"], check=True, capture_output=True, text=True).stdout.split()
    n, bad, worst = (int(v) for v in out)
    assert n == 2_000_000
    assert worst <= 1
    assert bad / n < 2e-3, f"{bad} of {n} differ from libm"
