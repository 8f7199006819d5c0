"""Build libb200rt.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2305_07450_b200.build [-v]

The FP64 validation kernel is compiled with -fmad=false (no a*b+c contraction,
like numba's reference build); the FP32 product kernel keeps FMA.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libb200rt.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC]
HOST_CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else None

SOURCES = {
    # host side: the skybox check splits its compare over OpenMP threads
    "rt_host.cu": ["-Xcompiler", "-fopenmp"],
    # FP32 product path: flush denormals, approximate sqrt/div (powf, atan2f
    # and asinf stay full precision: no --use_fast_math)
    "render_f32.cu": ["--ftz=true", "--prec-div=false", "--prec-sqrt=false"],
    "render_wave_f32.cu": ["--ftz=true", "--prec-div=false", "--prec-sqrt=false"],
    "render_fused_f32.cu": ["--ftz=true", "--prec-div=false", "--prec-sqrt=false"],
    "render_f64.cu": ["-fmad=false"],
    "render_fused_f64.cu": ["-fmad=false"],
    # compressed frame transfer: the GPU encoder and the host's AVX2 expander
    "frame_codec.cu": [],
    "frame_decode.cpp": ["-Xcompiler", "-fopenmp"],
}


def _ccbin():
    return ["-ccbin", HOST_CXX] if HOST_CXX else []


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, ptxas_verbose: bool = False, defines=(), out=None,
          f32_flags=None) -> str:
    """Compile (incrementally) and link libb200rt.so.  `defines` (e.g.
    ["RT_F32_MIN_BLOCKS=6"]), `f32_flags` (replacing the FP32 sources' own
    flags) and `out` build an experimental variant into a separate object
    directory."""
    if not os.path.exists(NVCC) and shutil.which("nvcc") is None:
        raise RuntimeError("nvcc not found: cannot build libb200rt.so")
    nvcc = NVCC if os.path.exists(NVCC) else shutil.which("nvcc")
    lib = out or LIB
    tag = [d.replace("=", "") for d in defines] + [f.strip("-").replace("=", "") for f in (f32_flags or [])]
    bdir = BUILD if not tag else os.path.join(BUILD, "v_" + "_".join(tag))
    os.makedirs(bdir, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(INCLUDE, "b200rt.h"))
    objs, cmds = [], []
    for src, extra in SOURCES.items():
        if f32_flags is not None and "f32" in src:
            extra = list(f32_flags)
        s = os.path.join(CSRC, src)
        o = os.path.join(bdir, os.path.splitext(src)[0] + ".o")
        objs.append(o)
        if force or _stale(o, [s, *headers, __file__]):
            cmd = [nvcc, *_ccbin(), *COMMON, *extra, *dflags, "-c", s, "-o", o]
            if ptxas_verbose:
                cmd += ["-Xptxas", "-v"]
            if verbose:
                print(" ".join(cmd), flush=True)
            cmds.append(cmd)
    # the translation units are independent: compile them side by side
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as pool:
        for r in list(pool.map(lambda c: subprocess.run(c, capture_output=not verbose), cmds)):
            if r.returncode != 0:
                if r.stderr:
                    sys.stderr.write(r.stderr.decode(errors="replace"))
                raise subprocess.CalledProcessError(r.returncode, r.args)
    if force or _stale(lib, objs):
        cmd = [nvcc, *_ccbin(), *ARCH, "-shared", "-o", lib, *objs, "-lgomp"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    if not tag:
        build_pyfast(verbose, force)
    return lib


def build_pyfast(verbose: bool = False, force: bool = False):
    """The CPython fast path of render_frame (csrc/pyfast.c): scene packing
    and the rt_render_v1 call without ctypes marshalling.  Optional: without
    a C compiler or Python headers the ctypes path serves."""
    import sysconfig

    src = os.path.join(CSRC, "pyfast.c")
    out = os.path.join(PKG, "_pyfast" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))
    cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else shutil.which("gcc")
    inc = sysconfig.get_paths().get("include")
    if not cc or not inc or not os.path.exists(os.path.join(inc, "Python.h")):
        return None
    if force or _stale(out, [src, __file__]):
        cmd = [cc, "-O2", "-shared", "-fPIC", "-I", inc, "-I", INCLUDE, src, "-o", out]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    f32 = [a[6:] for a in sys.argv[1:] if a.startswith("--f32=")]
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, ptxas_verbose="--ptxas" in sys.argv,
                defines=defs, out=outs[0] if outs else None, f32_flags=f32[0].split() if f32 else None))
