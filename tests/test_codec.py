"""The compressed frame transfer's host half (rt_frame_expand_v1, option
"codec"): frames encoded here in numpy by the layout include/b200rt.h
documents expand bit for bit, for ragged widths, runs crossing the 8- and
32-pixel groups, padded row pitches and any thread count.  CPU only: the
GPU encoder is checked against the raw copy in tests/test_gpu_codec.py."""

import ctypes

import numpy as np
import pytest

from paper_2305_07450_b200 import _native

PAD = 32  # frame_codec.h kCodecPad


def encode(frame: np.ndarray) -> tuple[np.ndarray, int]:
    """numpy restatement of frame_codec.cu's row runs (include/b200rt.h,
    rt_frame_expand_v1); returns the buffer and the words the runs occupy."""
    h, w = frame.shape
    mw = (w + 31) // 32
    nb = (mw + 31) // 32
    stride = (1 + nb + mw + w + 31) // 32 * 32
    buf = np.full(2 * PAD + h * stride, 0xDEADBEEF, dtype=np.uint32)  # stale words must never show
    total = 0
    for y in range(h):
        row = frame[y]
        is_lit = np.ones(w, dtype=bool)
        is_lit[1:] = row[1:] != row[:-1]
        bits = np.zeros(mw * 32, dtype=np.uint64)
        bits[:w] = is_lit
        words = (bits.reshape(mw, 32) << np.arange(32, dtype=np.uint64)).sum(axis=1).astype(np.uint32)
        nz = words != 0
        zb = np.zeros(nb * 32, dtype=np.uint64)
        zb[:mw] = nz
        bitmap = (zb.reshape(nb, 32) << np.arange(32, dtype=np.uint64)).sum(axis=1).astype(np.uint32)
        lits = row[is_lit]
        packed = bool(((lits >> 24) == 0xFF).all())
        if packed:
            b = lits.view(np.uint8).reshape(-1, 4)[:, :3].reshape(-1)
            b = np.concatenate([b, np.zeros((-len(b)) % 4, dtype=np.uint8)])
            lw = b.view(np.uint32)
        else:
            lw = lits
        run = np.concatenate([np.array([len(lits) | (packed << 31)], dtype=np.uint32), bitmap, words[nz], lw])
        base = PAD + y * stride
        buf[base:base + len(run)] = run
        total += len(run)
    return buf, total


def expand(buf, w, h, pitch=None, threads=1):
    pitch = pitch or w
    out = np.full((h, pitch), 0x12345678, dtype=np.uint32)
    n = ctypes.c_int64(-1)
    rc = _native.load().rt_frame_expand_v1(buf.ctypes.data, w, h, out.ctypes.data, pitch, threads, ctypes.byref(n))
    assert rc == 0, _native.load().rt_last_error()
    return out, n.value


def runs_frame(rng, h, w, mean_run, opaque=False):
    """Rows of runs of equal pixels (lengths ~ geometric), some rows constant;
    opaque: every pixel's top byte 0xFF (the frames' alpha: packed rows)."""
    f = np.empty((h, w), dtype=np.uint32)
    for y in range(h):
        if y % 5 == 3:
            f[y] = 0xFF000000
            continue
        starts = np.flatnonzero(rng.random(w) < 1.0 / mean_run)
        vals = rng.integers(0, 2**32, size=len(starts) + 1, dtype=np.uint64).astype(np.uint32)
        idx = np.searchsorted(starts, np.arange(w), side="right")
        f[y] = vals[idx]
        if opaque or y % 7 == 5:
            f[y] |= np.uint32(0xFF000000)
    return f


@pytest.mark.parametrize("w", [1, 2, 7, 8, 9, 31, 32, 33, 63, 64, 65, 129, 1025, 1280])
@pytest.mark.parametrize("mean_run", [1.0, 3.0, 40.0])
@pytest.mark.parametrize("opaque", [False, True])
def test_expand_round_trip(w, mean_run, opaque):
    rng = np.random.default_rng(w * 1000 + int(mean_run))
    h = 13
    f = runs_frame(rng, h, w, mean_run, opaque)
    buf, n_words = encode(f)
    for threads in (1, 3):
        out, n = expand(buf, w, h, threads=threads)
        assert n == n_words
        np.testing.assert_array_equal(out, f)


def test_expand_padded_pitch_leaves_the_gap():
    rng = np.random.default_rng(7)
    w, h, pitch = 45, 9, 64
    f = runs_frame(rng, h, w, 4.0)
    buf, _ = encode(f)
    out, _ = expand(buf, w, h, pitch=pitch, threads=2)
    np.testing.assert_array_equal(out[:, :w], f)
    assert (out[:, w:] == 0x12345678).all()


def test_expand_constant_and_alternating_rows():
    w, h = 100, 4
    f = np.zeros((h, w), dtype=np.uint32)
    f[1] = 0xFF0E0F11  # one packed literal, three zero mask words
    f[2, ::2] = 1  # every pixel a literal, unpacked
    f[3] = 0xFF000000 | (np.arange(w) // 9)  # runs of 9 across the 8-pixel groups, packed
    buf, n_words = encode(f)
    out, n = expand(buf, w, h)
    np.testing.assert_array_equal(out, f)
    # header + bitmap + listed mask words + literal words, per row: 1 unpacked
    # literal; 1 packed; 100 unpacked over 4 mask words; 12 packed (9 words)
    assert n == n_words == (1 + 1 + 1 + 1) + (1 + 1 + 1 + 1) + (1 + 1 + 4 + 100) + (1 + 1 + 4 + 9)


def test_expand_rejects_bad_sizes():
    lib = _native.load()
    buf = np.zeros(256, dtype=np.uint32)
    out = np.zeros(16, dtype=np.uint32)
    assert lib.rt_frame_expand_v1(buf.ctypes.data, 0, 1, out.ctypes.data, 1, 1, None) != 0
    assert lib.rt_frame_expand_v1(buf.ctypes.data, 4, 1, out.ctypes.data, 3, 1, None) != 0
    assert lib.rt_frame_expand_v1(None, 4, 1, out.ctypes.data, 4, 1, None) != 0


@pytest.mark.parametrize("isa", ["scalar", "avx2"])
def test_expand_narrower_isas(isa):
    """The AVX2 and scalar expanders ($B200RT_CODEC_ISA, read once per
    process) on the same frames as the default (AVX-512 where the CPU has it)."""
    import os
    import subprocess
    import sys

    code = (
        "import numpy as np, test_codec as t\n"
        "for w in (1, 7, 8, 9, 33, 65, 1025):\n"
        "    for opaque in (False, True):\n"
        "        f = t.runs_frame(np.random.default_rng(w), 9, w, 3.0, opaque)\n"
        "        buf, n = t.encode(f)\n"
        "        out, m = t.expand(buf, w, 9, threads=2)\n"
        "        assert m == n and (out == f).all(), (w, opaque)\n"
    )
    env = dict(os.environ, B200RT_CODEC_ISA=isa)
    here = os.path.dirname(os.path.abspath(__file__))
    env["PYTHONPATH"] = os.pathsep.join([here, os.path.dirname(here), env.get("PYTHONPATH", "")])
    subprocess.run([sys.executable, "-c", code], env=env, check=True, cwd=here, timeout=120)
