"""Parity gates of the north star, written once.

byte gate:     per 8-bit channel |delta| <= 1 on >= 99.9% of pixels
radiance gate: |delta| <= 1e-4 * max(|ref|, 1) per channel on >= 99.9% of pixels
relative gate: |delta| <= 1e-4 * |ref| per channel (the north star's literal
               "float radiance within 1e-4 relative"; a denormal-level floor
               of 1e-30 only so that ref == 0 demands got == 0) on >= 99.9% of pixels
"""

import numpy as np

BYTE_TOL = 1
BYTE_FRACTION = 0.999
RADIANCE_TOL = 1e-4
RADIANCE_FRACTION = 0.999
RELATIVE_FLOOR = 1e-30


def channels(pixels):
    p = np.asarray(pixels, dtype=np.uint32)
    return np.stack([(p >> 16) & 0xFF, (p >> 8) & 0xFF, p & 0xFF, p >> 24], axis=-1).astype(np.int32)


def byte_gate(got, want):
    """(fraction of pixels within ±1 on every channel, max |delta|)."""
    d = np.abs(channels(got) - channels(want))
    per_px = d.max(axis=-1)
    return float(np.mean(per_px <= BYTE_TOL)), int(per_px.max(initial=0))


def radiance_gate(got, want):
    """(fraction of pixels within 1e-4*max(|ref|,1) on every channel, max abs delta)."""
    got = np.asarray(got, dtype=np.float64).reshape(-1, 3)
    want = np.asarray(want, dtype=np.float64).reshape(-1, 3)
    err = np.abs(got - want)
    ok = (err <= RADIANCE_TOL * np.maximum(np.abs(want), 1.0)).all(axis=-1)
    return float(np.mean(ok)), float(err.max(initial=0.0))


def assert_byte_gate(got, want, label=""):
    frac, worst = byte_gate(got, want)
    assert frac >= BYTE_FRACTION, f"{label}: only {frac:.6%} of pixels within ±1 (worst delta {worst})"
    return frac, worst


def assert_radiance_gate(got, want, label=""):
    frac, worst = radiance_gate(got, want)
    assert frac >= RADIANCE_FRACTION, f"{label}: only {frac:.6%} of pixels within 1e-4 (worst {worst:.3g})"
    return frac, worst


def relative_gate(got, want):
    """(fraction of pixels within 1e-4*|ref| on every channel, max relative delta)."""
    got = np.asarray(got, dtype=np.float64).reshape(-1, 3)
    want = np.asarray(want, dtype=np.float64).reshape(-1, 3)
    err = np.abs(got - want)
    scale = np.maximum(np.abs(want), RELATIVE_FLOOR)
    ok = (err <= RADIANCE_TOL * scale).all(axis=-1)
    return float(np.mean(ok)), float((err / scale).max(initial=0.0))


def assert_relative_gate(got, want, label=""):
    frac, worst = relative_gate(got, want)
    assert frac >= RADIANCE_FRACTION, f"{label}: only {frac:.6%} of pixels within 1e-4 relative (worst {worst:.3g})"
    return frac, worst
