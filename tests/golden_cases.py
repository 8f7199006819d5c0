"""Loader for the golden parity fixtures (tests/golden/, made by
tests/golden/make_golden.py from the reference implementation)."""

from __future__ import annotations

import functools
import json
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GOLDEN_SHA_128x72_S200_B3 = "f9841b1c4ee5f6d6a2308d11b564de6c8b54d9e1def48e453a2d43175979ef14"


def sky_texels(recipe):
    """Same recipe as make_golden.sky_texels (gradient fixture of
    test_renderer.py:23-28, optionally with an HDR band > 1.0)."""
    kind, w, h = recipe.split(":")
    w, h = int(w), int(h)
    xs = np.arange(w, dtype=np.float64) / w
    ys = np.arange(h, dtype=np.float64) / h
    t = np.empty((h, w, 3), dtype=np.float32)
    t[:, :, 0] = xs[None, :]
    t[:, :, 1] = ys[:, None]
    t[:, :, 2] = 0.25
    if kind == "hdr":
        t[: h // 3] *= np.float32(3.0)
    return t


@functools.lru_cache(maxsize=None)
def _index():
    with open(os.path.join(GOLDEN_DIR, "cases.json")) as f:
        return json.load(f)


@functools.lru_cache(maxsize=None)
def _frames():
    return dict(np.load(os.path.join(GOLDEN_DIR, "frames.npz")))


@functools.lru_cache(maxsize=None)
def _rays():
    return dict(np.load(os.path.join(GOLDEN_DIR, "rays.npz")))


def packed_scene(entry):
    """Reference SoA layout (geometry.py:162-176, scene.py:100-104)."""
    s = entry["scene"]
    ps = dict(
        kinds=np.array(s["kinds"], dtype=np.int32),
        positions=np.array(s["positions"], dtype=np.float64).reshape(-1, 3),
        sizes=np.array(s["sizes"], dtype=np.float64),
        colors=np.array(s["colors"], dtype=np.float64).reshape(-1, 3),
        refls=np.array(s["refls"], dtype=np.float64),
        light_pos=np.array(s["light_pos"], dtype=np.float64),
        light_radius=float(s["light_radius"]),
        light_color=np.array(s["light_color"], dtype=np.float64),
        ambient=float(s["ambient"]),
        max_refl=float(s["max_refl"]),
    )
    if entry.get("sky"):
        t = sky_texels(entry["sky"])
        ps.update(sky=t, sky_w=t.shape[1], sky_h=t.shape[0], has_sky=True)
    else:
        ps.update(sky=np.zeros((1, 1, 3), np.float32), sky_w=1, sky_h=1, has_sky=False)
    return ps


def frame_cases():
    return _index()["frames"]


def frame_case(name):
    for c in frame_cases():
        if c["name"] == name:
            return c
    raise KeyError(name)


def frame_pixels(name):
    return _frames()[f"{name}/pixels"]


def frame_radiance(name):
    return _frames().get(f"{name}/radiance")


def ray_cases():
    return _index()["rays"]


def ray_arrays(name):
    r = _rays()
    return {k.split("/", 1)[1]: v for k, v in r.items() if k.startswith(name + "/")}
