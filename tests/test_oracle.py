"""The oracle (oracle/rt_oracle.c) is pinned against the reference before it
is trusted: the reference's golden sha256 (pkg/tests/test_acceptance.py:31),
every framebuffer / radiance / per-ray fixture produced by the reference
itself (tests/golden/make_golden.py), and the reference tests' scalar KATs."""

import hashlib
import math

import numpy as np
import pytest

import golden_cases as G
import oracle

CASES = [c["name"] for c in G.frame_cases()]


def _render(c, radiance=False):
    cam = c["camera"]
    return oracle.render(G.packed_scene(c), cam["position"], cam["yaw"], cam["pitch"], cam["fov"], c["width"],
                         c["height"], c["samples"], c["bounces"], radiance=radiance)


def test_golden_sha256_128x72_s200_b3():
    c = G.frame_case("bench_128x72_s200_b3")
    px = _render(c)
    assert hashlib.sha256(px.tobytes()).hexdigest() == G.GOLDEN_SHA_128x72_S200_B3


@pytest.mark.parametrize("name", CASES)
def test_frames_bit_exact(name):
    c = G.frame_case(name)
    px, rad = _render(c, radiance=True)
    assert hashlib.sha256(px.tobytes()).hexdigest() == c["sha256"]
    np.testing.assert_array_equal(px, G.frame_pixels(name))
    want = G.frame_radiance(name)
    if want is not None:
        np.testing.assert_array_equal(rad, want)


def test_row_subset_matches_full_frame():
    c = G.frame_case("sweep_160x90_s16_b5_sky")
    full = G.frame_pixels(c["name"]).reshape(c["height"], c["width"])
    cam = c["camera"]
    part = oracle.render(G.packed_scene(c), cam["position"], cam["yaw"], cam["pitch"], cam["fov"], c["width"],
                         c["height"], c["samples"], c["bounces"], row0=3, row_step=7).reshape(c["height"], -1)
    np.testing.assert_array_equal(part[3::7], full[3::7])
    assert not part[0].any()


@pytest.mark.parametrize("rc", [r["name"] for r in G.ray_cases()])
def test_rays_match_reference_iterative_and_recursive(rc):
    entry = next(r for r in G.ray_cases() if r["name"] == rc)
    a = G.ray_arrays(rc)
    ps = G.packed_scene(entry)
    got = np.zeros_like(a["iterative"])
    for lim in range(4):
        m = a["limits"] == lim
        got[m] = oracle.trace_rays(ps, a["origins"][m], a["dirs"][m], entry["samples"], lim)
    np.testing.assert_array_equal(got, a["iterative"])
    # the reference's recursive oracle tolerance (test_acceptance.py:155)
    assert np.abs(got - a["recursive"]).max() < 1e-4


def test_camera_kats():
    # test_camera.py:66-100
    d = oracle.primary_directions([640], [360], 1280, 720, 0.0, 0.0, 60.0)[0]
    np.testing.assert_allclose(d, (0, 0, 1), atol=1e-9)
    d = oracle.primary_directions([640], [360], 1280, 720, math.pi / 2, 0.0, 60.0)[0]
    np.testing.assert_allclose(d, (1, 0, 0), atol=1e-9)
    d = oracle.primary_directions([0], [360], 1280, 720, 0.0, 0.0, 90.0)[0]
    w = np.array([-1.7777777777777777, 0.0, 1.0])
    np.testing.assert_allclose(d, w / np.linalg.norm(w), atol=1e-9)
    assert oracle.viewport_distance(60.0) == pytest.approx(1.7320508075688772, abs=1e-9)


def test_disc_table_kats():
    # shading.py:29 / test_shading.py:78-83: second of four samples at r = 0.5
    t = oracle.disc_table(4, 0.5)
    assert t[0].tolist() == [0.0, 0.0]
    assert math.hypot(*t[1]) == pytest.approx(0.5, abs=1e-9)
    assert math.atan2(t[1][1], t[1][0]) == pytest.approx(2.399963229728653, abs=1e-12)


def test_sky_kats():
    # test_renderer.py:76-97 on the 8x4 gradient fixture
    sky = G.sky_texels("grad:8:4")
    out = oracle.sky_samples([(0.0, 1.0, 0.0), (0.0, -1.0, 0.0), (0.0, 0.0, 1.0)], sky)
    assert out[0][1] == pytest.approx(0.0)
    assert out[1][1] == pytest.approx(3 / 4)
    assert out[2][0] == pytest.approx(4 / 8) and out[2][1] == pytest.approx(2 / 4)
    hdr = np.full((2, 2, 3), 7.5, dtype=np.float32)
    assert oracle.sky_samples([(0.0, 0.0, 1.0)], hdr)[0].tolist() == [1.0, 1.0, 1.0]
