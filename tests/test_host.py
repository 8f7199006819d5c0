"""CPU tests of the host side: the reference-mirroring types and their
validation, scene packing against the reference's own packed arrays, the
pure-integer pack_color, argument errors raised before any device work, and
`install()` rebinding a reference-shaped package."""

import math
import sys
import types

import numpy as np
import pytest

import golden_cases as G
import paper_2305_07450_b200 as rt
from paper_2305_07450_b200 import _native


def test_constants_match_reference():
    assert rt.MAX_BOUNCE_LIMIT == 31 and rt.REFLECT_EPS == 1e-3 and rt.SHADOW_EPS == 1e-3
    assert rt.GRAZE_EPS == 1e-7 and rt.DEFAULT_AMBIENT == 0.15 and rt.DEFAULT_MAX_REFLECTIVITY == 128.0
    assert rt.GOLDEN_ANGLE == pytest.approx(2.399963229728653, abs=1e-12)
    assert rt.PITCH_LIMIT == pytest.approx(math.pi / 2 - 1e-3)


def test_pack_color_kats():
    # test_renderer.py:61-73
    assert rt.pack_color((0.0, 0.0, 0.0)) == 0xFF000000
    assert rt.pack_color((1.0, 1.0, 1.0)) == 0xFFFFFFFF
    assert rt.pack_color((1.0, 0.0, 0.0)) == 0xFFFF0000
    assert rt.pack_color((0.0, 1.0, 0.0)) == 0xFF00FF00
    assert rt.pack_color((0.0, 0.0, 1.0)) == 0xFF0000FF
    with pytest.raises(ValueError):
        rt.pack_color((1.5, 0.0, 0.0))


def test_viewport_distance_kats():
    # test_camera.py:51-63
    assert rt.camera_viewport_distance(90.0) == pytest.approx(1.0, abs=1e-12)
    assert rt.camera_viewport_distance(60.0) == pytest.approx(1.7320508075688772, abs=1e-9)
    assert rt.camera_viewport_distance(120.0) == pytest.approx(0.5773502691896257, abs=1e-9)


def test_validation_mirrors_reference():
    with pytest.raises(ValueError):
        rt.Body.sphere((0, 0, 0), -1.0, (1, 0, 0))
    with pytest.raises(ValueError):
        rt.Body.sphere((0, 0, 0), 1.0, (2, 0, 0))
    with pytest.raises(ValueError):
        rt.Body.sphere((0, 0, 0), 1.0, (1, 0, 0), reflectivity=-5)
    with pytest.raises(ValueError):
        rt.Ray((0, 0, 0), (0, 0, 2))
    with pytest.raises(ValueError):
        rt.Light((0, 1, 0), 0.0)
    with pytest.raises(ValueError):
        rt.Camera(fov=0.0)
    with pytest.raises(ValueError):
        rt.Camera(fov=180.0)
    assert rt.Camera(pitch=2.0).pitch == pytest.approx(math.pi / 2 - 1e-3)
    assert rt.Camera(pitch=-2.0).pitch == pytest.approx(-(math.pi / 2 - 1e-3))
    with pytest.raises(ValueError):
        rt.Scene(bodies=[], light=rt.Light((0, 1, 0), 1.0), ambient=1.5)
    with pytest.raises(ValueError):
        rt.Scene(bodies=[rt.Body.sphere((0, 0, 0), 1.0, (1, 1, 1), 200.0)], light=rt.Light((0, 1, 0), 1.0))
    with pytest.raises(ValueError):
        rt.RenderParams(0, 1, 4, 4)
    with pytest.raises(ValueError):
        rt.RenderParams(1, -1, 4, 4)
    with pytest.raises(ValueError):
        rt.RenderParams(1, 1, 0, 4)
    with pytest.raises(ValueError):
        rt.Framebuffer(2, 2, np.zeros(3, np.uint32))
    with pytest.raises(ValueError):
        rt.Framebuffer(2, 2, np.zeros(4, np.int32))
    with pytest.raises(ValueError):
        rt.Skybox(2, 2, np.zeros((2, 3, 3), np.float32))
    assert rt.Ray((1.0, 0.0, 0.0), (0.0, 0.0, 1.0)).at(3.0) == (1.0, 0.0, 3.0)
    assert rt.Body.plane(2.5, (1, 1, 1)).height == 2.5


def test_pack_scene_equals_reference_packing():
    # the fixture holds the reference's own pack_bodies output (geometry.py:162-176)
    c = G.frame_case("bench_128x72_s200_b3")
    ps = rt.pack_scene(rt.build_benchmark_scene())
    want = G.packed_scene(c)
    for k in ("kinds", "positions", "sizes", "colors", "refls", "light_pos", "light_color"):
        np.testing.assert_array_equal(getattr(ps, k), want[k])
        assert getattr(ps, k).flags.c_contiguous
    assert ps.light_radius == want["light_radius"] and ps.ambient == want["ambient"]
    assert ps.max_refl == want["max_refl"] and not ps.has_sky
    assert ps.kinds.dtype == np.int32 and ps.positions.dtype == np.float64


def test_pack_scene_stress_and_sky():
    c = G.frame_case("stress_96x54_s500_b8")
    ps = rt.pack_scene(rt.stress_scene())
    want = G.packed_scene(c)
    for k in ("kinds", "positions", "sizes", "colors", "refls"):
        np.testing.assert_array_equal(getattr(ps, k), want[k])
    sky = rt.synthetic_skybox(64, 32)
    np.testing.assert_array_equal(sky.texels, G.sky_texels("grad:64:32"))
    s = rt.build_benchmark_scene()
    s.skybox = sky
    ps = rt.pack_scene(s)
    assert ps.has_sky and (ps.sky_w, ps.sky_h) == (64, 32) and ps.sky.dtype == np.float32


def test_pack_scene_duck_types_foreign_objects():
    ns = types.SimpleNamespace
    scene = ns(bodies=[ns(kind=0, position=(1, 2, 3), size=0.5, color=(0.1, 0.2, 0.3), reflectivity=4.0)],
               light=ns(position=(0, 9, 0), radius=0.4, color=(1, 1, 1)), skybox=None, ambient=0.2,
               max_reflectivity=64.0)
    ps = rt.pack_scene(scene)
    assert ps.n_bodies == 1 and ps.positions.tolist() == [[1.0, 2.0, 3.0]] and ps.max_refl == 64.0


def test_render_frame_argument_errors_precede_device_work():
    scene = rt.build_benchmark_scene()
    with pytest.raises(ValueError):
        rt.render_frame(scene, rt.Camera(), rt.RenderParams(1, 1, 8, 8), rt.Framebuffer.create(4, 4))
    with pytest.raises(ValueError):
        rt.render_frame(scene, rt.Camera(), rt.RenderParams(1, 32, 4, 4), rt.Framebuffer.create(4, 4))
    with pytest.raises(ValueError):
        rt.render_frame(scene, rt.Camera(), rt.RenderParams(1, 1, 4, 4), rt.Framebuffer.create(4, 4),
                        precision="fp16")
    with pytest.raises(ValueError):
        rt.ray_trace_iterative(rt.Ray((0, 1, -3), (0, 0, 1)), scene, rt.RenderParams(4, 32, 1, 1))


@pytest.mark.skipif(_native.device_count() > 0, reason="checks the GPU-less behaviour")
def test_no_cpu_fallback_without_a_device():
    """The product path fails loudly: no CUDA device, no frame."""
    with pytest.raises(_native.NativeError):
        rt.render_frame(rt.build_benchmark_scene(), rt.benchmark_camera(), rt.RenderParams(1, 1, 4, 4),
                        rt.Framebuffer.create(4, 4))
    with pytest.raises(_native.NativeError):
        rt.trace_rays([(0, 1, -3)], [(0, 0, 1)], rt.build_benchmark_scene(), rt.RenderParams(1, 1, 1, 1))


def test_install_rebinds_every_importer(monkeypatch):
    """raytracer.bench/cli/server import render_frame by name (bench.py:15,
    cli.py:17, server.py:43): install() must rebind all of them."""
    pkg = types.ModuleType("fakeraytracer")
    pkg.__path__ = []
    mods = {}
    sentinel = object()
    for sub in ("renderer", "bench", "cli", "server"):
        m = types.ModuleType(f"fakeraytracer.{sub}")
        m.render_frame = sentinel
        mods[sub] = m
        monkeypatch.setitem(sys.modules, m.__name__, m)
    mods["renderer"].ray_trace_iterative = sentinel
    monkeypatch.setitem(sys.modules, "fakeraytracer", pkg)
    patched = rt.install(package="fakeraytracer")
    try:
        assert len(patched) == 4
        for m in mods.values():
            assert m.render_frame is rt.render_frame
        assert mods["renderer"].ray_trace_iterative is rt.ray_trace_iterative
    finally:
        rt.uninstall()
    for m in mods.values():
        assert m.render_frame is sentinel


def test_work_counts_cover_every_config():
    import json
    import os

    with open(os.path.join(os.path.dirname(rt.__file__), "work_counts.json")) as f:
        wc = json.load(f)["configs"]
    assert set(wc) == set(rt.CONFIGS)
    # SURVEY.md §8d measured numerators
    assert wc["C1"]["flops"] == pytest.approx(4.911e7, rel=1e-3)
    assert wc["C2"]["rays"] == 129_330_618
    assert wc["C4"]["rays"] == 1_164_482_622


def test_cpython_fast_path_packs_or_declines():
    """csrc/pyfast.c: with a null context the C ABI rejects the call after the
    scene was read (RT_ERR_INVALID); a scene it cannot read is declined (None)
    so the ctypes path raises the reference's errors."""
    from paper_2305_07450_b200 import renderer

    fast = renderer._fast()
    if fast is None:
        pytest.skip("the CPython fast path is not built")
    scene = rt.build_benchmark_scene()
    cam = rt.benchmark_camera()
    assert fast.render(0, 1, 0, 8, 8, cam.position, 0.0, 0.0, 1.7, scene, 1, 1, 1, 0) == -1

    class Broken:
        bodies = [object()]
        light = None

    assert fast.render(0, 1, 0, 8, 8, cam.position, 0.0, 0.0, 1.7, Broken(), 1, 1, 1, 0) is None
    sky_scene = rt.build_benchmark_scene()
    sky_scene.skybox = types.SimpleNamespace(width=4, height=2, texels=np.zeros((2, 4, 3)))  # float64: declined
    assert fast.render(0, 1, 0, 8, 8, cam.position, 0.0, 0.0, 1.7, sky_scene, 1, 1, 1, 0) is None
    sky_scene.skybox = rt.Skybox(4, 2, np.zeros((2, 4, 3), dtype=np.float32))  # taken
    assert fast.render(0, 1, 0, 8, 8, cam.position, 0.0, 0.0, 1.7, sky_scene, 1, 1, 1, 0) == -1
