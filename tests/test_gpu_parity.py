"""GPU parity: the sm_100a kernels through the C ABI (render_frame /
trace_rays / skybox_sample) against the reference's golden fixtures and the
oracle, at fixture sizes and at BASELINE.json's full sizes.

FP64 kernel: bit-identical framebuffers (the reference's golden sha256 and
every fixture frame).  FP32 kernel: the north-star gates — per 8-bit channel
|delta| <= 1 on >= 99.9% of pixels, radiance |delta| <= 1e-4*max(|ref|,1) on
>= 99.9% of pixels (tests/parity.py).
"""

import hashlib

import numpy as np
import pytest

import golden_cases as G
import oracle
import parity
import paper_2305_07450_b200 as rt
from paper_2305_07450_b200 import _native

pytestmark = pytest.mark.gpu

CASES = [c["name"] for c in G.frame_cases()]

# FP32 execution paths: wavefront + exact culling with the silhouette-form
# penumbra test (default), the same with the ray form, wavefront without
# culling, and the one-thread-per-pixel megakernel
MODES = {"cull": dict(wave=True, cull=True, conic=True), "ray": dict(wave=True, cull=True, conic=False),
         "wave": dict(wave=True, cull=False), "mega": dict(wave=False, cull=False)}


@pytest.fixture(params=list(MODES))
def fp32_mode(request):
    _native.set_options(**MODES[request.param])
    yield request.param
    _native.set_options(**MODES["cull"])


class _Sky:
    def __init__(self, texels):
        self.texels = texels
        self.height, self.width = texels.shape[:2]


def scene_from_case(c):
    """Reference-layout fixture -> this package's Scene (through the public types)."""
    s = c["scene"]
    bodies = []
    for k, p, size, col, refl in zip(s["kinds"], s["positions"], s["sizes"], s["colors"], s["refls"]):
        if k == 0:
            bodies.append(rt.Body.sphere(tuple(p), size, tuple(col), refl))
        else:
            bodies.append(rt.Body.plane(p[1], tuple(col), refl))
    sky = None
    if c.get("sky"):
        t = G.sky_texels(c["sky"])
        sky = rt.Skybox(t.shape[1], t.shape[0], t)
    return rt.Scene(bodies=bodies, light=rt.Light(tuple(s["light_pos"]), s["light_radius"], tuple(s["light_color"])),
                    skybox=sky, ambient=s["ambient"], max_reflectivity=s["max_refl"])


def render_case(c, precision, workers=None, radiance=False):
    scene = scene_from_case(c)
    cam = rt.Camera(**{**c["camera"], "position": tuple(c["camera"]["position"])})
    params = rt.RenderParams(c["samples"], c["bounces"], c["width"], c["height"])
    fb = rt.Framebuffer.create(c["width"], c["height"])
    rad = None
    if radiance:
        rad = np.zeros((c["width"] * c["height"], 3), np.float64 if precision == "fp64" else np.float32)
    rt.render_frame(scene, cam, params, fb, workers=workers, precision=precision, radiance=rad)
    return fb.pixels.copy(), rad


def test_device_visible_and_library_loaded():
    assert _native.device_count() >= 1
    assert _native.load().rt_version() == 1


def test_golden_sha256_fp64():
    c = G.frame_case("bench_128x72_s200_b3")
    px, _ = render_case(c, "fp64")
    assert hashlib.sha256(px.tobytes()).hexdigest() == G.GOLDEN_SHA_128x72_S200_B3


@pytest.mark.parametrize("name", CASES)
def test_fp64_frames_bit_exact(name):
    c = G.frame_case(name)
    px, rad = render_case(c, "fp64", radiance=True)
    np.testing.assert_array_equal(px, G.frame_pixels(name))
    want = G.frame_radiance(name)
    if want is not None:
        # device pow/atan2/asin may differ from glibc in the last ulp
        np.testing.assert_allclose(rad, want, rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", CASES)
def test_fp32_frames_byte_and_radiance_gates(name, fp32_mode):
    c = G.frame_case(name)
    px, rad = render_case(c, "fp32", radiance=True)
    frac, worst = parity.assert_byte_gate(px, G.frame_pixels(name), f"{name} [{fp32_mode}]")
    assert np.all(px >> 24 == 0xFF)
    cam = c["camera"]
    _, want = oracle.render(G.packed_scene(c), cam["position"], cam["yaw"], cam["pitch"], cam["fov"], c["width"],
                            c["height"], c["samples"], c["bounces"], radiance=True)
    parity.assert_radiance_gate(rad, want, f"{name} [{fp32_mode}]")


def test_culled_path_is_exact_against_unculled():
    """Culling only skips bodies that cannot block: the culled FP32 frames
    (ray form) equal, bit for bit, those of the same kernels with every body
    left undecided (option cull_check: each hit sampled against all bodies),
    and the unculled wavefront's within the parity gates."""
    for name in ("bench_128x72_s200_b3", "sweep_160x90_s16_b5_sky", "stress_96x54_s500_b8", "random4_64x36_s16_b4",
                 "c3like_192x108_s200_b3_sky", "blocked_32x18_s4_b1"):
        c = G.frame_case(name)
        try:
            _native.set_options(wave=True, cull=True, conic=False, cull_check=True)
            ref, rref = render_case(c, "fp32", radiance=True)
            _native.set_options(wave=True, cull=True, conic=False, cull_check=False)
            got, rgot = render_case(c, "fp32", radiance=True)
            _native.set_options(wave=True, cull=False)
            wave, rwave = render_case(c, "fp32", radiance=True)
        finally:
            _native.set_options(cull_check=False, **MODES["cull"])
        np.testing.assert_array_equal(got, ref, err_msg=name)
        np.testing.assert_array_equal(rgot, rref, err_msg=name)
        parity.assert_byte_gate(got, wave, name)
        parity.assert_radiance_gate(rgot, rwave, name)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_worker_counts_do_not_change_pixels(precision, fp32_mode):
    # test_renderer.py:229-238 / test_acceptance.py:115-118 with workers = row-block partitions
    c = G.frame_case("sweep_160x90_s16_b5_sky")
    base, _ = render_case(c, precision)
    for workers in (1, 2, 3, 8, 13):
        px, _ = render_case(c, precision, workers=workers)
        np.testing.assert_array_equal(px, base)


def test_repeated_renders_bit_identical():
    c = G.frame_case("bench_128x72_s200_b3")
    first, _ = render_case(c, "fp32")
    for _ in range(3):
        again, _ = render_case(c, "fp32")
        np.testing.assert_array_equal(again, first)


@pytest.mark.parametrize("rc", [r["name"] for r in G.ray_cases()])
def test_trace_rays_against_reference(rc):
    entry = next(r for r in G.ray_cases() if r["name"] == rc)
    a = G.ray_arrays(rc)
    scene = scene_from_case(entry)
    for lim in range(4):
        m = a["limits"] == lim
        params = rt.RenderParams(entry["samples"], lim, 1, 1)
        got64 = rt.trace_rays(a["origins"][m], a["dirs"][m], scene, params, precision="fp64")
        np.testing.assert_allclose(got64, a["iterative"][m], rtol=0, atol=1e-12)
        got32 = rt.trace_rays(a["origins"][m], a["dirs"][m], scene, params, precision="fp32")
        frac, _ = parity.radiance_gate(got32, a["iterative"][m])
        # 15 rays per limit: at most one shadow-sample decision flip
        assert frac >= 14 / 15


def test_empty_scene_renders_black():
    # test_renderer.py:217-221
    scene = rt.Scene(bodies=[], light=rt.Light((0, 5, 0), 0.5))
    for prec in ("fp32", "fp64"):
        fb = rt.Framebuffer.create(1, 1)
        rt.render_frame(scene, rt.Camera(), rt.RenderParams(1, 1, 1, 1), fb, precision=prec)
        assert fb.pixels[0] == 0xFF000000


def test_dimension_mismatch_and_bounce_cap_rejected():
    scene = rt.build_benchmark_scene()
    with pytest.raises(ValueError):
        rt.render_frame(scene, rt.Camera(), rt.RenderParams(1, 1, 8, 8), rt.Framebuffer.create(4, 4))
    with pytest.raises(ValueError):
        rt.render_frame(scene, rt.Camera(), rt.RenderParams(1, 32, 4, 4), rt.Framebuffer.create(4, 4))
    with pytest.raises(ValueError):
        rt.ray_trace_iterative(rt.Ray((0, 1, -3), (0, 0, 1)), scene, rt.RenderParams(4, 32, 1, 1))


def _small_scene(skybox=None):  # test_renderer.py:31-40
    return rt.Scene(
        bodies=[
            rt.Body.sphere((0.0, 1.0, 4.0), 1.0, (0.8, 0.2, 0.1), 64.0),
            rt.Body.sphere((1.5, 0.6, 2.5), 0.6, (0.2, 0.7, 0.3), 128.0),
            rt.Body.plane(0.0, (0.5, 0.5, 0.55), 16.0),
        ],
        light=rt.Light((-3.0, 6.0, -1.0), 0.5),
        skybox=skybox,
    )


def test_reductions_exact_fp64():
    # test_acceptance.py:177-227, test_renderer.py:124-188
    blocked = rt.Scene(
        bodies=[rt.Body.sphere((0.0, 5.0, 0.0), 3.0, (0.3, 0.3, 0.3)), rt.Body.plane(0.0, (0.6, 0.5, 0.4))],
        light=rt.Light((0.0, 10.0, 0.0), 0.5),
        ambient=0.15,
    )
    down = np.array((0.0, -1.0, 0.02))
    down /= np.sqrt(down @ down)
    got = rt.ray_trace_iterative(rt.Ray((0.0, 1.0, 0.0), tuple(down)), blocked, rt.RenderParams(1, 0, 1, 1),
                                 precision="fp64")
    assert got == tuple(c * 0.15 for c in (0.6, 0.5, 0.4))
    # zero-reflectivity scene: output invariant in the bounce limit, exactly
    flat = rt.build_benchmark_scene()
    for b in flat.bodies:
        b.reflectivity = 0.0
    for prec in ("fp32", "fp64"):
        imgs = []
        for limit in (0, 1, 3, 5):
            fb = rt.Framebuffer.create(48, 27)
            rt.render_frame(flat, rt.benchmark_camera(), rt.RenderParams(2, limit, 48, 27), fb, precision=prec)
            imgs.append(fb.tobytes())
        assert all(i == imgs[0] for i in imgs)
    # miss: unshaded sky, or black without a sky
    sky = _Sky(G.sky_texels("grad:8:4"))
    d = np.array((0.3, 0.8, -0.5))
    d /= np.sqrt(d @ d)
    params = rt.RenderParams(4, 2, 1, 1)
    sc = _small_scene(skybox=rt.Skybox(8, 4, sky.texels))
    got = rt.ray_trace_iterative(rt.Ray((0.0, 1.0, -3.0), tuple(d)), sc, params, precision="fp64")
    assert got == rt.skybox_sample(tuple(d), sky)
    assert rt.ray_trace_iterative(rt.Ray((0.0, 1.0, -3.0), tuple(d)), _small_scene(), params,
                                  precision="fp64") == (0.0, 0.0, 0.0)


def test_skybox_sample_kats_and_oracle():
    sky = _Sky(G.sky_texels("grad:8:4"))
    assert rt.skybox_sample((0.0, 1.0, 0.0), sky)[1] == pytest.approx(0.0)
    assert rt.skybox_sample((0.0, -1.0, 0.0), sky)[1] == pytest.approx(3 / 4)
    got = rt.skybox_sample((0.0, 0.0, 1.0), sky)
    assert got[0] == pytest.approx(4 / 8) and got[1] == pytest.approx(2 / 4)
    assert rt.skybox_sample((0.0, 0.0, 1.0), _Sky(np.full((2, 2, 3), 7.5, np.float32))) == (1.0, 1.0, 1.0)
    rng = np.random.default_rng(5)
    dirs = rng.normal(size=(500, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    big = _Sky(G.sky_texels("hdr:64:32"))
    np.testing.assert_array_equal(rt.skybox_sample(dirs, big), oracle.sky_samples(dirs, big.texels))


@pytest.mark.slow
def test_full_size_c2_fp64_bit_exact_vs_oracle_and_fp32_gate():
    """C2 at its full size (1280x720 s200 b3): FP64 kernel == oracle bit for
    bit, FP32 kernel within the byte gate."""
    cfg = rt.CONFIGS["C2"]
    scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
    fb64 = rt.Framebuffer.create(cfg.width, cfg.height)
    rt.render_frame(scene, cam, params, fb64, precision="fp64")
    ps = rt.pack_scene(scene)
    want = oracle.render(vars(ps), cam.position, cam.yaw, cam.pitch, cam.fov, cfg.width, cfg.height, cfg.samples,
                         cfg.bounces)
    np.testing.assert_array_equal(fb64.pixels, want)
    fb32 = rt.Framebuffer.create(cfg.width, cfg.height)
    rt.render_frame(scene, cam, params, fb32, precision="fp32")
    parity.assert_byte_gate(fb32.pixels, want, "C2 fp32")


@pytest.mark.slow
@pytest.mark.parametrize("key", ["C3", "C4"])
def test_full_size_sky_configs_fp32_vs_fp64(key):
    """C3/C4 at full size with the 2048x1024 sky: FP32 within the byte gate of
    the bit-exact FP64 kernel; row-block partitions do not change a byte."""
    cfg = rt.CONFIGS[key]
    scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
    fb64 = rt.Framebuffer.create(cfg.width, cfg.height)
    rt.render_frame(scene, cam, params, fb64, precision="fp64")
    fb32 = rt.Framebuffer.create(cfg.width, cfg.height)
    rt.render_frame(scene, cam, params, fb32, precision="fp32")
    parity.assert_byte_gate(fb32.pixels, fb64.pixels, f"{key} fp32 vs fp64")
    fb8 = rt.Framebuffer.create(cfg.width, cfg.height)
    rt.render_frame(scene, cam, params, fb8, workers=8, precision="fp32")
    np.testing.assert_array_equal(fb8.pixels, fb32.pixels)
    # exact on a strided row subset against the oracle
    ps = rt.pack_scene(scene)
    sub = oracle.render(vars(ps), cam.position, cam.yaw, cam.pitch, cam.fov, cfg.width, cfg.height, cfg.samples,
                        cfg.bounces, row0=5, row_step=97).reshape(cfg.height, cfg.width)
    np.testing.assert_array_equal(fb64.pixels.reshape(cfg.height, cfg.width)[5::97], sub[5::97])


@pytest.mark.slow
def test_full_size_c5_stress_row_subset_vs_oracle():
    """C5 (256 spheres + plane, s500 b8) at its full 3840x2160: every 216th row
    against the oracle — the clustered closest hit and the cluster-level cone
    cull must leave the FP32 frame within the byte gate; the FP64 kernel is
    exact on the same rows."""
    cfg = rt.CONFIGS["C5"]
    scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
    fb = rt.Framebuffer.create(cfg.width, cfg.height)
    rt.render_frame(scene, cam, params, fb, precision="fp32")
    ps = rt.pack_scene(scene)
    want = oracle.render(vars(ps), cam.position, cam.yaw, cam.pitch, cam.fov, cfg.width, cfg.height, cfg.samples,
                         cfg.bounces, row0=100, row_step=216).reshape(cfg.height, cfg.width)[100::216]
    got = fb.pixels.reshape(cfg.height, cfg.width)[100::216]
    parity.assert_byte_gate(got.reshape(-1), want.reshape(-1), "C5 fp32 rows")
    fb64 = rt.Framebuffer.create(cfg.width, cfg.height)
    rt.render_frame(scene, cam, params, fb64, precision="fp64")
    np.testing.assert_array_equal(fb64.pixels.reshape(cfg.height, cfg.width)[100::216], want)


def test_clustered_scene_modes_agree():
    """A 40-sphere scene (clustered: > 8 spheres) renders the same bytes on the
    culled wavefront, the unculled wavefront and the megakernel."""
    s = rt.stress_scene(count=40, seed=7)
    cam = rt.Camera(position=(0.0, 2.0, -6.0), yaw=0.1, pitch=-0.12, fov=70.0)
    params = rt.RenderParams(32, 4, 160, 90)
    frames = {}
    for mode, opts in MODES.items():
        _native.set_options(**opts)
        fb = rt.Framebuffer.create(160, 90)
        rt.render_frame(s, cam, params, fb)
        frames[mode] = fb.pixels.copy()
    _native.set_options(**MODES["cull"])
    parity.assert_byte_gate(frames["ray"], frames["wave"], "clustered ray vs wave")
    fb64 = rt.Framebuffer.create(160, 90)
    rt.render_frame(s, cam, params, fb64, precision="fp64")
    for mode, px in frames.items():
        parity.assert_byte_gate(px, fb64.pixels, f"clustered [{mode}]")


def test_moving_bodies_between_frames():
    """The physics step moves spheres between frames (physics.py:49-72); the
    scene cache must upload the change (the paper's per-frame streamIn)."""
    scene, cam = rt.build_benchmark_scene(), rt.benchmark_camera()
    params = rt.RenderParams(16, 2, 64, 36)
    for step in range(3):
        fb = rt.Framebuffer.create(64, 36)
        rt.render_frame(scene, cam, params, fb, precision="fp64")
        ps = rt.pack_scene(scene)
        want = oracle.render(vars(ps), cam.position, cam.yaw, cam.pitch, cam.fov, 64, 36, 16, 2)
        np.testing.assert_array_equal(fb.pixels, want)
        for i in (3, 4):  # BENCHMARK_DYNAMIC_SPHERES (sceneio.py:311)
            b = scene.bodies[i]
            b.position = (b.position[0] + 0.15, b.position[1] + 0.05 * (step + 1), b.position[2] - 0.1)
        scene.light.position = (scene.light.position[0] + 0.2, scene.light.position[1], scene.light.position[2])


@pytest.mark.parametrize("count,samples", [(300, 1), (300, 16), (1100, 4)])
def test_large_scenes_take_the_memory_paths(count, samples):
    """Scenes beyond the launch-parameter layout (> 256 spheres) run from
    shared / global memory; FP32 stays within the byte gate of the FP64
    kernel, which matches the oracle exactly."""
    s = rt.stress_scene(count=count, seed=11)
    cam = rt.Camera(position=(0.0, 2.0, -5.0), yaw=0.05, pitch=-0.15, fov=70.0)
    w, h = (48, 27) if count > 1000 else (96, 54)
    params = rt.RenderParams(samples, 3, w, h)
    fb32 = rt.Framebuffer.create(w, h)
    rt.render_frame(s, cam, params, fb32)
    fb64 = rt.Framebuffer.create(w, h)
    rt.render_frame(s, cam, params, fb64, precision="fp64")
    ps = rt.pack_scene(s)
    want = oracle.render(vars(ps), cam.position, cam.yaw, cam.pitch, cam.fov, w, h, samples, 3)
    np.testing.assert_array_equal(fb64.pixels, want)
    parity.assert_byte_gate(fb32.pixels, want, f"{count} spheres")


def test_many_planes():
    """More planes than the launch-parameter layout holds (8)."""
    s = rt.build_benchmark_scene()
    for k in range(10):
        s.bodies.append(rt.Body.plane(-1.0 - 0.1 * k, (0.2, 0.3, 0.4 + 0.05 * k), 8.0))
    s.bodies.append(rt.Body.plane(9.0, (0.9, 0.9, 0.9), 0.0))  # a ceiling above the light: shadows everything
    cam, params = rt.benchmark_camera(), rt.RenderParams(12, 2, 64, 36)
    fb32 = rt.Framebuffer.create(64, 36)
    rt.render_frame(s, cam, params, fb32)
    ps = rt.pack_scene(s)
    want = oracle.render(vars(ps), cam.position, cam.yaw, cam.pitch, cam.fov, 64, 36, 12, 2)
    parity.assert_byte_gate(fb32.pixels, want, "many planes")


def test_zero_copy_option_gives_the_same_frame():
    c = G.frame_case("sweep_160x90_s16_b5_sky")
    base, _ = render_case(c, "fp32")
    _native.set_options(zero_copy=1)
    try:
        scene = scene_from_case(c)
        cam = rt.Camera(**{**c["camera"], "position": tuple(c["camera"]["position"])})
        params = rt.RenderParams(c["samples"], c["bounces"], c["width"], c["height"])
        fb = rt.Framebuffer.create(c["width"], c["height"])
        _native.context(1).pin(fb.pixels)  # registered + mapped: the kernels write it directly
        rt.render_frame(scene, cam, params, fb)
        np.testing.assert_array_equal(fb.pixels, base)
    finally:
        _native.set_options(zero_copy=0)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_copy_overlap_bands_do_not_change_pixels(precision):
    """rt_render_v1's row bands (option bands, 1-8, each on its own stream,
    copied as soon as it is done; band_first sizes band 0) partition the
    frame: same bytes, same radiance, with and without several partitions
    inside each band."""
    s = rt.build_benchmark_scene()
    cam = rt.benchmark_camera()
    params = rt.RenderParams(32, 3, 240, 136)
    dt = np.float32 if precision == "fp32" else np.float64
    ref = None
    ctx = _native.context(1)
    try:
        for bands, first in ((1, 0), (2, 0), (3, 0), (5, 0), (8, 0), (2, 700), (4, 450), (3, 999), (6, 1)):
            for workers in (None, 3):
                _native.set_options(bands=bands, band_first=first, band_times=1)
                fb = rt.Framebuffer.create(240, 136)
                rad = np.zeros((240 * 136, 3), dt)
                rt.render_frame(s, cam, params, fb, workers, precision=precision, radiance=rad)
                if ref is None:
                    ref = (fb.pixels.copy(), rad.copy())
                tag = f"bands={bands} first={first} workers={workers}"
                np.testing.assert_array_equal(fb.pixels, ref[0], err_msg=tag)
                np.testing.assert_array_equal(rad, ref[1], err_msg=tag)
                if workers is None:  # band_times: per band, kernels end before the copy ends, in band order
                    times = ctx.band_times_ms()
                    assert len(times) == bands, tag
                    assert all(0.0 <= k <= c for k, c in times), (tag, times)
                    assert all(a[1] <= b[1] for a, b in zip(times, times[1:])), (tag, times)
    finally:
        _native.set_options(bands=0, band_first=0, band_times=0)


def _edge_cases():
    """Small scenes at the edges of the renderer's domain, each rendered on
    every path and checked against the oracle."""
    bench = rt.build_benchmark_scene()
    cam = rt.benchmark_camera()
    cases = {}
    # frame shapes off the 16x8 tile grid, and a 1-pixel frame
    cases["1x1_s200_b3"] = (bench, cam, rt.RenderParams(200, 3, 1, 1))
    cases["17x9_s200_b3"] = (bench, cam, rt.RenderParams(200, 3, 17, 9))
    cases["9x31_s16_b2"] = (bench, cam, rt.RenderParams(16, 2, 9, 31))
    # the wavefront threshold (8 samples) and one below it
    cases["48x27_s8_b3"] = (bench, cam, rt.RenderParams(8, 3, 48, 27))
    cases["48x27_s7_b3"] = (bench, cam, rt.RenderParams(7, 3, 48, 27))
    # the deepest bounce budget, in a hall of mirrors
    mirrors = rt.Scene(bodies=[rt.Body.sphere((-1.1, 1.0, 2.0), 1.0, (0.9, 0.9, 0.9), 128.0),
                               rt.Body.sphere((1.1, 1.0, 2.0), 1.0, (0.9, 0.9, 0.9), 128.0),
                               rt.Body.plane(0.0, (0.5, 0.5, 0.5), 128.0)],
                       light=rt.Light((0.0, 6.0, -2.0), 0.4), max_reflectivity=128.0)
    cases["mirrors_32x18_s16_b31"] = (mirrors, cam, rt.RenderParams(16, 31, 32, 18))
    # a near-point light (the reference requires a positive radius)
    point = rt.Scene(bodies=list(bench.bodies), light=rt.Light((-4.0, 7.0, -2.0), 1e-6))
    cases["pointlight_48x27_s16_b2"] = (point, cam, rt.RenderParams(16, 2, 48, 27))
    # the light inside a sphere, and the camera inside a sphere
    inside = rt.Scene(bodies=list(bench.bodies) + [rt.Body.sphere((-4.0, 7.0, -2.0), 1.5, (0.9, 0.9, 0.2), 8.0)],
                      light=rt.Light((-4.0, 7.0, -2.0), 0.6))
    cases["light_inside_48x27_s32_b2"] = (inside, cam, rt.RenderParams(32, 2, 48, 27))
    shell = rt.Scene(bodies=list(bench.bodies) + [rt.Body.sphere(cam.position, 0.5, (0.3, 0.6, 0.9), 16.0)],
                     light=rt.Light((-4.0, 7.0, -2.0), 0.6))
    cases["camera_inside_48x27_s32_b2"] = (shell, cam, rt.RenderParams(32, 2, 48, 27))
    # a light larger than the distance to the nearest surfaces
    huge = rt.Scene(bodies=list(bench.bodies), light=rt.Light((0.0, 3.0, 1.0), 2.5))
    cases["hugelight_48x27_s64_b2"] = (huge, cam, rt.RenderParams(64, 2, 48, 27))
    return cases


EDGE = _edge_cases()


@pytest.mark.parametrize("name", sorted(EDGE))
def test_edge_cases_against_oracle(name):
    scene, cam, params = EDGE[name]
    w, h = params.width, params.height
    ps = rt.pack_scene(scene)
    want, want_rad = oracle.render(vars(ps), cam.position, cam.yaw, cam.pitch, cam.fov, w, h,
                                   params.shadow_samples, params.bounce_limit, radiance=True)
    fb = rt.Framebuffer.create(w, h)
    rt.render_frame(scene, cam, params, fb, precision="fp64")
    np.testing.assert_array_equal(fb.pixels, want, err_msg=f"{name} fp64")
    try:
        for mode, opts in MODES.items():
            _native.set_options(**opts)
            fb = rt.Framebuffer.create(w, h)
            rad = np.zeros((w * h, 3), np.float32)
            rt.render_frame(scene, cam, params, fb, precision="fp32", radiance=rad)
            if w * h >= 1000:
                parity.assert_byte_gate(fb.pixels, want, f"{name} [{mode}]")
                parity.assert_radiance_gate(rad, want_rad, f"{name} [{mode}]")
            else:  # too few pixels for a 99.9% gate: every channel within 1
                frac, worst = parity.byte_gate(fb.pixels, want)
                assert worst <= 1, f"{name} [{mode}]: worst channel delta {worst}"
    finally:
        _native.set_options(**MODES["cull"])


def test_512_sphere_scene_culled_path():
    """SURVEY.md §8d's 512-sphere stress scene takes the culled path (launch-
    parameter scene of up to 512 spheres, candidate lists in chunks): exact
    against its own cull_check frame, within the gates of the oracle, and the
    FP64 frame bit-identical to it."""
    s = rt.stress_scene(count=512)
    cam = rt.CONFIGS["C5"].camera()
    params = rt.RenderParams(32, 4, 96, 54)
    ps = rt.pack_scene(s)
    want, want_rad = oracle.render(vars(ps), cam.position, cam.yaw, cam.pitch, cam.fov, 96, 54, 32, 4, radiance=True)
    frames = {}
    try:
        for name, opts in (("check", dict(wave=True, cull=True, conic=False, cull_check=True)),
                           ("ray", dict(wave=True, cull=True, conic=False, cull_check=False)),
                           ("cull", dict(wave=True, cull=True, conic=True, cull_check=False))):
            _native.set_options(**opts)
            fb = rt.Framebuffer.create(96, 54)
            rad = np.zeros((96 * 54, 3), np.float32)
            rt.render_frame(s, cam, params, fb, radiance=rad)
            frames[name] = (fb.pixels.copy(), rad)
    finally:
        _native.set_options(cull_check=False, **MODES["cull"])
    np.testing.assert_array_equal(frames["ray"][0], frames["check"][0])
    np.testing.assert_array_equal(frames["ray"][1], frames["check"][1])
    for name, (px, rad) in frames.items():
        parity.assert_byte_gate(px, want, f"512 spheres [{name}]")
        parity.assert_radiance_gate(rad, want_rad, f"512 spheres [{name}]")
    fb = rt.Framebuffer.create(96, 54)
    rt.render_frame(s, cam, params, fb, precision="fp64")
    np.testing.assert_array_equal(fb.pixels, want)


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_frame_pipeline_matches_render_frame(depth):
    """FramePipeline (rt_render_async_v1 / rt_frame_wait_v1): a sequence of
    frames with a moving camera and a moving body, several in flight, each
    equal to render_frame's bytes."""
    scene = rt.build_benchmark_scene()
    params = rt.RenderParams(64, 3, 320, 180)
    pipe = rt.FramePipeline(depth)
    cams, outs, tickets, wants = [], [], [], []
    try:
        for i in range(7):
            cam = rt.Camera(position=(0.1 * i, 1.4, -4.5), yaw=0.02 * i, pitch=-0.08, fov=60.0)
            scene.bodies[0].position = (-2.4 + 0.05 * i, 1.0, 2.8)
            fb = rt.Framebuffer.create(320, 180)
            tickets.append(pipe.submit(scene, cam, params, fb))
            outs.append(fb)
            want = rt.Framebuffer.create(320, 180)
            rt.render_frame(scene, cam, params, want)
            wants.append(want.pixels.copy())
        for t, fb, want in zip(tickets, outs, wants):
            if t in pipe._pending:
                pipe.wait(t)
            np.testing.assert_array_equal(fb.pixels, want, err_msg=f"frame {t}")
    finally:
        pipe.close()
    with pytest.raises(ValueError):
        rt.FramePipeline(5)


def test_fast_and_ctypes_paths_give_the_same_frame():
    from paper_2305_07450_b200 import renderer

    cfg = rt.CONFIGS["C3"]
    scene, cam = cfg.scene(), cfg.camera()
    params = rt.RenderParams(64, 3, 320, 180)
    a = rt.Framebuffer.create(320, 180)
    rt.render_frame(scene, cam, params, a)
    saved = list(renderer._FAST)
    renderer._FAST[:] = [None]
    try:
        b = rt.Framebuffer.create(320, 180)
        rt.render_frame(scene, cam, params, b)
    finally:
        renderer._FAST[:] = saved
    np.testing.assert_array_equal(a.pixels, b.pixels)
