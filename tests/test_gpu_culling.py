"""Exactness of the culled paths on randomised scenes.

The culls (shadow-cone classification, cluster bounds, warp ray bundles) only
skip tests that cannot change a result, so on any scene:
  FP32 (ray form): culled frame == the same kernels with every body left
      undecided (option cull_check), bit for bit;
  FP32 (silhouette form, the default): within the parity gates of the FP64
      oracle, like every FP32 frame;
  FP64: culled frame == literal megakernel frame, bit for bit (and == the oracle).
"""

import numpy as np
import pytest

import oracle
import paper_2305_07450_b200 as rt
import parity
from paper_2305_07450_b200 import _native

pytestmark = pytest.mark.gpu

MODES = {"cull": dict(wave=1, cull=1, conic=1, cull_check=0), "ray": dict(wave=1, cull=1, conic=0, cull_check=0),
         "check": dict(wave=1, cull=1, conic=0, cull_check=1),
         "wave": dict(wave=1, cull=0, conic=1, cull_check=0), "mega": dict(wave=0, cull=0, conic=1, cull_check=0),
         "mega_grid": dict(wave=0, cull=1, conic=1, cull_check=0)}


def random_scene(rng, n_spheres, with_plane=True, light_radius=None, sky=False):
    bodies = []
    for _ in range(n_spheres):
        r = rng.uniform(0.15, 1.2)
        bodies.append(rt.Body.sphere((rng.uniform(-4, 4), rng.uniform(-0.5, 3.0), rng.uniform(0, 8)), r,
                                     tuple(rng.uniform(0.05, 0.95, size=3)), rng.uniform(0, 128)))
    if with_plane:
        bodies.insert(int(rng.integers(0, len(bodies) + 1)), rt.Body.plane(rng.uniform(-1.0, 0.2),
                                                                           tuple(rng.uniform(0.2, 0.8, size=3)),
                                                                           rng.uniform(0, 64)))
    lr = light_radius if light_radius is not None else rng.uniform(0.1, 1.5)
    light = rt.Light((rng.uniform(-5, 5), rng.uniform(3, 9), rng.uniform(-4, 6)), lr)
    s = rt.Scene(bodies=bodies, light=light)
    if sky:
        s.skybox = rt.synthetic_skybox(64, 32)
    return s


def render(scene, cam, params, precision, mode, radiance=False):
    _native.set_options(**MODES[mode])
    try:
        fb = rt.Framebuffer.create(params.width, params.height)
        rad = None
        if radiance:
            rad = np.zeros((params.width * params.height, 3), np.float32 if precision == "fp32" else np.float64)
        rt.render_frame(scene, cam, params, fb, precision=precision, radiance=rad)
        return (fb.pixels.copy(), rad) if radiance else fb.pixels.copy()
    finally:
        _native.set_options(**MODES["cull"])


CASES = [
    # (seed, spheres, samples, bounces, plane, light radius)
    (1, 5, 200, 3, True, None),
    (2, 8, 64, 5, True, 0.05),
    (3, 3, 33, 2, False, 2.5),   # large light: wide cones, many undecided hits
    (4, 12, 16, 4, True, None),  # > 8 spheres: clustered scene, bundle closest hits
    (5, 40, 24, 3, True, None),
    (6, 1, 2049, 1, True, 0.4),  # table beyond shared memory
    (7, 6, 9, 31, True, None),   # deepest bounce budget
    (8, 20, 47, 6, True, 0.8),
]


@pytest.mark.parametrize("seed,n,samples,bounces,plane,lr", CASES)
def test_fp32_paths_bit_identical(seed, n, samples, bounces, plane, lr):
    rng = np.random.default_rng(seed)
    scene = random_scene(rng, n, plane, lr, sky=seed % 2 == 0)
    cam = rt.Camera(position=(rng.uniform(-1, 1), rng.uniform(0.5, 2.5), -5.0), yaw=rng.uniform(-0.3, 0.3),
                    pitch=rng.uniform(-0.3, 0.1), fov=rng.uniform(40, 90))
    params = rt.RenderParams(samples, bounces, 120, 68)
    ray = render(scene, cam, params, "fp32", "ray")
    check = render(scene, cam, params, "fp32", "check")
    np.testing.assert_array_equal(ray, check)
    wave = render(scene, cam, params, "fp32", "wave")
    parity.assert_byte_gate(ray, wave, f"ray vs unculled, seed {seed}")
    # the silhouette form: the reference's predicate, FP32 rounding near silhouettes
    px, rad = render(scene, cam, params, "fp32", "cull", radiance=True)
    ps = rt.pack_scene(scene)
    want, want_rad = oracle.render(vars(ps), cam.position, cam.yaw, cam.pitch, cam.fov, 120, 68, samples, bounces,
                                   radiance=True)
    parity.assert_byte_gate(px, want, f"silhouette seed {seed}")
    parity.assert_radiance_gate(rad, want_rad, f"silhouette seed {seed}")


MEGA_CASES = [
    # (seed, spheres, samples, bounces, plane, light radius)
    (11, 5, 1, 1, True, None),
    (12, 8, 1, 0, True, 2.0),
    (13, 3, 4, 3, False, 0.3),
    (14, 6, 7, 2, True, 1.2),
    (15, 5, 40, 3, True, None),   # soft shadows on the megakernel (option wave off)
    (16, 12, 1, 1, True, None),   # > 8 spheres: no grid
]


@pytest.mark.parametrize("seed,n,samples,bounces,plane,lr", MEGA_CASES)
def test_fp32_megakernel_shadow_grid_exact(seed, n, samples, bounces, plane, lr):
    """The FP32 megakernel skips the spheres the shadow grid rules out for a
    shadow origin's cell (option cull): frames equal the unfiltered ones bit
    for bit, with tiles and with persistent warps."""
    rng = np.random.default_rng(seed)
    scene = random_scene(rng, n, plane, lr, sky=seed % 2 == 0)
    cam = rt.Camera(position=(rng.uniform(-1, 1), rng.uniform(0.5, 2.5), -5.0), yaw=rng.uniform(-0.3, 0.3),
                    pitch=rng.uniform(-0.3, 0.1), fov=rng.uniform(40, 90))
    params = rt.RenderParams(samples, bounces, 160, 90)
    frames = []
    for tiles in (-1, 0, 1):
        _native.set_options(mega_tiles=tiles)
        try:
            frames += [render(scene, cam, params, "fp32", "mega_grid"), render(scene, cam, params, "fp32", "mega")]
        finally:
            _native.set_options(mega_tiles=-1)
    for f in frames[1:]:
        np.testing.assert_array_equal(frames[0], f)
    ps = rt.pack_scene(scene)
    want = oracle.render(vars(ps), cam.position, cam.yaw, cam.pitch, cam.fov, 160, 90, samples, bounces)
    parity.assert_byte_gate(frames[0], want, f"megakernel seed {seed}")


@pytest.mark.parametrize("fov,samples,bounces", [(150.0, 1, 1), (100.0, 200, 2), (60.0, 1, 0), (170.0, 16, 3)])
def test_fp32_primary_boxes_around_the_eye(fov, samples, bounces):
    """Primary-ray sphere boxes (option cull) with spheres behind, beside,
    around and just in front of the eye and wide fields of view: frames equal
    the unboxed ones bit for bit (megakernel: cull off; wavefront: cull_check)."""
    eye = (0.3, 1.2, -2.0)
    bodies = [
        rt.Body.sphere((0.3, 1.2, -5.0), 0.8, (0.8, 0.2, 0.2), 40.0),     # behind
        rt.Body.sphere((0.35, 1.25, -2.05), 0.5, (0.2, 0.8, 0.2), 0.0),   # around the eye
        rt.Body.sphere((2.5, 1.2, -1.9), 0.7, (0.2, 0.2, 0.8), 90.0),     # beside (horizon of the image plane)
        rt.Body.sphere((0.3, 1.1, -1.2), 0.3, (0.9, 0.9, 0.2), 10.0),     # just in front
        rt.Body.sphere((-1.0, 0.8, 3.0), 1.0, (0.5, 0.5, 0.5), 120.0),
        rt.Body.plane(0.0, (0.4, 0.4, 0.4), 16.0),
    ]
    scene = rt.Scene(bodies=bodies, light=rt.Light((-3.0, 6.0, -1.0), 0.5))
    params = rt.RenderParams(samples, bounces, 160, 90)
    for yaw, pitch in [(0.0, 0.0), (3.0, 0.2), (1.57, -0.6), (-2.2, 0.9)]:
        cam = rt.Camera(position=eye, yaw=yaw, pitch=pitch, fov=fov)
        if samples < 8:
            np.testing.assert_array_equal(render(scene, cam, params, "fp32", "mega_grid"),
                                          render(scene, cam, params, "fp32", "mega"))
        else:
            np.testing.assert_array_equal(render(scene, cam, params, "fp32", "ray"),
                                          render(scene, cam, params, "fp32", "check"))


@pytest.mark.parametrize("seed,n,samples,bounces,plane,lr", CASES[:6])
def test_fp64_culled_equals_literal_and_oracle(seed, n, samples, bounces, plane, lr):
    rng = np.random.default_rng(100 + seed)
    scene = random_scene(rng, n, plane, lr, sky=seed % 2 == 1)
    cam = rt.Camera(position=(rng.uniform(-1, 1), rng.uniform(0.5, 2.5), -5.0), yaw=rng.uniform(-0.3, 0.3),
                    pitch=rng.uniform(-0.3, 0.1), fov=rng.uniform(40, 90))
    w, h = (64, 36) if samples > 1000 else (96, 54)
    params = rt.RenderParams(samples, bounces, w, h)
    culled = render(scene, cam, params, "fp64", "cull")
    literal = render(scene, cam, params, "fp64", "mega")
    np.testing.assert_array_equal(culled, literal)
    ps = rt.pack_scene(scene)
    want = oracle.render(vars(ps), cam.position, cam.yaw, cam.pitch, cam.fov, w, h, samples, bounces)
    np.testing.assert_array_equal(culled, want)


def adversarial_scene(kind, rng):
    """Scenes that stress the FP64 lane sampler's exactness band: tiny far
    occluders (badly conditioned silhouettes), a light nearly touching a
    sphere, terminator self-shadowing, and a scene far from the origin."""
    bodies = []
    off = np.array([0.0, 0.0, 0.0])
    lr = 0.6
    if kind == "tiny":
        for _ in range(12):
            bodies.append(rt.Body.sphere(tuple(rng.uniform([-3, 0.5, -1], [3, 5, 8])), rng.uniform(0.005, 0.05),
                                         (0.8, 0.8, 0.8), 16.0))
    elif kind == "near_light":
        bodies.append(rt.Body.sphere((-3.2, 6.1, -1.7), 0.5, (0.9, 0.2, 0.2), 8.0))
        bodies.append(rt.Body.sphere((0.0, 0.8, 1.6), 0.8, (0.1, 0.5, 0.1), 32.0))
        lr = 1.1
    elif kind == "terminator":
        for i in range(6):
            bodies.append(rt.Body.sphere((-3.0 + 1.2 * i, 0.5, 2.0 + 0.3 * i), 0.5, (0.7, 0.7, 0.2), 64.0))
    elif kind == "far":
        off = np.array([1000.0, 0.0, -2000.0])
        for _ in range(6):
            c = rng.uniform([-3, 0.3, 0], [3, 2.5, 6]) + off
            bodies.append(rt.Body.sphere(tuple(c), rng.uniform(0.2, 1.0), (0.5, 0.6, 0.7), 32.0))
    bodies.append(rt.Body.plane(0.0, (0.4, 0.45, 0.5), 16.0))
    light = rt.Light(tuple(np.array([-4.0, 7.0, -2.0]) + off), lr)
    cam = rt.Camera(position=tuple(np.array([0.0, 1.4, -4.5]) + off), yaw=0.0, pitch=-0.08, fov=60.0)
    return rt.Scene(bodies=bodies, light=light), cam


@pytest.mark.parametrize("kind", ["tiny", "near_light", "terminator", "far"])
def test_fp64_lane_sampler_exact_on_adversarial_scenes(kind):
    scene, cam = adversarial_scene(kind, np.random.default_rng(7))
    params = rt.RenderParams(64, 3, 128, 72)
    culled = render(scene, cam, params, "fp64", "cull")
    literal = render(scene, cam, params, "fp64", "mega")
    np.testing.assert_array_equal(culled, literal)


@pytest.mark.parametrize("seed,n,bounces,w,h", [(21, 12, 4, 120, 68), (22, 40, 8, 97, 53), (23, 300, 6, 64, 36),
                                                 (24, 24, 31, 33, 17)])
def test_fp32_compaction_bit_identical(seed, n, bounces, w, h):
    """The many-sphere trace's CTA-level compaction of live rays (option
    compact: ray state migrated between threads, records in HBM, pixels
    finished when their ray ends) changes no bit: frames and radiance equal
    the uncompacted kernel's, with 1 and 3 row partitions, silhouette and ray
    forms, frame after frame."""
    rng = np.random.default_rng(seed)
    scene = random_scene(rng, n, True, None, sky=seed % 2 == 1)
    for b in scene.bodies:  # mirrors: deep chains
        if b.kind == rt.BodyKind.SPHERE:
            b.reflectivity = 128.0
    cam = rt.Camera(position=(0.0, 1.2, -5.0), yaw=0.05, pitch=-0.1, fov=70.0)
    params = rt.RenderParams(16, bounces, w, h)
    try:
        for conic in (1, 0):
            out = {}
            for compact in (0, 1):
                _native.set_options(wave=1, cull=1, conic=conic, cull_check=0, compact=compact)
                for workers in (None, 3):
                    for rep in range(2):
                        fb = rt.Framebuffer.create(w, h)
                        rad = np.zeros((w * h, 3), np.float32)
                        rt.render_frame(scene, cam, params, fb, workers, radiance=rad)
                        out.setdefault((workers, rep), []).append((fb.pixels.copy(), rad))
            for key, ((p0, r0), (p1, r1)) in out.items():
                np.testing.assert_array_equal(p1, p0, err_msg=f"seed {seed} conic {conic} {key}")
                np.testing.assert_array_equal(r1, r0, err_msg=f"seed {seed} conic {conic} {key}")
    finally:
        _native.set_options(compact=1, **MODES["cull"])
