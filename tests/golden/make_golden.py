"""Generate the golden parity fixtures from the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the reference package (/root/reference/pkg/src/raytracer), renders
every case below through the reference's own public ``render_frame``
(renderer.py:316-349), computes float64 radiance frames by calling the
reference's own ``_trace`` per pixel (renderer.py:108-224) and per-ray
``ray_trace_iterative`` (renderer.py:303-313) results, and writes

    tests/golden/cases.json   scene / camera / params per case (packed SoA)
    tests/golden/frames.npz   uint32 framebuffers + float64 radiance frames
    tests/golden/rays.npz     per-ray iterative + recursive-oracle radiance

The GPU box never runs this script; the tests only read its outputs.
"""

import hashlib
import json
import math
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import numpy as np  # noqa: E402
from numba import njit, prange  # noqa: E402

import oracles as ref_oracles  # noqa: E402  (reference's independent recursive oracle)
from raytracer import renderer as R  # noqa: E402
from raytracer import vecmath as vm  # noqa: E402
from raytracer.camera import Camera, camera_viewport_distance, primary_direction  # noqa: E402
from raytracer.geometry import Body, Ray  # noqa: E402
from raytracer.scene import Framebuffer, RenderParams, Scene, Skybox  # noqa: E402
from raytracer.sceneio import benchmark_camera, build_benchmark_scene  # noqa: E402
from raytracer.shading import Light  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN_SHA = "f9841b1c4ee5f6d6a2308d11b564de6c8b54d9e1def48e453a2d43175979ef14"


# --- sky recipes (also implemented in tests/golden_cases.py) -----------------
def sky_texels(recipe):
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


def make_sky(recipe):
    if recipe is None:
        return None
    t = sky_texels(recipe)
    return Skybox(t.shape[1], t.shape[0], t)


# --- scenes -----------------------------------------------------------------
def small_scene(skybox=None):  # test_renderer.py:31-40
    return Scene(
        bodies=[
            Body.sphere((0.0, 1.0, 4.0), 1.0, (0.8, 0.2, 0.1), 64.0),
            Body.sphere((1.5, 0.6, 2.5), 0.6, (0.2, 0.7, 0.3), 128.0),
            Body.plane(0.0, (0.5, 0.5, 0.55), 16.0),
        ],
        light=Light((-3.0, 6.0, -1.0), 0.5),
        skybox=skybox,
    )


def random_scene(rng, with_plane, skybox):  # after test_renderer.py:43-58
    bodies = []
    for _ in range(int(rng.integers(1, 5))):
        bodies.append(Body.sphere((rng.uniform(-3, 3), rng.uniform(0.3, 2.5), rng.uniform(0, 5)),
                                  rng.uniform(0.3, 1.2), tuple(rng.uniform(0.05, 0.95, size=3)),
                                  rng.uniform(0.0, 128.0)))
    if with_plane:
        bodies.append(Body.plane(0.0, tuple(rng.uniform(0.2, 0.8, size=3)), rng.uniform(0, 64)))
    light = Light((rng.uniform(-4, 4), rng.uniform(4, 8), rng.uniform(-4, 4)), rng.uniform(0.2, 0.8))
    return Scene(bodies=bodies, light=light, skybox=skybox)


def stress_scene(count=256, seed=230507450):
    rng = np.random.default_rng(seed)
    bench = build_benchmark_scene()
    bodies = []
    for _ in range(count):
        r = rng.uniform(0.2, 0.6)
        c = (rng.uniform(-10, 10), r + rng.uniform(0, 2), rng.uniform(0.5, 25))
        col = tuple(rng.uniform(0.05, 0.95, size=3))
        bodies.append(Body.sphere(c, r, col, rng.uniform(0, 128)))
    bodies.append(bench.bodies[-1])
    return Scene(bodies=bodies, light=bench.light, ambient=bench.ambient, max_reflectivity=bench.max_reflectivity)


def blocked_scene():  # test_acceptance.py:196-204
    return Scene(
        bodies=[Body.sphere((0.0, 5.0, 0.0), 3.0, (0.3, 0.3, 0.3)), Body.plane(0.0, (0.6, 0.5, 0.4))],
        light=Light((0.0, 10.0, 0.0), 0.5),
        ambient=0.15,
    )


SWEEP_CAMERA = dict(position=(1.35, 0.25, 2.2), yaw=0.75, pitch=-0.12, fov=40.0)  # test_acceptance.py:36
BENCH_CAMERA = dict(position=(0.0, 1.4, -4.5), yaw=0.0, pitch=-0.08, fov=60.0)  # sceneio.py:332-333


def packed(scene):
    kinds, positions, sizes, colors, refls = R.pack_bodies(scene.bodies)
    return dict(
        kinds=kinds.tolist(), positions=positions.tolist(), sizes=sizes.tolist(), colors=colors.tolist(),
        refls=refls.tolist(), light_pos=list(scene.light.position), light_radius=scene.light.radius,
        light_color=list(scene.light.color), ambient=scene.ambient, max_refl=scene.max_reflectivity,
    )


@njit(parallel=True, cache=False)
def _radiance_frame(width, height, cam_pos, yaw, pitch, vdist, kinds, positions, sizes, colors, refls,
                    light_pos, light_radius, light_color, ambient, max_refl, sky, sky_w, sky_h, has_sky,
                    samples, bounces, out):
    # The reference's own per-pixel path (renderer.py:253-278) minus the pack.
    for idx in prange(width * height):
        x = idx % width
        y = idx // width
        d = primary_direction(float(x), float(y), float(width), float(height), yaw, pitch, vdist)
        c = R._trace(cam_pos, d, kinds, positions, sizes, colors, refls, light_pos, light_radius, light_color,
                     ambient, max_refl, sky, sky_w, sky_h, has_sky, samples, bounces)
        out[idx, 0] = c[0]
        out[idx, 1] = c[1]
        out[idx, 2] = c[2]


def radiance_frame(scene, cam, params):
    out = np.zeros((params.width * params.height, 3))
    _radiance_frame(params.width, params.height, cam.position, cam.yaw, cam.pitch,
                    camera_viewport_distance(cam.fov), *R._scene_args(scene), params.shadow_samples,
                    params.bounce_limit, out)
    return out


def main():
    cases = []
    arrays = {}

    def add(name, scene, cam, w, h, s, b, sky=None, radiance=False):
        scene.skybox = make_sky(sky)
        camera = Camera(**cam)
        params = RenderParams(s, b, w, h)
        fb = Framebuffer.create(w, h)
        R.render_frame(scene, camera, params, fb)
        arrays[f"{name}/pixels"] = fb.pixels.copy()
        entry = dict(name=name, scene=packed(scene), sky=sky, camera=cam, width=w, height=h, samples=s,
                     bounces=b, sha256=hashlib.sha256(fb.tobytes()).hexdigest(), radiance=radiance)
        if radiance:
            rad = radiance_frame(scene, camera, params)
            # the radiance path packs exactly like render_frame
            packed_rad = np.array([R.pack_color(tuple(c)) for c in rad], dtype=np.uint32)
            assert np.array_equal(packed_rad, fb.pixels), name
            arrays[f"{name}/radiance"] = rad
        cases.append(entry)
        print(f"{name}: {entry['sha256'][:16]}", flush=True)

    add("bench_128x72_s200_b3", build_benchmark_scene(), BENCH_CAMERA, 128, 72, 200, 3, radiance=True)
    assert cases[-1]["sha256"] == GOLDEN_SHA
    add("c1_640x360_s1_b0", build_benchmark_scene(), BENCH_CAMERA, 640, 360, 1, 0)
    add("paper_256x144_s1_b1", build_benchmark_scene(), BENCH_CAMERA, 256, 144, 1, 1)
    add("sweep_160x90_s16_b5_sky", build_benchmark_scene(), SWEEP_CAMERA, 160, 90, 16, 5, sky="grad:64:32",
        radiance=True)
    add("small_sky_48x27_s5_b2", small_scene(), dict(position=(0.0, 1.2, -4.0), yaw=0.0, pitch=0.0, fov=60.0),
        48, 27, 5, 2, sky="grad:8:4")
    add("hdr_sky_64x36_s8_b3", build_benchmark_scene(), dict(BENCH_CAMERA, yaw=0.5), 64, 36, 8, 3,
        sky="hdr:32:16")
    rng = np.random.default_rng(2305)
    for i, (s, b) in enumerate([(1, 0), (4, 1), (8, 2), (3, 3), (16, 4), (2, 6)]):
        sky = "grad:12:6" if i % 2 else None
        cam = dict(position=(0.0, 1.5, -4.0), yaw=float(rng.uniform(-0.3, 0.3)),
                   pitch=float(rng.uniform(-0.3, 0.1)), fov=float(rng.uniform(40, 90)))
        add(f"random{i}_64x36_s{s}_b{b}", random_scene(rng, i % 3 != 0, None), cam, 64, 36, s, b, sky=sky,
            radiance=(i < 2))
    add("stress_96x54_s500_b8", stress_scene(), BENCH_CAMERA, 96, 54, 500, 8)
    add("deep_64x36_s4_b31", build_benchmark_scene(), SWEEP_CAMERA, 64, 36, 4, 31, sky="grad:16:8")
    add("tall_36x64_s8_b2", build_benchmark_scene(), BENCH_CAMERA, 36, 64, 8, 2)
    add("empty_8x8_s1_b1", Scene(bodies=[], light=Light((0, 5, 0), 0.5)),
        dict(position=(0.0, 0.0, 0.0), yaw=0.0, pitch=0.0, fov=60.0), 8, 8, 1, 1)
    add("empty_sky_16x8_s3_b2", Scene(bodies=[], light=Light((0, 5, 0), 0.5)),
        dict(position=(0.0, 0.0, 0.0), yaw=1.0, pitch=0.3, fov=90.0), 16, 8, 3, 2, sky="grad:16:8")
    add("one_pixel_1x1_s200_b3", build_benchmark_scene(), BENCH_CAMERA, 1, 1, 200, 3)
    add("ragged_37x23_s7_b1", small_scene(), dict(position=(0.3, 1.0, -3.5), yaw=-0.2, pitch=0.05, fov=75.0),
        37, 23, 7, 1, sky="grad:8:4")
    add("blocked_32x18_s4_b1", blocked_scene(), dict(position=(0.0, 2.0, -6.0), yaw=0.0, pitch=-0.2, fov=70.0),
        32, 18, 4, 1)
    add("c3like_192x108_s200_b3_sky", build_benchmark_scene(), BENCH_CAMERA, 192, 108, 200, 3,
        sky="grad:2048:1024", radiance=True)

    # --- the frame server's wire format (server.py:56-64) of the golden frame ----
    from raytracer.server import encode_frame as ref_encode_frame

    fb = Framebuffer.create(128, 72)
    fb.pixels[:] = arrays["bench_128x72_s200_b3/pixels"]
    arrays["encode/bench_128x72_s200_b3_id7"] = np.frombuffer(ref_encode_frame(7, fb), dtype=np.uint8).copy()

    # --- per-ray fixtures: iterative (reference) + recursive oracle -------------
    rng = np.random.default_rng(303)
    ray_cases = []
    rays = {}
    for si in range(8):
        sky = "grad:12:6" if si % 2 else None
        scene = random_scene(rng, si % 3 != 0, make_sky(sky))
        origins, dirs, iters, recs, limits = [], [], [], [], []
        for limit in (0, 1, 2, 3):
            params = RenderParams(8, limit, 1, 1)
            for _ in range(15):
                o = (rng.uniform(-2, 2), rng.uniform(0.5, 3.0), rng.uniform(-6, -3))
                d = vm.normalize((rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.3), 1.0))
                origins.append(o)
                dirs.append(d)
                limits.append(limit)
                iters.append(R.ray_trace_iterative(Ray(o, d), scene, params))
                recs.append(ref_oracles.ray_trace_recursive(o, d, scene, 8, limit))
        rays[f"scene{si}/origins"] = np.array(origins)
        rays[f"scene{si}/dirs"] = np.array(dirs)
        rays[f"scene{si}/limits"] = np.array(limits, dtype=np.int32)
        rays[f"scene{si}/iterative"] = np.array(iters)
        rays[f"scene{si}/recursive"] = np.array(recs)
        ray_cases.append(dict(name=f"scene{si}", scene=packed(scene), sky=sky, samples=8))

    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump(dict(frames=cases, rays=ray_cases, golden_sha256=GOLDEN_SHA,
                       generator="tests/golden/make_golden.py",
                       reference="/root/reference/pkg (raytracer 0.1.0, numba float64)"), f, indent=1)
        f.write("\n")
    np.savez_compressed(os.path.join(HERE, "frames.npz"), **arrays)
    np.savez_compressed(os.path.join(HERE, "rays.npz"), **rays)


if __name__ == "__main__":
    main()
