"""The measured inputs: the paper's benchmark scene and camera, the synthetic
skybox and stress scene of BASELINE.md §3, and the configurations C1-C5.

`build_benchmark_scene` / `benchmark_camera` restate
/root/reference/pkg/src/raytracer/sceneio.py:314-333 (the constants are
pinned by the reference's golden hash, pkg/tests/test_acceptance.py:31).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .model import Body, Camera, Light, RenderParams, Scene, Skybox


def build_benchmark_scene() -> Scene:
    """One light, five spheres (reflectivities 96/32/128/64/0), one plane."""
    spheres = [
        ((-2.4, 1.0, 2.8), 1.0, (0.85, 0.10, 0.10), 96.0),
        ((0.0, 0.8, 1.6), 0.8, (0.10, 0.55, 0.12), 32.0),
        ((2.3, 1.2, 3.2), 1.2, (0.12, 0.30, 0.85), 128.0),
        ((1.1, 0.5, 0.4), 0.5, (0.90, 0.75, 0.12), 64.0),
        ((-0.9, 0.4, 0.0), 0.4, (0.90, 0.90, 0.90), 0.0),
    ]
    bodies = [Body.sphere(*s) for s in spheres] + [Body.plane(0.0, (0.42, 0.45, 0.50), 16.0)]
    return Scene(
        bodies=bodies,
        light=Light(position=(-4.0, 7.0, -2.0), radius=0.6, color=(1.0, 1.0, 1.0)),
        ambient=0.15,
        max_reflectivity=128.0,
    )


def benchmark_camera() -> Camera:
    return Camera(position=(0.0, 1.4, -4.5), yaw=0.0, pitch=-0.08, fov=60.0)


def gradient_texels(width: int, height: int, hdr: bool = False) -> np.ndarray:
    """texel[y, x] = (x/W, y/H, 0.25) in float32 — the reference's test
    fixture formula (pkg/tests/test_renderer.py:23-28); `hdr` triples the top
    third so the [0,1] clamp of renderer.py:74 is exercised."""
    xs = np.arange(width, dtype=np.float64) / width
    ys = np.arange(height, dtype=np.float64) / height
    t = np.empty((height, width, 3), dtype=np.float32)
    t[:, :, 0] = xs[None, :]
    t[:, :, 1] = ys[:, None]
    t[:, :, 2] = 0.25
    if hdr:
        t[: height // 3] *= np.float32(3.0)
    return t


def synthetic_skybox(width: int = 2048, height: int = 1024) -> Skybox:
    """C3/C4 skybox: the gradient fixture at 2048x1024 (25.2 MB float32)."""
    return Skybox(width, height, gradient_texels(width, height))


def stress_scene(count: int = 256, seed: int = 230507450) -> Scene:
    """C5: `count` random spheres, then the benchmark plane
    last, with the benchmark light."""
    rng = np.random.default_rng(seed)
    bench = build_benchmark_scene()
    bodies = []
    for _ in range(count):
        r = rng.uniform(0.2, 0.6)
        centre = (rng.uniform(-10, 10), r + rng.uniform(0, 2), rng.uniform(0.5, 25))
        colour = tuple(rng.uniform(0.05, 0.95, size=3))
        bodies.append(Body.sphere(centre, r, colour, rng.uniform(0, 128)))
    bodies.append(bench.bodies[-1])
    return Scene(bodies=bodies, light=bench.light, ambient=bench.ambient,
                 max_reflectivity=bench.max_reflectivity)


@dataclass(frozen=True)
class Config:
    name: str
    width: int
    height: int
    samples: int
    bounces: int
    sky: bool = False
    stress: bool = False
    spheres: int = 256  # stress scenes: sphere count

    def params(self) -> RenderParams:
        return RenderParams(self.samples, self.bounces, self.width, self.height)

    def scene(self, skybox: Optional[Skybox] = None) -> Scene:
        scene = stress_scene(self.spheres) if self.stress else build_benchmark_scene()
        if self.sky:
            scene.skybox = skybox if skybox is not None else synthetic_skybox()
        return scene

    def camera(self) -> Camera:
        return benchmark_camera()


# BASELINE.json "configs" (concretised in BASELINE.md §3 / SURVEY.md §8d)
CONFIGS = {
    "C1": Config("C1 640x360 s1 b0", 640, 360, 1, 0),
    "C2": Config("C2 1280x720 s200 b3", 1280, 720, 200, 3),
    "C3": Config("C3 1920x1080 s200 b3 sky", 1920, 1080, 200, 3, sky=True),
    "C4": Config("C4 3840x2160 s200 b3 sky", 3840, 2160, 200, 3, sky=True),
    "C5": Config("C5 3840x2160 s500 b8 stress256", 3840, 2160, 500, 8, stress=True),
    # "also report 512"
    "C5_512": Config("C5 3840x2160 s500 b8 stress512", 3840, 2160, 500, 8, stress=True, spheres=512),
    # the paper's measurement condition: 1 sample, 1 bounce
    "P720": Config("paper 1280x720 s1 b1", 1280, 720, 1, 1),
    "P1080": Config("paper 1920x1080 s1 b1", 1920, 1080, 1, 1),
    "P4K": Config("paper 3840x2160 s1 b1", 3840, 2160, 1, 1),
}

# Published fps of the paper's engine (RTX 2060, s1 b1)
PAPER_FPS = {"P720": 234.0, "P1080": 152.0, "P4K": 45.0}
