"""Scene, camera and frame containers of the render call, plus SoA packing.

Mirrors the public types the reference's `render_frame` consumes —
`Body`/`BodyKind`/`Ray` (/root/reference/pkg/src/raytracer/geometry.py:27-73),
`Light` (shading.py:32-42), `Camera` (camera.py:23-33), `Skybox`/`Scene`/
`RenderParams`/`Framebuffer` (scene.py:21-94) — with the same field names,
defaults and `ValueError` validation, so code written against the reference
constructs them unchanged.  The renderer duck-types its inputs: the
reference's own dataclass instances are accepted as well.
"""

from __future__ import annotations

import array
import enum
import math
from dataclasses import dataclass
from typing import List, Optional, Tuple

import numpy as np

Vec3 = Tuple[float, float, float]

# Module constants of the reference, one place (SURVEY.md §5 "Config / flags").
MISS = math.inf                          # geometry.py:22
GRAZE_EPS = 1e-7                         # geometry.py:24
SHADOW_EPS = 1e-3                        # shading.py:27
REFLECT_EPS = 1e-3                       # renderer.py:33
MAX_BOUNCE_LIMIT = 31                    # renderer.py:36
DEFAULT_AMBIENT = 0.15                   # shading.py:23
DEFAULT_MAX_REFLECTIVITY = 128.0         # scene.py:18
GOLDEN_ANGLE = math.pi * (3.0 - math.sqrt(5.0))  # shading.py:29
PITCH_LIMIT = math.pi / 2 - 1e-3         # camera.py:20


def _norm(v: Vec3) -> float:
    return math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])


class BodyKind(enum.IntEnum):
    SPHERE = 0
    HORIZONTAL_PLANE = 1


@dataclass
class Body:
    """Sphere (center, radius) or horizontal plane at height position.y."""

    kind: BodyKind
    position: Vec3
    size: float
    color: Vec3
    reflectivity: float = 0.0

    def __post_init__(self):
        if self.kind == BodyKind.SPHERE and not self.size > 0:
            raise ValueError(f"sphere radius must be positive, got {self.size}")
        if any(not (0.0 <= c <= 1.0) for c in self.color):
            raise ValueError(f"color components must be in [0, 1], got {self.color}")
        if self.reflectivity < 0:
            raise ValueError("reflectivity must be non-negative")

    @classmethod
    def sphere(cls, position, radius, color, reflectivity=0.0) -> "Body":
        return cls(BodyKind.SPHERE, position, radius, color, reflectivity)

    @classmethod
    def plane(cls, height, color, reflectivity=0.0) -> "Body":
        return cls(BodyKind.HORIZONTAL_PLANE, (0.0, height, 0.0), 1.0, color, reflectivity)

    @property
    def height(self) -> float:
        return self.position[1]


@dataclass
class Ray:
    origin: Vec3
    direction: Vec3  # unit length (±1e-5)

    def __post_init__(self):
        if abs(_norm(self.direction) - 1.0) > 1e-5:
            raise ValueError(f"ray direction must be unit length, got {self.direction}")

    def at(self, t: float) -> Vec3:
        o, d = self.origin, self.direction
        return (o[0] + d[0] * t, o[1] + d[1] * t, o[2] + d[2] * t)


@dataclass
class Light:
    """Spherical emitter; soft shadows sample a disc of radius 2*radius."""

    position: Vec3
    radius: float
    color: Vec3 = (1.0, 1.0, 1.0)

    def __post_init__(self):
        if not self.radius > 0:
            raise ValueError("light radius must be positive")


@dataclass
class Camera:
    position: Vec3 = (0.0, 0.0, 0.0)
    yaw: float = 0.0
    pitch: float = 0.0
    fov: float = 60.0  # degrees, open interval (0, 180)

    def __post_init__(self):
        if not (0.0 < self.fov < 180.0):
            raise ValueError(f"fov must be in (0, 180) degrees, got {self.fov}")
        self.pitch = max(-PITCH_LIMIT, min(self.pitch, PITCH_LIMIT))


@dataclass
class Skybox:
    """Equirectangular panorama, texels (height, width, 3) float32, HDR allowed."""

    width: int
    height: int
    texels: np.ndarray

    def __post_init__(self):
        if self.texels.shape != (self.height, self.width, 3):
            raise ValueError(
                f"texel array shape {self.texels.shape} does not match {self.height}x{self.width}x3"
            )
        self.texels = np.ascontiguousarray(self.texels, dtype=np.float32)


@dataclass
class Scene:
    bodies: List[Body]
    light: Light
    skybox: Optional[Skybox] = None
    ambient: float = DEFAULT_AMBIENT
    max_reflectivity: float = DEFAULT_MAX_REFLECTIVITY

    def __post_init__(self):
        if not (0.0 <= self.ambient <= 1.0):
            raise ValueError("ambient strength must be in [0, 1]")
        if not self.max_reflectivity > 0:
            raise ValueError("max reflectivity must be positive")
        for i, b in enumerate(self.bodies):
            if b.reflectivity > self.max_reflectivity:
                raise ValueError(
                    f"body {i} reflectivity {b.reflectivity} exceeds max {self.max_reflectivity}"
                )


@dataclass
class RenderParams:
    shadow_samples: int
    bounce_limit: int
    width: int
    height: int

    def __post_init__(self):
        if self.shadow_samples < 1:
            raise ValueError("shadow sample count must be >= 1")
        if self.bounce_limit < 0:
            raise ValueError("bounce limit must be >= 0")
        if self.width < 1 or self.height < 1:
            raise ValueError("frame dimensions must be positive")


@dataclass
class Framebuffer:
    """Row-major uint32 0xAARRGGBB pixels, pixel (x, y) at x + y * width."""

    width: int
    height: int
    pixels: np.ndarray

    @classmethod
    def create(cls, width: int, height: int) -> "Framebuffer":
        return cls(width, height, np.zeros(width * height, dtype=np.uint32))

    def __post_init__(self):
        if self.pixels.shape != (self.width * self.height,):
            raise ValueError("pixel buffer length must equal width * height")
        if self.pixels.dtype != np.uint32:
            raise ValueError("pixel buffer must be uint32")

    def tobytes(self) -> bytes:
        return self.pixels.tobytes()


# --- structure-of-arrays packing (the C-ABI scene arguments) ----------------

_NO_SKY = np.zeros((1, 1, 3), dtype=np.float32)


@dataclass
class PackedScene:
    """The reference's kernel-side scene layout (geometry.py:162-176,
    scene.py:100-104, renderer.py:282-300), contiguous and C-ABI ready."""

    kinds: np.ndarray        # int32[n]
    positions: np.ndarray    # float64[n, 3]
    sizes: np.ndarray        # float64[n]
    colors: np.ndarray       # float64[n, 3]
    refls: np.ndarray        # float64[n]
    light_pos: np.ndarray    # float64[3]
    light_radius: float
    light_color: np.ndarray  # float64[3]
    ambient: float
    max_refl: float
    sky: np.ndarray          # float32[H, W, 3] (1x1 zero placeholder when absent)
    sky_w: int
    sky_h: int
    has_sky: bool

    @property
    def n_bodies(self) -> int:
        return int(self.kinds.shape[0])


def _address(a: np.ndarray) -> int:
    return a.__array_interface__["data"][0]


_NO_SKY_ADDR = _address(_NO_SKY)
_sky_addr = {}  # id(texels) -> (texels, address): skyboxes are re-packed every frame


def _pack_core(scene):
    """The float64 block (positions | sizes | colors | refls | light position |
    light colour), the int32 kinds and the sky, as the C ABI takes them
    (array.array buffers: their addresses cost no numpy round trip)."""
    bodies = scene.bodies
    n = len(bodies)
    light = scene.light
    lp, lc = light.position, light.color
    flat = [b.position[i] for b in bodies for i in (0, 1, 2)]
    flat += [b.size for b in bodies]
    flat += [b.color[i] for b in bodies for i in (0, 1, 2)]
    flat += [b.reflectivity for b in bodies]
    flat += (lp[0], lp[1], lp[2], lc[0], lc[1], lc[2])
    try:
        buf = array.array("d", flat)
    except TypeError:
        buf = array.array("d", [float(v) for v in flat])
    if len(buf) != 8 * n + 6:
        raise ValueError("body positions and colours must be 3-vectors of numbers")
    kinds = array.array("i", [int(b.kind) for b in bodies])
    sky = getattr(scene, "skybox", None)
    if sky is None:
        texels, sw, sh, has, sky_addr = _NO_SKY, 1, 1, False, _NO_SKY_ADDR
    else:
        texels = np.ascontiguousarray(sky.texels, dtype=np.float32)
        sw, sh, has = int(sky.width), int(sky.height), True
        hit = _sky_addr.get(id(texels))
        if hit is not None and hit[0] is texels:
            sky_addr = hit[1]
        else:
            if len(_sky_addr) > 16:
                _sky_addr.clear()
            sky_addr = _address(texels)
            _sky_addr[id(texels)] = (texels, sky_addr)
    base = buf.buffer_info()[0]
    radius, ambient, max_refl = float(light.radius), float(scene.ambient), float(scene.max_reflectivity)
    # C-ABI scene arguments of rt_render_v1 / rt_render_async_v1 / rt_trace_rays_v1 (b200rt.h)
    argv = (n, kinds.buffer_info()[0] if n else 0, base, base + 24 * n, base + 32 * n, base + 56 * n,
            base + 64 * n, radius, base + 64 * n + 24, ambient, max_refl, sky_addr, sw, sh, int(has))
    return buf, kinds, texels, argv


def scene_argv(scene):
    """(C-ABI scene arguments, the arrays they point into) — render_frame's
    per-frame packing without the PackedScene views."""
    buf, kinds, texels, argv = _pack_core(scene)
    return argv, (buf, kinds, texels)


def pack_scene(scene) -> PackedScene:
    """Pack any object with the reference Scene's attributes (duck-typed).

    The float64 columns are views of ONE buffer (positions | sizes | colors |
    refls | light position | light colour) so the C-ABI pointers come from a
    single address lookup: the reference re-packs the scene every frame
    (renderer.py:331), and so does render_frame here."""
    buf_a, kinds_a, texels, argv = _pack_core(scene)
    buf = np.frombuffer(buf_a, dtype=np.float64)
    kinds = np.frombuffer(kinds_a, dtype=np.int32) if len(kinds_a) else np.zeros(0, dtype=np.int32)
    n = argv[0]
    ps = PackedScene(
        kinds=kinds,
        positions=buf[0:3 * n].reshape(n, 3),
        sizes=buf[3 * n:4 * n],
        colors=buf[4 * n:7 * n].reshape(n, 3),
        refls=buf[7 * n:8 * n],
        light_pos=buf[8 * n:8 * n + 3],
        light_radius=argv[7],
        light_color=buf[8 * n + 3:8 * n + 6],
        ambient=argv[9],
        max_refl=argv[10],
        sky=texels,
        sky_w=argv[12],
        sky_h=argv[13],
        has_sky=bool(argv[14]),
    )
    ps.argv = (argv[0], _address(kinds)) + argv[2:] if argv[0] else argv
    ps._keep = (buf_a, kinds_a)
    return ps


def camera_viewport_distance(fov_degrees: float) -> float:
    """1 / tan(fov / 2) with Python's libm, as the reference (camera.py:64-67)."""
    return 1.0 / math.tan(math.radians(fov_degrees) / 2.0)
