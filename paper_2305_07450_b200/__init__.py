"""B200-native frame render of arXiv 2305.07450's ray tracer.

A drop-in for the reference's `raytracer.renderer.render_frame`
(/root/reference/pkg/src/raytracer/renderer.py:316-349): the same Python API
over a C ABI (include/b200rt.h, libb200rt.so) whose kernels are hand-written
CUDA for sm_100a.  There is no CPU path.
"""

from .model import (
    DEFAULT_AMBIENT,
    DEFAULT_MAX_REFLECTIVITY,
    GOLDEN_ANGLE,
    GRAZE_EPS,
    MAX_BOUNCE_LIMIT,
    MISS,
    PITCH_LIMIT,
    REFLECT_EPS,
    SHADOW_EPS,
    Body,
    BodyKind,
    Camera,
    Framebuffer,
    Light,
    PackedScene,
    Ray,
    RenderParams,
    Scene,
    Skybox,
    camera_viewport_distance,
    pack_scene,
)
from .renderer import (
    FramePipeline,
    default_precision,
    last_kernel_ms,
    pack_color,
    ray_trace_iterative,
    render_frame,
    skybox_sample,
    trace_rays,
)
from .workloads import CONFIGS, benchmark_camera, build_benchmark_scene, stress_scene, synthetic_skybox
from .integration import install, uninstall

__version__ = "0.1.0"
