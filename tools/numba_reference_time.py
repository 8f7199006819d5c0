"""Time the unmodified reference (numba `render_frame` from the reference
package pip-installed into baseline/_ref, tools/install_reference.sh) on the
host cores: whole frames of a configuration after the JIT warm-up, workers =
all host CPUs.  Prints one JSON object.  bench.py runs it as a subprocess
(its numba threads stay out of the benchmark process).

    python tools/numba_reference_time.py C2 [frames]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
t0 = time.perf_counter()
from raytracer import renderer, sceneio  # noqa: E402
from raytracer.scene import Framebuffer, RenderParams  # noqa: E402

# the benchmark scene's configurations without a skybox (BASELINE.json configs[0, 1], the paper's rows)
SIZES = {"C1": (640, 360, 1, 0), "C2": (1280, 720, 200, 3), "P720": (1280, 720, 1, 1), "P1080": (1920, 1080, 1, 1),
         "P4K": (3840, 2160, 1, 1)}


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "C2"
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    w, h, s, b = SIZES[key]
    scene, cam = sceneio.build_benchmark_scene(), sceneio.benchmark_camera()
    workers = os.cpu_count()
    small = Framebuffer.create(16, 9)
    renderer.render_frame(scene, cam, RenderParams(s, b, 16, 9), small, workers=workers)  # numba JIT
    t1 = time.perf_counter()
    fb = Framebuffer.create(w, h)
    params = RenderParams(s, b, w, h)
    renderer.render_frame(scene, cam, params, fb, workers=workers)  # warm at full size
    t = time.perf_counter()
    for _ in range(frames):
        renderer.render_frame(scene, cam, params, fb, workers=workers)
    dt = (time.perf_counter() - t) / frames
    print(json.dumps({"config": key, "value": 1.0 / dt, "unit": "frames/s", "frames": frames, "workers": workers,
                      "jit_s": t1 - t0, "kind": "reference",
                      "sample": f"{frames} whole frames of {key} ({w}x{h} s{s} b{b}) through the unmodified "
                                f"reference raytracer.renderer.render_frame (numba, baseline/_ref), "
                                f"workers={workers}, after the JIT warm-up"}))


if __name__ == "__main__":
    main()
