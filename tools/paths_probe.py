"""A few small frames through every path and option (FP32 culled with and
without the silhouette form, unculled wavefront, megakernel, FP64, partitions,
the frame pipeline): a quick check that every kernel variant runs."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2305_07450_b200 as rt  # noqa: E402
from paper_2305_07450_b200 import _native  # noqa: E402


def main():
    cam = rt.benchmark_camera()
    scenes = {"bench": rt.build_benchmark_scene(), "stress40": rt.stress_scene(40), "stress300": rt.stress_scene(300)}
    sky = rt.build_benchmark_scene()
    sky.skybox = rt.synthetic_skybox(64, 32)
    scenes["sky"] = sky
    for name, scene in scenes.items():
        for samples, bounces in ((1, 1), (16, 3), (64, 2)):
            params = rt.RenderParams(samples, bounces, 67, 37)
            for prec in ("fp32", "fp64"):
                for opts in (dict(wave=1, cull=1, conic=1), dict(wave=1, cull=1, conic=0), dict(wave=1, cull=0),
                             dict(wave=0, cull=0)):
                    _native.set_options(**opts)
                    fb = rt.Framebuffer.create(67, 37)
                    rad = np.zeros((67 * 37, 3), np.float32 if prec == "fp32" else np.float64)
                    rt.render_frame(scene, cam, params, fb, precision=prec, radiance=rad)
                    if prec == "fp64":
                        break
            _native.set_options(wave=1, cull=1, conic=1)
            rt.render_frame(scene, cam, params, rt.Framebuffer.create(67, 37), workers=3)
    pipe = rt.FramePipeline(2)
    fbs = [rt.Framebuffer.create(67, 37) for _ in range(2)]
    for i in range(4):
        pipe.submit(scenes["bench"], cam, rt.RenderParams(32, 3, 67, 37), fbs[i % 2])
    pipe.close()
    print("sanitize probe done", flush=True)


if __name__ == "__main__":
    main()
