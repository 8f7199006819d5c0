"""Pipelined frames/s (FramePipeline, the frame server's loop) under option
sets, interleaved rounds: python tools/pipeline_ab.py C2 --set codec=0 --set codec=1"""
import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_07450_b200 as rt  # noqa: E402
from paper_2305_07450_b200 import _native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="C2")
    ap.add_argument("--frames", type=int, default=200)
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--depth", type=int, default=3)
    ap.add_argument("--set", action="append", default=[])
    a = ap.parse_args()
    cfg = rt.CONFIGS[a.config]
    scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
    cams = [rt.Camera(position=cam.position, yaw=cam.yaw + 1e-4 * i, pitch=cam.pitch, fov=cam.fov) for i in range(2)]
    res = {s: [] for s in a.set}
    for _ in range(a.rounds):
        for spec in a.set:
            _native.set_options(**{k: int(v) for k, v in (kv.split("=") for kv in spec.split(","))})
            pipe = rt.FramePipeline(a.depth)
            fbs = [rt.Framebuffer.create(cfg.width, cfg.height) for _ in range(a.depth)]
            for i in range(10):
                pipe.submit(scene, cams[i % 2], params, fbs[i % a.depth])
            pipe.drain()
            t = time.perf_counter()
            for i in range(a.frames):
                pipe.submit(scene, cams[i % 2], params, fbs[i % a.depth])
            pipe.drain()
            res[spec].append(a.frames / (time.perf_counter() - t))
            pipe.close()
    for spec, v in res.items():
        print(f"{a.config} {spec:36s} median {statistics.median(v):9.1f} frames/s  (min {min(v):.1f}, max {max(v):.1f})",
              flush=True)


if __name__ == "__main__":
    main()
