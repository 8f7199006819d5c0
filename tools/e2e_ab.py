"""End-to-end render_frame time (wall clock around each synchronous call, a
new camera every frame, like bench.py's e2e) under several option sets.

    python tools/e2e_ab.py C2 [--frames 300] [--rounds 10] [--set bands=1 --set bands=2,zero_copy=1 ...]

Option sets run in interleaved rounds (frames / rounds each), so host and GPU
drift during the run hits every set alike.
"""
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
    ap.add_argument("--frames", type=int, default=300)
    ap.add_argument("--set", action="append", default=[])
    ap.add_argument("--rounds", type=int, default=10, help="interleaved rounds over the option sets")
    a = ap.parse_args()
    cfg = rt.CONFIGS[a.config]
    scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
    cams = [rt.Camera(position=cam.position, yaw=cam.yaw + 1e-4 * i, pitch=cam.pitch, fov=cam.fov) for i in range(2)]
    fb = rt.Framebuffer.create(cfg.width, cfg.height)
    base = _native.get_options()
    # (with explicit sets there is no "default" run: in interleaved rounds it
    # would inherit whatever option the previous set left on the context)
    specs = a.set if a.set else ["default"]
    times = {spec: [] for spec in specs}
    kernel = {}

    def apply(spec):
        opts = dict(base)
        if spec != "default":
            for kv in spec.split(","):
                k, v = kv.split("=")
                opts[k] = int(v)
        _native.set_options(**opts)

    # interleaved rounds: every option set sees the same host and GPU drift
    per_round = max(1, a.frames // a.rounds)
    for _ in range(a.rounds):
        for spec in specs:
            apply(spec)
            for i in range(5):
                rt.render_frame(scene, cams[i % 2], params, fb)
            for i in range(per_round):
                t = time.perf_counter()
                rt.render_frame(scene, cams[i % 2], params, fb)
                times[spec].append(time.perf_counter() - t)
            kernel[spec] = rt.last_kernel_ms()
    for spec in specs:
        ts = sorted(times[spec])
        print(f"{a.config} {spec:40s} median {1e6 * statistics.median(ts):7.1f} us  mean {1e6 * statistics.mean(ts):7.1f}"
              f"  p10 {1e6 * ts[len(ts) // 10]:7.1f}  p90 {1e6 * ts[9 * len(ts) // 10]:7.1f}  "
              f"kernel {1e3 * kernel[spec]:.1f} us", flush=True)
    _native.set_options(**base)


if __name__ == "__main__":
    main()
