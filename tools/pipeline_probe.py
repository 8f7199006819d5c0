"""FramePipeline throughput against depth, with the submit cost alone."""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2305_07450_b200 as rt  # noqa: E402


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "C2"
    cfg = rt.CONFIGS[key]
    scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
    for depth in (1, 2, 3, 4):
        pipe = rt.FramePipeline(depth)
        fbs = [rt.Framebuffer.create(cfg.width, cfg.height) for _ in range(depth)]
        for i in range(10):
            pipe.submit(scene, cam, params, fbs[i % depth])
        pipe.drain()
        n = 200
        sub = 0.0
        t = time.perf_counter()
        for i in range(n):
            s0 = time.perf_counter()
            pipe.submit(scene, cam, params, fbs[i % depth])
            sub += time.perf_counter() - s0
        pipe.drain()
        dt = time.perf_counter() - t
        pipe.close()
        print(f"{key} depth={depth}: {1e6 * dt / n:.1f} us/frame ({n / dt:.0f} fps), submit incl. waits {1e6 * sub / n:.1f} us",
              flush=True)


if __name__ == "__main__":
    main()
