"""Where the end-to-end render_frame time goes (host packing, library call,
device kernels, device-to-host copy)."""

import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


import paper_2305_07450_b200 as rt  # noqa: E402
from paper_2305_07450_b200 import _native  # noqa: E402


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "C2"
    cfg = rt.CONFIGS[key]
    scene, cam, params = cfg.scene(), cfg.camera(), cfg.params()
    fb = rt.Framebuffer.create(cfg.width, cfg.height)
    for _ in range(5):
        rt.render_frame(scene, cam, params, fb)
    ctx = _native.context(1)
    tot, pack, kern = [], [], []
    for _ in range(50):
        t0 = time.perf_counter()
        rt.pack_scene(scene)
        t1 = time.perf_counter()
        rt.render_frame(scene, cam, params, fb)
        t2 = time.perf_counter()
        pack.append(t1 - t0)
        tot.append(t2 - t1)
        kern.append(ctx.last_kernel_ms() * 1e-3)
    med = lambda v: 1e6 * statistics.median(v)  # noqa: E731
    print(f"{key}: render_frame {med(tot):.1f} us | pack_scene {med(pack):.1f} us | kernels {med(kern):.1f} us | "
          f"frame {fb.pixels.nbytes / 1e6:.2f} MB")
    # raw D2H of the same size from pinned memory
    import torch
    d = torch.empty(fb.pixels.size, dtype=torch.int32, device="cuda")
    h = torch.empty(fb.pixels.size, dtype=torch.int32, pin_memory=True)
    for _ in range(3):
        h.copy_(d)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        t = time.perf_counter()
        h.copy_(d)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    print(f"  pinned D2H of {h.numel() * 4 / 1e6:.2f} MB: {med(ts):.1f} us ({h.numel() * 4 / statistics.median(ts) / 1e9:.1f} GB/s)")


if __name__ == "__main__":
    main()
