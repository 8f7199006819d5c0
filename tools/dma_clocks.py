"""SM clock and throttle reasons while D2H copies run back to back (nvml)."""
import threading
import time

import pynvml
import torch

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
src = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
dst = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
a = torch.randn(8192, 8192, device="cuda")


def sample(tag, fn, secs=1.5):
    stop = [False]
    out = []

    def loop():
        while not stop[0]:
            fn()
            torch.cuda.synchronize()

    t = threading.Thread(target=loop)
    t.start()
    time.sleep(0.3)
    t0 = time.time()
    while time.time() - t0 < secs:
        out.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                    pynvml.nvmlDeviceGetCurrentClocksEventReasons(h), pynvml.nvmlDeviceGetPowerUsage(h) / 1000))
        time.sleep(0.05)
    stop[0] = True
    t.join()
    clocks = sorted(c for c, _, _ in out)
    reasons = sorted({r for _, r, _ in out})
    print(f"{tag:28s} SM MHz median {clocks[len(clocks) // 2]} min {clocks[0]} | reasons {reasons} | power {out[-1][2]:.0f} W")


sample("idle", lambda: time.sleep(0.01))
sample("D2H DMA loop", lambda: dst.copy_(src, non_blocking=True))
sample("H2D DMA loop", lambda: src.copy_(dst, non_blocking=True))
sample("matmul loop", lambda: a @ a)
