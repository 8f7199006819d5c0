"""Device-to-host copy of a 720p frame into pinned memory: one copy against the same bytes split over 2-4 streams (concurrent copies are slower)."""
import torch, time, statistics
n = 1280*720
d = torch.empty(n, dtype=torch.int32, device="cuda")
h = torch.empty(n, dtype=torch.int32, pin_memory=True)
ss = [torch.cuda.Stream() for _ in range(4)]
for k in (1, 2, 4):
    ts = []
    for it in range(60):
        torch.cuda.synchronize()
        t = time.perf_counter()
        c = n // k
        for i in range(k):
            with torch.cuda.stream(ss[i]):
                h[i*c:(i+1)*c].copy_(d[i*c:(i+1)*c], non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    m = statistics.median(ts[10:])
    print(k, "streams", f"{m*1e6:.1f} us {n*4/m/1e9:.1f} GB/s")
for mb in (1, 8, 33, 128):
    n2 = mb * 262144
    d2 = torch.empty(n2, dtype=torch.int32, device="cuda"); h2 = torch.empty(n2, dtype=torch.int32, pin_memory=True)
    ts=[]
    for it in range(20):
        torch.cuda.synchronize(); t=time.perf_counter(); h2.copy_(d2, non_blocking=True); torch.cuda.synchronize(); ts.append(time.perf_counter()-t)
    m=statistics.median(ts[5:]); print(mb, "MB", f"{m*1e6:.1f} us {n2*4/m/1e9:.1f} GB/s")
