"""Host expansion speed of the compressed frame transfer (rt_frame_expand_v1)
by thread count, on a real frame encoded by tests/test_codec.py's numpy
restatement (frames: tools/micro/_data/<key>.bin, raw uint32 rows).

    python tools/codec_expand_bench.py C2 1280 720
"""
import ctypes
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from paper_2305_07450_b200 import _native  # noqa: E402
from test_codec import encode  # noqa: E402

key, w, h = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
f = np.fromfile(os.path.join(ROOT, "tools", "micro", "_data", f"{key}.bin"), dtype=np.uint32).reshape(h, w)
buf, n = encode(f)
print(f"{key}: {4 * n} B over PCIe of {f.nbytes} ({4 * n / f.nbytes:.3f})")
lib = _native.load()
out = np.zeros_like(f)
for th in (1, 2, 4, 8, 12, 16):
    ts = []
    for _ in range(300):
        t = time.perf_counter()
        lib.rt_frame_expand_v1(buf.ctypes.data, w, h, out.ctypes.data, w, th, None)
        ts.append(time.perf_counter() - t)
        g = time.perf_counter()
        while time.perf_counter() - g < 60e-6:
            pass
    assert (out == f).all()
    print(f"  threads {th:2d}: median {1e6 * statistics.median(ts):6.1f} us  p10 {1e6 * np.percentile(ts, 10):6.1f}")
