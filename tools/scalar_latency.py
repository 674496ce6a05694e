"""Latency of the reference-signature scalar calls through the cuda backend (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1606_06508_b200 as fn  # noqa: E402
from paper_1606_06508_b200 import _backend  # noqa: E402

p = fn.preset("double")
ka = fn.kernel_args(p)
k = _backend.scalar_kernel("normalize3", "double")
for _ in range(50):
    k(*ka, 3.0, 4.0, 12.0)
n = 2000
t0 = time.perf_counter()
for _ in range(n):
    k(*ka, 3.0, 4.0, 12.0)
t1 = time.perf_counter()
print(f"raw registry scalar normalize3_f64: {(t1 - t0) / n * 1e6:.1f} us/call")
t0 = time.perf_counter()
for _ in range(n):
    fn.normalize3(p, 3.0, 4.0, 12.0)
t1 = time.perf_counter()
print(f"public normalize3(p, x1, x2, x3): {(t1 - t0) / n * 1e6:.1f} us/call")
