"""Latency of the host-array path for small batches (dev probe)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402

p = fn.preset("double")
for n in (1, 16, 256, 4096, 65536, 1 << 20):
    x = np.random.default_rng(0).standard_normal((n, 3))
    r, u = np.empty(n), np.empty((n, 3))
    for _ in range(20):
        fn.normalize3(p, x, out=(r, u))
    reps = 2000 if n <= 4096 else 200
    t0 = time.perf_counter()
    for _ in range(reps):
        fn.normalize3(p, x, out=(r, u))
    dt = (time.perf_counter() - t0) / reps
    print(f"n={n:8d}: {dt * 1e6:8.1f} us/call  {n / dt / 1e6:9.2f} Mvec/s", flush=True)

# raw ABI for the small path (no Python layers)
from paper_1606_06508_b200 import _lib  # noqa: E402
L = _lib.lib()
ka = np.array(fn.kernel_args(p))
for n in (16, 256, 4096):
    x = np.random.default_rng(0).standard_normal((n, 3))
    r, u = np.empty(n), np.empty((n, 3))
    args = (1, 3, 1, x.ctypes.data, n, r.ctypes.data, u.ctypes.data, None, ka.ctypes.data)
    for _ in range(20):
        L.fn_host_run(*args)
    t0 = time.perf_counter()
    for _ in range(2000):
        L.fn_host_run(*args)
    print(f"raw fn_host_run n={n}: {(time.perf_counter() - t0) / 2000 * 1e6:.1f} us/call", flush=True)
