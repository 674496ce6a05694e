"""Host-side cost of one batched public call on a CUDA tensor (dev probe): wall time per
call for back-to-back calls on a tiny batch (GPU time negligible), with and without
preallocated outputs, and the raw ctypes entry for comparison."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402
from paper_1606_06508_b200 import _cuda_kernels, _lib  # noqa: E402

p = fn.preset("double")
x = torch.randn(4096, 3, dtype=torch.float64, device="cuda")
r = torch.empty(4096, dtype=torch.float64, device="cuda")
u = torch.empty_like(x)
ka = np.array(fn.kernel_args(p))
L = _lib.lib()
s = torch.cuda.current_stream().cuda_stream


def timeit(f, n=3000):
    for _ in range(200):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


print(f"fn.normalize3(p, x)              : {timeit(lambda: fn.normalize3(p, x)):.2f} us/call")
print(f"fn.normalize3(p, x, out=(r, u))  : {timeit(lambda: fn.normalize3(p, x, out=(r, u))):.2f} us/call")
k = _cuda_kernels.batch_kernel("normalize3", "f64")
print(f"batch_kernel(x, ka, out)         : {timeit(lambda: k(x, ka, out=(r, u))):.2f} us/call")
xp, rp, up, kp = x.data_ptr(), r.data_ptr(), u.data_ptr(), ka.ctypes.data
print(f"ctypes fn_run                    : {timeit(lambda: L.fn_run(1, 3, 1, xp, 4096, rp, up, None, kp, s)):.2f} us/call")
