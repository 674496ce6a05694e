"""Host cost of one public device call, fn.normalize3(p, X, out=(r, u)) on 1000 rows:
microseconds per call over 20000 calls, then a cProfile of the same loop."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402

p = fn.preset("double")
X = torch.zeros((1000, 3), dtype=torch.float64, device="cuda")
r = torch.empty(1000, dtype=torch.float64, device="cuda"); u = torch.empty((1000, 3), dtype=torch.float64, device="cuda")
for _ in range(1000): fn.normalize3(p, X, out=(r, u))
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20000): fn.normalize3(p, X, out=(r, u))
t1 = time.perf_counter(); torch.cuda.synchronize()
print("us per call:", (t1 - t0) / 20000 * 1e6)
pr = cProfile.Profile(); pr.enable()
for _ in range(20000): fn.normalize3(p, X, out=(r, u))
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
