"""normalize3(p, X[:, 0], X[:, 1], X[:, 2]) (columns of one record array, run as AoS in place) against separate SoA arrays and the AoS call; 2^27 f64 rows, CUDA events."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402
p = fn.preset("double"); n = 1 << 27
X = torch.randn((n, 3), dtype=torch.float64, device="cuda")
cols = [X[:, k] for k in range(3)]
sep = [c.contiguous() for c in cols]
def timed(f, reps=10):
    for _ in range(3): f()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)
for name, f in (("columns_of_records", lambda: fn.normalize3(p, *cols)), ("separate_arrays_soa", lambda: fn.normalize3(p, *sep)), ("aos", lambda: fn.normalize3(p, X))):
    ms = timed(f); print(json.dumps({"path": name, "rows": n, "ms": round(ms, 4), "G_rows_per_s": round(n / ms / 1e6, 2)}))
