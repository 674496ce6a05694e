"""Throughput of the structure-of-arrays kernel (dev probe): normalize3 / normalize2 f64 and
normalize3 f32 over 2^28 rows of component arrays."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6537.3
for dim, dt, prec in ((3, torch.float64, "double"), (2, torch.float64, "double"), (3, torch.float32, "single")):
    n = 1 << 28
    p = fn.preset(prec)
    comps = [torch.randn(n, dtype=dt, device="cuda") for _ in range(dim)]
    f = getattr(fn, f"normalize{dim}")
    for _ in range(3):
        f(p, *comps)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            f(p, *comps)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 5)
    ms = statistics.median(ts)
    bpr = comps[0].element_size() * (2 * dim + 1)
    print(json.dumps({"kernel": f"normalize{dim} SoA {prec}", "rows": n, "ms": ms, "Gvec_per_s": n / ms / 1e6,
                      "GB_per_s": n * bpr / ms / 1e6, "frac": n * bpr / ms / 1e6 / peak}), flush=True)
    del comps
    torch.cuda.empty_cache()
