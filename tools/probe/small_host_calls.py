"""Per-call latency of small host calls: AoS rows and SoA component arrays (numpy),
100 and 10000 rows, normalize3 f64; wall clock per call, median of 200."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402

p = fn.preset("double")
for n in (100, 10000):
    X = np.random.default_rng(0).standard_normal((n, 3))
    comps = [np.ascontiguousarray(X[:, k]) for k in range(3)]
    for name, f in (("aos", lambda: fn.normalize3(p, X)), ("soa", lambda: fn.normalize3(p, *comps))):
        for _ in range(20):
            f()
        ts = []
        for _ in range(200):
            t0 = time.perf_counter()
            f()
            ts.append(time.perf_counter() - t0)
        print(json.dumps({"rows": n, "layout": name, "us_per_call": round(statistics.median(ts) * 1e6, 1)}), flush=True)
