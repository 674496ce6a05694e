"""Host (numpy) structure-of-arrays calls -- the reference's scalar signature with one
array per component, normalize3(p, x1, x2, x3) -- against the AoS host path, 2^24 f64
rows, pageable and page-locked inputs; wall clock, best of 3."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402

n = 1 << 24
p = fn.preset("double")
rng = np.random.default_rng(0)
X = rng.standard_normal((n, 3))
comps = [np.ascontiguousarray(X[:, k]) for k in range(3)]
pinned = []
for c in comps:
    h = fn.host_empty((n,))
    h[:] = c
    pinned.append(h)


def wall(f, reps=3):
    f()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return min(ts)


for name, f in (("soa_pageable", lambda: fn.normalize3(p, *comps)),
                ("soa_pinned", lambda: fn.normalize3(p, *pinned)),
                ("aos_pageable", lambda: fn.normalize3(p, X))):
    t = wall(f)
    print(json.dumps({"path": name, "rows": n, "ms": round(t * 1e3, 2), "G_rows_per_s": round(n / t / 1e9, 3)}),
          flush=True)
