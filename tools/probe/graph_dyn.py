"""Captured launches under the dynamic tile schedule (dev probe): each workload's kernel is
captured four times into a CUDA graph and the graph replayed; run with
FASTNORM_B200_DYN_CAPTURE=0 (captured launches static) and =1 (own counter per node)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402
from paper_1606_06508_b200 import workloads  # noqa: E402

CASES = [("normalize3", 5, 28, 56), ("norm3", 5, 28, 32), ("normalize2", 2, 26, 40), ("normalize4_sq", 3, 27, 80),
         ("quotient3_robust", 5, 26, 56), ("normalize3", 4, 28, 28), ("normalize3", 1, 20, 56)]
mode = os.environ.get("FASTNORM_B200_DYN_CAPTURE", "1") + "v" + os.environ.get("FASTNORM_B200_DYN_VARIANT", "0")
only = os.environ.get("GRAPH_DYN_ONLY")
if only:
    CASES = [c for c in CASES if c[0] in only.split(",")]
for name, cfg, lg, bpr in CASES:
    c = workloads.CONFIGS[cfg]
    dt = torch.float64 if c.dtype == "float64" else torch.float32
    p = fn.preset("double" if dt == torch.float64 else "single")
    n = 1 << lg
    x = torch.empty((n, c.dim), dtype=dt, device="cuda")
    workloads.generate_device(cfg, x)
    f = getattr(fn, name)
    call = (lambda out=None: f(x, out=out)) if name.startswith("quotient") else (lambda out=None: f(p, x, out=out))
    first = call()
    out = first if torch.is_tensor(first) else tuple(first)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    reps = 4 if lg > 22 else 32
    with torch.cuda.stream(s):
        call(out)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                call(out)
    ts = []
    for _ in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3 / reps)
    t = statistics.median(ts[1:])
    print(json.dumps({"capture_dyn": mode, "kernel": name, "cfg": cfg, "log2_rows": lg, "us_per_launch": round(t * 1e6, 2),
                      "GB_per_s": round(n * bpr / t / 1e9)}), flush=True)
    del x, out, first, g
    torch.cuda.empty_cache()
