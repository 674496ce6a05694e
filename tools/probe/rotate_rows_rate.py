"""Throughput of the two-input rotation kernels through the library (dev probe)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import json  # noqa: E402

import torch  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402
from paper_1606_06508_b200 import workloads  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6537.3
n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
p = fn.preset("double")
q = torch.empty((n, 4), dtype=torch.float64, device="cuda")
workloads.generate_device(3, q)
v = torch.empty((n, 3), dtype=torch.float64, device="cuda")
workloads.generate_device(5, v)
R = fn.rotation_unit(fn.normalize4(p, q).unit).reshape(n, 9).contiguous()
out = torch.empty((n, 3), dtype=torch.float64, device="cuda")
cases = {"normalize4_rotate": (lambda: fn.normalize4_rotate(p, q, v, out=out, strict=False), 32 + 24 + 24),
         "apply_rotations": (lambda: fn.apply_rotations(R, v, out=out), 72 + 24 + 24),
         "rotate_vectors (one matrix)": (lambda: fn.rotate_vectors((0.1, 0.2, 0.3, 0.9), v, out=out), 48)}
for name, (f, bpr) in cases.items():
    for _ in range(3):
        f()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            f()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 10)
    ms = statistics.median(ts)
    print(json.dumps({"kernel": name, "rows": n, "bytes_per_row": bpr, "ms": ms,
                      "Gvec_per_s": n / ms / 1e6, "GB_per_s": n * bpr / ms / 1e6,
                      "frac": n * bpr / ms / 1e6 / peak}), flush=True)
