"""A stream of config-1-sized batches (1e6 x 3 f64 rows each, 8 buffer sets cycled,
448 MB > L2): 32 separate normalize3 launches captured in a CUDA graph (bench.py's
stream_of_batches) against normalize_many over the same 32 batches (fn_run_many: one
launch per 48 batches).  CUDA events, median of 10."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402
from paper_1606_06508_b200 import workloads  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6544.0
rows, sets, per_set = 1_000_000, 8, 4
p = fn.preset("double")
bufs = []
for s in range(sets):
    x = torch.empty((rows, 3), dtype=torch.float64, device="cuda")
    workloads.generate_device(1, x, row0=s * rows)
    bufs.append((x, torch.empty(rows, dtype=torch.float64, device="cuda"),
                 torch.empty((rows, 3), dtype=torch.float64, device="cuda")))
order = [bufs[i % sets] for i in range(sets * per_set)]


def timed(f, reps=10):
    for _ in range(3):
        f()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return statistics.median(ts)


def separate():
    for x, r, u in order:
        fn.normalize3(p, x, out=(r, u))


g = torch.cuda.CUDAGraph()
separate()
torch.cuda.synchronize()
with torch.cuda.graph(g):
    separate()
xs = [b[0] for b in order]
outs = [(b[1], b[2]) for b in order]
gm = torch.cuda.CUDAGraph()
fn.normalize_many(p, xs, out=outs)
torch.cuda.synchronize()
with torch.cuda.graph(gm):
    fn.normalize_many(p, xs, out=outs)
for name, f in (("graph_of_32_launches", g.replay), ("eager_32_launches", separate),
                ("normalize_many_32_eager", lambda: fn.normalize_many(p, xs, out=outs)),
                ("normalize_many_32_graph", gm.replay)):
    t = timed(f)
    n = rows * len(order)
    print(json.dumps({"path": name, "batches": len(order), "rows_per_batch": rows,
                      "us_per_batch": round(t / len(order) * 1e6, 2), "G_rows_per_s": round(n / t / 1e9, 1),
                      "frac": round(n * 56 / t / 1e9 / peak, 3)}), flush=True)
