"""SoA calls whose component arrays are off the 16-byte grid (a[1:]-style views) against
aligned arrays: normalize3 f64 / f32 at 2^27 rows, CUDA events, median of 10."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402


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


n = 1 << 27
for prec, dt in (("double", torch.float64), ("single", torch.float32)):
    p = fn.preset(prec)
    w = 8 if dt == torch.float64 else 4
    aligned = [torch.randn(n, dtype=dt, device="cuda") for _ in range(3)]
    shifted = []
    for k in range(3):
        buf = torch.randn(n + 1, dtype=dt, device="cuda")
        shifted.append(buf[1:] if k != 1 else buf[:n])  # two arrays one element off the grid
    for name, comps in (("aligned", aligned), ("misaligned", shifted)):
        t = timed(lambda: fn.normalize3(p, *comps))
        print(json.dumps({"prec": prec, "rows": n, "case": name, "ms": round(t * 1e3, 4),
                          "GB_per_s": round(n * 7 * w / t / 1e9, 1)}), flush=True)
    del aligned, shifted
    torch.cuda.empty_cache()
