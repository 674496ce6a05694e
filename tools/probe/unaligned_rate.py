"""Device rows whose storage is not 16-byte aligned (x[1:] of a contiguous array) take
the per-row kernel; how fast is that against the bulk-copy kernel on aligned rows?
normalize{2,3,4} f64 and f32 at 2^27 rows, CUDA events, median of 10."""
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
    for dim in (2, 3, 4):
        big = torch.randn((n + 1, dim), dtype=dt, device="cuda")
        f = getattr(fn, f"normalize{dim}")
        r = torch.empty(n, dtype=dt, device="cuda")
        u = torch.empty((n, dim), dtype=dt, device="cuda")
        for name, x in (("aligned", big[:n]), ("offset_1_row", big[1:])):
            t = timed(lambda: f(p, x, out=(r, u)))
            print(json.dumps({"prec": prec, "dim": dim, "rows": n, "case": name,
                              "misaligned_bytes": x.data_ptr() % 16, "ms": round(t * 1e3, 4),
                              "GB_per_s": round(n * (2 * dim + 1) * w / t / 1e9, 1)}), flush=True)
        del big, r, u
        torch.cuda.empty_cache()
