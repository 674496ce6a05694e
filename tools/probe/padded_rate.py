"""xyz rows out of xyzw records (fn_run_ld, ldx 4) against gathering them first and
against dense [N, 3] rows: normalize3, f64 and f32, rows in HBM (> L2), CUDA events.

Algorithmic bytes per row: strided 4w in + 4w out (r + unit), dense 3w + 4w, the gather
path 3w + 4w plus the copy (4w read, 3w written... counted as the bytes it moves).

    python tools/probe/padded_rate.py [log2_rows=27]
"""
import json
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)

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


def main():
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 27
    n = 1 << lg
    dev = torch.device("cuda", 0)
    out = []
    for prec, dt in (("double", torch.float64), ("single", torch.float32)):
        w = 8 if dt == torch.float64 else 4
        p = fn.preset(prec)
        rec = torch.randn((n, 4), dtype=dt, device=dev)
        xv = rec[:, :3]
        dense = xv.contiguous()
        r = torch.empty(n, dtype=dt, device=dev)
        u = torch.empty((n, 3), dtype=dt, device=dev)
        t_str = timed(lambda: fn.normalize3(p, xv, out=(r, u)))
        t_gather = timed(lambda: fn.normalize3(p, xv.contiguous(), out=(r, u)))
        t_dense = timed(lambda: fn.normalize3(p, dense, out=(r, u)))
        for name, t, b in (("strided_ldx4", t_str, 8 * w), ("gather_then_dense", t_gather, 7 * w),
                           ("dense", t_dense, 7 * w)):
            out.append({"prec": prec, "rows": n, "path": name, "ms": round(t * 1e3, 4),
                        "G_rows_per_s": round(n / t / 1e9, 2), "algo_B_per_row": b,
                        "GB_per_s": round(n * b / t / 1e9, 1)})
        del rec, xv, dense, r, u
        torch.cuda.empty_cache()
    # host arrays (page-locked records and outputs), end to end over PCIe
    import time

    import numpy as np

    nh = n // 2
    for prec, dt in (("double", np.float64), ("single", np.float32)):
        p = fn.preset(prec)
        rec = fn.host_empty((nh, 4), dtype=dt)
        rec[:] = np.random.default_rng(0).standard_normal((nh, 4))
        xv = rec[:, :3]
        dense = fn.host_empty((nh, 3), dtype=dt)
        dense[:] = xv
        r = fn.host_empty((nh,), dtype=dt)
        u = fn.host_empty((nh, 3), dtype=dt)

        def wall(f, reps=3):
            f()
            ts = []
            for _ in range(reps):
                t0 = time.perf_counter()
                f()
                ts.append(time.perf_counter() - t0)
            return min(ts)

        t_str = wall(lambda: fn.normalize3(p, xv, out=(r, u)))
        t_gather = wall(lambda: fn.normalize3(p, np.ascontiguousarray(xv), out=(r, u)))
        t_dense = wall(lambda: fn.normalize3(p, dense, out=(r, u)))
        for name, t in (("host_strided_ldx4", t_str), ("host_gather_then_dense", t_gather), ("host_dense", t_dense)):
            out.append({"prec": prec, "rows": nh, "path": name, "ms": round(t * 1e3, 3),
                        "G_rows_per_s": round(nh / t / 1e9, 3), "timing": "wall, best of 3, pinned buffers"})
        del rec, xv, dense, r, u
    for o in out:
        print(json.dumps(o), flush=True)


if __name__ == "__main__":
    main()
