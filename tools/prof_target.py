"""Short, self-contained target for ncu captures (developer tool).

python tools/prof_target.py [--cfg 5] [--log2-rows 26] [--iters 3] [--op normalize]
Generates rows of a BASELINE config in HBM and runs the chosen kernel family `iters`
times through the public batched API (one launch each).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402
from paper_1606_06508_b200 import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=5)
    ap.add_argument("--log2-rows", type=int, default=26)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--op", default="normalize",
                    choices=["normalize", "normalize_sq", "norm", "quotient", "quotient3_fast", "naive", "scale",
                             "normalize4_rotation"])
    ap.add_argument("--padded", action="store_true",
                    help="rows as xyz of xyzw records (3-D configs; fn_run_ld with ldx 4)")
    ap.add_argument("--offset-rows", type=int, default=0,
                    help="start the rows this many rows into the buffer (storage off the 16-byte grid)")
    a = ap.parse_args()
    c = workloads.CONFIGS[a.cfg]
    dt = torch.float64 if c.dtype == "float64" else torch.float32
    n = 1 << a.log2_rows
    x = torch.empty((n, c.dim), dtype=dt, device="cuda")
    workloads.generate_device(a.cfg, x)
    if a.offset_rows:
        big = torch.empty((n + a.offset_rows, c.dim), dtype=dt, device="cuda")
        big[a.offset_rows:] = x
        x = big[a.offset_rows:]
    if a.padded:
        rec = torch.zeros((n, c.dim + 1), dtype=dt, device="cuda")
        rec[:, :c.dim] = x
        x = rec[:, :c.dim]
    p = fn.preset("double" if dt == torch.float64 else "single")
    d = c.dim
    for _ in range(a.iters):
        if a.op == "normalize":
            getattr(fn, f"normalize{d}")(p, x)
        elif a.op == "normalize_sq":
            getattr(fn, f"normalize{d}_sq")(p, x)
        elif a.op == "norm":
            getattr(fn, f"norm{d}")(p, x)
        elif a.op == "scale":
            getattr(fn, f"scale{d}")(p, x)
        elif a.op == "quotient":
            {2: fn.quotient2, 3: fn.quotient3_robust, 4: fn.quotient4}[d](x)
        elif a.op == "normalize4_rotation":
            fn.normalize4_rotation(p, x)
        elif a.op == "quotient3_fast":
            fn.quotient3_fast(x)
        else:
            {2: fn.naive_normalize2, 3: fn.naive_normalize3, 4: fn.naive_normalize4}[d](x)
    torch.cuda.synchronize()
    print("ok", a)


if __name__ == "__main__":
    main()
