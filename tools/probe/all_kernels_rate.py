"""Every kernel family x dimension x precision on one build (dev probe): back-to-back launches
through the C ABI's generic entry (batch.run), CUDA events, GB/s of algorithmic traffic and the
fraction of the measured copy peak.  Workload: the reference harness's "normal" regime (all
magnitudes inside the band) and "mixed" (the full exponent range), 2^26 rows by default.
python tools/probe/all_kernels_rate.py [--log2-rows 26] [--reps 10]"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402
from paper_1606_06508_b200 import _lib, batch, workloads  # noqa: E402
from paper_1606_06508_b200.scale import kernel_args_array  # noqa: E402

OPS = [("scale", _lib.OP_SCALE, True), ("normalize", _lib.OP_NORMALIZE, True), ("norm", _lib.OP_NORM, True),
       ("normalize_sq", _lib.OP_NORMALIZE_SQ, True), ("naive", _lib.OP_NAIVE, False),
       ("quotient", _lib.OP_QUOTIENT, False), ("quotient3_fast", _lib.OP_QUOTIENT3_FAST, False)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2-rows", type=int, default=26)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--regimes", default="normal,mixed")
    ap.add_argument("--precs", default="double,single")
    ap.add_argument("--dims", default="2,3,4")
    ap.add_argument("--kernels", default="")
    a = ap.parse_args()
    n = 1 << a.log2_rows
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6458.0
    for regime in a.regimes.split(","):
        for dt, prec in ((torch.float64, "double"), (torch.float32, "single")):
            if prec not in a.precs.split(","):
                continue
            ka = kernel_args_array(fn.preset(prec))
            for dim in (int(d) for d in a.dims.split(",")):
                x = torch.empty((n, dim), dtype=dt, device="cuda")
                workloads.generate_regime_device(regime, x)
                for name, op, needs_ka in OPS:
                    if op == _lib.OP_QUOTIENT3_FAST and dim != 3:
                        continue
                    if a.kernels and name not in a.kernels.split(","):
                        continue
                    k = ka if needs_ka else None
                    first = batch.run(op, dim, x, k)
                    out = tuple(t for t in first if t is not None)
                    for _ in range(3):
                        batch.run(op, dim, x, k, out=out)
                    ts = []
                    for _ in range(3):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        for _ in range(a.reps):
                            batch.run(op, dim, x, k, out=out)
                        e1.record()
                        torch.cuda.synchronize()
                        ts.append(e0.elapsed_time(e1) / 1e3 / a.reps)
                    t = statistics.median(ts)
                    w = sum(int(o.numel() // n) for o in out) + dim
                    bpr = w * x.element_size()
                    print(json.dumps({"regime": regime, "prec": prec, "dim": dim, "kernel": name, "rows": n,
                                      "bytes_per_row": bpr, "ms": round(t * 1e3, 4), "GB_per_s": round(n * bpr / t / 1e9),
                                      "frac": round(n * bpr / t / 1e9 / peak, 3)}), flush=True)
                    del first, out
                del x
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
