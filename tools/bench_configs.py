"""Per-config measurements of the BASELINE.json workloads (developer tool, 1 GPU).

For each config: generate the rows in HBM, run the config's kernel families through the
public batched API, time every launch with CUDA events on the launching stream (L2
flushed before each timed launch by reading a 512 MiB buffer, so even the 56 MB config-1
batch is read from HBM), and report vectors/s, GB/s and the fraction of the measured
copy peak.  Config 1 additionally reports CUDA-graph replay (launch overhead removed)
and the L2-resident rate (no flush; informational only).

    python tools/bench_configs.py [--reps 10] > profiles/rXX_configs.jsonl
"""
import argparse
import json
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402
from paper_1606_06508_b200 import workloads  # noqa: E402

PEAK = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(REPO, "MEASURED_PEAKS.json")) else 6650.0

PLAN = {
    1: [("normalize3", 56)],
    2: [("normalize2", 40), ("quotient2", 40)],
    3: [("normalize4_sq", 80), ("normalize4", 72), ("normalize4_rotation", 144)],
    4: [("normalize3", 28), ("quotient3", 28)],
    5: [("normalize3", 56), ("norm3", 32), ("quotient3", 56), ("quotient3_fast", 56), ("scale3", 56)],
}


def call(name, p, x):
    if name == "quotient2":
        return fn.quotient2(x)
    if name == "quotient3":
        return fn.quotient3_robust(x)
    if name == "quotient3_fast":
        return fn.quotient3_fast(x)
    if name == "normalize4_rotation":
        return fn.normalize4_rotation(p, x)
    return getattr(fn, name)(p, x)


def timed(fnc, reps, flush):
    times = []
    s = torch.cuda.current_stream()
    for _ in range(reps):
        if flush is not None:
            # read (not write) 512 MiB: evicts the batch from L2 with clean lines, so no
            # write-back of flush data competes with the timed kernel; it also keeps the
            # GPU busy while the host enqueues the timed launch
            flush.sum(dtype=torch.int32)
        else:
            torch.cuda._sleep(400_000)  # ~0.2 ms of GPU work hides the host enqueue latency
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fnc()
        e1.record(s)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    return statistics.median(times)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--configs", default="1,2,3,4,5")
    a = ap.parse_args()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for cfg in [int(c) for c in a.configs.split(",")]:
        c = workloads.CONFIGS[cfg]
        dt = torch.float64 if c.dtype == "float64" else torch.float32
        p = fn.preset("double" if dt == torch.float64 else "single")
        x = torch.empty((c.rows, c.dim), dtype=dt, device="cuda")
        workloads.generate_device(cfg, x)
        for name, bpr in PLAN[cfg]:
            f = (lambda: call(name, p, x))
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            t = timed(f, a.reps, flush)
            gbs = c.rows * bpr / t / 1e9
            line = {"config": cfg, "kernel": name, "rows": c.rows, "dtype": c.dtype, "bytes_per_row": bpr,
                    "ms": t * 1e3, "vectors_per_s": c.rows / t, "GB_per_s": gbs,
                    "frac_of_measured_peak": gbs / PEAK, "l2": "flushed before every launch"}
            if cfg == 1:
                line["l2_resident_ms"] = timed(f, a.reps, None) * 1e3
                # CUDA graph of 20 back-to-back launches with preallocated outputs
                r = torch.empty(c.rows, dtype=dt, device="cuda")
                u = torch.empty((c.rows, c.dim), dtype=dt, device="cuda")
                g = torch.cuda.CUDAGraph()
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(s):
                    fn.normalize3(p, x, out=(r, u))
                    torch.cuda.synchronize()
                    with torch.cuda.graph(g, stream=s):
                        for _ in range(20):
                            fn.normalize3(p, x, out=(r, u))
                torch.cuda.synchronize()
                tg = timed(g.replay, a.reps, None) / 20
                line["graph_replay_ms_per_launch_l2_resident"] = tg * 1e3
            print(json.dumps(line), flush=True)
        del x
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
