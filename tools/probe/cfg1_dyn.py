"""Developer probe (GPU): lone config-1 launch (1e6 3-D f64 rows) with the static and the
dynamic tile schedule, the way bench.py times it (512 MiB read flush, CUDA events on the
launching stream, median), plus the 2^28-row steady state as a no-regression check.
Usage: python tools/probe/cfg1_dyn.py   (spawns one process per FASTNORM_B200_DYN mode)"""

import json
import os
import statistics
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def child():
    sys.path.insert(0, REPO)
    import torch

    import paper_1606_06508_b200 as fn
    from paper_1606_06508_b200 import workloads

    p = fn.preset("double")
    dev = torch.device("cuda:0")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    out = {"mode": os.environ.get("FASTNORM_B200_DYN", "default")}
    for n, reps in ((1_000_000, 400), (1 << 28, 10)):
        x = torch.empty((n, 3), dtype=torch.float64, device=dev)
        workloads.generate_device(1 if n == 1_000_000 else 5, x)
        r = torch.empty(n, dtype=torch.float64, device=dev)
        u = torch.empty_like(x)
        for _ in range(5):
            fn.normalize3(p, x, out=(r, u))
        ts = []
        s = torch.cuda.current_stream()
        for _ in range(reps):
            flush.sum(dtype=torch.int32)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn.normalize3(p, x, out=(r, u))
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        t = statistics.median(ts)
        out[str(n)] = {"us_mean": statistics.fmean(ts), "us_median": t, "us_p10": sorted(ts)[len(ts) // 10], "frac_mean": n * 56 / (statistics.fmean(ts) * 1e-6) / 1e9 / 6544.0}
        del x, r, u
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child()
    else:
        for rep in range(2):
            for mode in ("0", "1", None):
                env = dict(os.environ)
                env.pop("FASTNORM_B200_DYN", None)
                if mode is not None:
                    env["FASTNORM_B200_DYN"] = mode
                r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
                print(r.stdout.strip() or r.stderr[-2000:], flush=True)
