"""Config 1 (1e6 x 3 f64 normalize3) launch-shape probe: one lone launch after an L2
flush, and the stream-of-batches graph rate (bench._batch_stream_rate).  Launch shape
from the environment (FASTNORM_B200_CTAS_PER_SM, FASTNORM_B200_PATH=direct).

    FASTNORM_B200_CTAS_PER_SM=4 python tools/cfg1_probe.py
"""
import json
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1606_06508_b200 as fn  # noqa: E402
from paper_1606_06508_b200 import workloads  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    peak, _ = bench._peaks()
    c = workloads.CONFIGS[1]
    x = torch.empty((c.rows, 3), dtype=torch.float64, device=dev)
    workloads.generate_device(1, x)
    p = fn.preset("double")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        fn.normalize3(p, x)
    times = []
    for _ in range(30):
        flush.sum(dtype=torch.int32)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn.normalize3(p, x)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    t = statistics.median(times)
    # the same harness around a 1-row launch: the launch + event floor of a lone launch
    x1 = x[:1].contiguous()
    floor = []
    for _ in range(30):
        flush.sum(dtype=torch.int32)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn.normalize3(p, x1)
        e1.record()
        torch.cuda.synchronize()
        floor.append(e0.elapsed_time(e1) / 1e3)
    t_floor = statistics.median(floor)
    sob = bench._batch_stream_rate(fn, p, x, 56, peak, 10)
    print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("FASTNORM_B200")},
                      "lone_ms": t * 1e3, "lone_frac": c.rows * 56 / t / 1e9 / peak,
                      "one_row_launch_ms": t_floor * 1e3,
                      "lone_minus_floor_frac": c.rows * 56 / (t - t_floor) / 1e9 / peak,
                      "stream_ms": sob["ms_per_launch"], "stream_frac": sob["frac"],
                      "eager_ms": sob["eager_public_api"]["ms_per_launch"],
                      "eager_frac": sob["eager_public_api"]["frac"]}), flush=True)


if __name__ == "__main__":
    main()
