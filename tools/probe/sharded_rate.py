"""Single-process multi-GPU driver rate (dev tool): normalize3 f64 over config-5 rows held as
device-resident shards (multigpu.DeviceShards, fn_run_sharded), per device list.
Job time = max over shards of the device time of its launch (CUDA events on the shard's
stream); wall = host time of the call (enqueue on every device + synchronise).
python tools/probe/sharded_rate.py [--log2-rows 28] [--reps 10]"""
import argparse
import json
import statistics
import sys
import time

sys.path.insert(0, ".")


def main():
    import torch

    import paper_1606_06508_b200 as fn
    from paper_1606_06508_b200 import multigpu

    ap = argparse.ArgumentParser()
    ap.add_argument("--log2-rows", type=int, default=28)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    rows = 1 << a.log2_rows
    p = fn.preset("double")
    ndev = torch.cuda.device_count()
    lists = [[0], [0, 0], [0, 0, 0, 0]]
    if ndev >= 2:
        lists += [list(range(k)) for k in (2, 4, 8) if k <= ndev]
    for devs in lists:
        x = multigpu.DeviceShards.generate(5, rows, devs)
        r = multigpu.DeviceShards.empty(rows, 0, torch.float64, devs)
        u = multigpu.DeviceShards.empty(rows, 3, torch.float64, devs)
        for _ in range(3):
            multigpu.normalize_sharded(p, x, out=(r, u))
        dev_ms, wall_ms = [], []
        for _ in range(a.reps):
            for d in set(devs):
                torch.cuda.synchronize(d)
            t0 = time.perf_counter()
            res = multigpu.normalize_sharded(p, x, out=(r, u))
            wall_ms.append((time.perf_counter() - t0) * 1e3)
            dev_ms.append(max(res.elapsed_ms))
        td, tw = statistics.median(dev_ms) / 1e3, statistics.median(wall_ms) / 1e3
        print(json.dumps({"devices": devs, "rows": rows, "shard_ms_max": td * 1e3, "wall_ms": tw * 1e3,
                          "G_rows_per_s_device": rows / td / 1e9, "GB_per_s_device": rows * 56 / td / 1e9,
                          "G_rows_per_s_wall": rows / tw / 1e9, "GB_per_s_wall": rows * 56 / tw / 1e9}), flush=True)
        del x, r, u
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
