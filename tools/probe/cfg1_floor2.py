"""Where the fixed cost of a lone config-1 launch goes (1e6 x 3 f64 normalize3).

Each case is timed 30 times with CUDA events on the launching stream (median):
  events_only        e0, e1 back to back after the flush: the event floor;
  one_row[_noflush]  a 1-row launch (direct kernel) after / without a flush;
  full[_noflush]     the 1e6-row launch after / without a flush (no flush leaves the
                     previous launch's 56 MB in L2: a diagnostic, not a bench number);
  full_writeflush    flush by writing 512 MB instead of reading it (dirty L2 lines);
  full_after_tiny    flush, then an unrelated tiny torch kernel, then e0 + the launch:
                     separates "first launch after the flush kernel" from the flush.

    python tools/probe/cfg1_floor2.py
"""
import json
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402
from paper_1606_06508_b200 import workloads  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    rows = workloads.CONFIGS[1].rows
    x = torch.empty((rows, 3), dtype=torch.float64, device=dev)
    workloads.generate_device(1, x)
    r = torch.empty((rows,), dtype=torch.float64, device=dev)
    u = torch.empty((rows, 3), dtype=torch.float64, device=dev)
    x1, r1, u1 = x[:1].contiguous(), r[:1], u[:1]
    p = fn.preset("double")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    tiny = torch.zeros(1, device=dev)
    for _ in range(5):
        fn.normalize3(p, x, out=(r, u))
        fn.normalize3(p, x1, out=(r1, u1))
    torch.cuda.synchronize()

    def case(pre, body, reps=30):
        ts = []
        for _ in range(reps):
            pre()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            body()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        return round(statistics.median(ts), 2)

    read_flush = lambda: flush.sum(dtype=torch.int32)  # noqa: E731
    write_flush = lambda: flush.fill_(1)  # noqa: E731
    none = lambda: None  # noqa: E731
    full = lambda: fn.normalize3(p, x, out=(r, u))  # noqa: E731
    one = lambda: fn.normalize3(p, x1, out=(r1, u1))  # noqa: E731

    def flush_then_tiny():
        read_flush()
        tiny.add_(1)

    out = {
        "events_only": case(read_flush, none),
        "one_row": case(read_flush, one),
        "one_row_noflush": case(none, one),
        "full": case(read_flush, full),
        "full_noflush": case(none, full),
        "full_writeflush": case(write_flush, full),
        "full_after_tiny": case(flush_then_tiny, full),
        "unit": "us (median of 30, CUDA events)",
        "ideal_us_at_6544GBps": round(rows * 56 / 6544e9 * 1e6, 2),
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
