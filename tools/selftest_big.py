"""Long division self-test (dev tool): SEEDS x 2^32 operand pairs per precision."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1606_06508_b200 import _lib  # noqa: E402

seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 8
out = torch.zeros(3, dtype=torch.int64, device="cuda")
for name, dt in (("f32", _lib.F32), ("f64", _lib.F64)):
    bad = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for seed in range(100, 100 + seeds):
        out.zero_()
        _lib.check(_lib.lib().fn_selftest_div(dt, seed, 1 << 32, out.data_ptr(),
                                              torch.cuda.current_stream().cuda_stream), "selftest")
        b, a, bb = out.tolist()
        if b:
            print(name, "seed", seed, "mismatches", b, hex(a & (2**64 - 1)), hex(bb & (2**64 - 1)), flush=True)
        bad += b
    e1.record()
    e1.synchronize()
    print(f"{name}: {seeds} x 2^32 pairs, mismatches {bad}, {e0.elapsed_time(e1) / 1e3:.1f} s", flush=True)
