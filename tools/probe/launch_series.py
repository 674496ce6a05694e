"""Per-launch times of one kernel family over a regime batch (dev probe):
python tools/probe/launch_series.py [dim] [log2 rows] [regime] [algo]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402
from paper_1606_06508_b200 import _backend, workloads  # noqa: E402
from paper_1606_06508_b200.scale import kernel_args_array  # noqa: E402

dim = int(sys.argv[1]) if len(sys.argv) > 1 else 2
lg = int(sys.argv[2]) if len(sys.argv) > 2 else 24
regime = sys.argv[3] if len(sys.argv) > 3 else "normal"
algo = sys.argv[4] if len(sys.argv) > 4 else "scaling"
n = 1 << lg
x = torch.empty((n, dim), dtype=torch.float64, device="cuda")
k = _backend.batch_kernel(_backend.scalar_base(algo, dim), "double")
ka = kernel_args_array(fn.preset("double")) if algo == "scaling" else None
for exp in range(3):
    workloads.generate_regime_device(regime, x, seed=exp)
    out = None
    ts = []
    for i in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = k(x, ka, out=out and (out.head, out.body))
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    bpr = 8 * (2 * dim + 1)
    print(f"exp {exp}: " + " ".join(f"{t:.1f}" for t in ts) + f" us  (best {n * bpr / min(ts) / 1e3:.0f} GB/s)", flush=True)
