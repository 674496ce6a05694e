"""Short ncu target: normalize_many over 32 config-1 batches (8 buffer sets), two calls."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402
from paper_1606_06508_b200 import workloads  # noqa: E402

p = fn.preset("double")
rows = 1_000_000
xs = []
for s in range(8):
    x = torch.empty((rows, 3), dtype=torch.float64, device="cuda")
    workloads.generate_device(1, x, row0=s * rows)
    xs.append(x)
outs = [(torch.empty(rows, dtype=torch.float64, device="cuda"), torch.empty_like(x)) for x in xs]
batches = [xs[i % 8] for i in range(32)]
bouts = [outs[i % 8] for i in range(32)]
for _ in range(2):
    fn.normalize_many(p, batches, out=bouts)
torch.cuda.synchronize()
print("ok")
