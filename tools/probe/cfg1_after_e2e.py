"""Does the host pipeline (fn_host_run) running first change a lone config-1 launch?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1606_06508_b200 as fn  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
print("before:", [(o["kernel"], round(o["ms"] * 1e3, 2)) for o in bench.measure_other_configs(dev) if o["config"] == 1], flush=True)
p = fn.preset("double")
small = torch.empty((1000, 3), dtype=torch.float64, pin_memory=True)
small.uniform_(-1, 1)
fn.normalize3(p, small.numpy())
print("after a 1000-row host call:", [(o["kernel"], round(o["ms"] * 1e3, 2)) for o in bench.measure_other_configs(dev) if o["config"] == 1], flush=True)
n = 1 << 27
x = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
x.uniform_(-1, 1)
r = torch.empty(n, dtype=torch.float64, pin_memory=True)
u = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
fn.normalize3(p, x.numpy(), out=(r.numpy(), u.numpy()))
print("after host path:", [(o["kernel"], round(o["ms"] * 1e3, 2)) for o in bench.measure_other_configs(dev) if o["config"] == 1], flush=True)
