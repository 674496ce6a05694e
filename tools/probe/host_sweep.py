"""Developer probe (GPU): host-path staging settings for the default call (pageable numpy
in, pooled page-locked outputs) and for page-locked caller buffers (the bench's e2e),
one process per setting (the settings are read at first use).
Usage: python tools/probe/host_sweep.py [log2_rows]"""

import json
import os
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def child(log2):
    sys.path.insert(0, REPO)
    import numpy as np
    import torch

    import paper_1606_06508_b200 as fn
    from paper_1606_06508_b200 import workloads

    n = 1 << log2
    p = fn.preset("double")
    xd = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    workloads.generate_device(5, xd)
    x = xd.cpu().numpy()
    del xd
    torch.cuda.empty_cache()
    out = {"env": {k: v for k, v in os.environ.items() if k.startswith("FASTNORM_B200")}, "rows": n}
    res = fn.normalize3(p, x)
    del res
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        res = fn.normalize3(p, x)
        ts.append(time.perf_counter() - t0)
        del res
    out["default_Gvec_s"] = n / min(ts) / 1e9
    xh = fn.host_empty((n, 3))
    np.copyto(xh, x)
    del x
    rh, uh = fn.host_empty((n,)), fn.host_empty((n, 3))
    fn.normalize3(p, xh, out=(rh, uh))
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        fn.normalize3(p, xh, out=(rh, uh))
        ts.append(time.perf_counter() - t0)
    out["pinned_Gvec_s"] = n / min(ts) / 1e9
    # pageable caller outputs (touched), pageable input: both sides staged
    xp = np.array(xh)
    rp, up = np.zeros(n), np.zeros((n, 3))
    del xh, rh, uh
    fn.normalize3(p, xp, out=(rp, up))
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        fn.normalize3(p, xp, out=(rp, up))
        ts.append(time.perf_counter() - t0)
    out["pageable_out_Gvec_s"] = n / min(ts) / 1e9
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "child":
        child(int(sys.argv[2]))
    else:
        log2 = int(sys.argv[1]) if len(sys.argv) > 1 else 28
        settings = [{}, {"FASTNORM_B200_COPY_THREADS": "16"}, {"FASTNORM_B200_COPY_THREADS": "8"}]
        for st in settings:
            env = dict(os.environ, **st)
            subprocess.run([sys.executable, __file__, "child", str(log2)], env=env, timeout=300)
