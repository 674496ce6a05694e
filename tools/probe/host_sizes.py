"""Host path throughput across array sizes, pageable and page-locked (dev probe)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1606_06508_b200 as fn  # noqa: E402

p = fn.preset("double")
for n in (1 << 16, 1 << 18, 1 << 20, 1 << 22, 1 << 24, 1 << 26):
    for pinned in (False, True):
        x = torch.randn(n, 3, dtype=torch.float64, pin_memory=pinned).numpy()
        r = torch.empty(n, dtype=torch.float64, pin_memory=pinned).numpy()
        u = torch.empty(n, 3, dtype=torch.float64, pin_memory=pinned).numpy()
        r.fill(0)
        u.fill(0)
        fn.normalize3(p, x, out=(r, u))
        reps = max(3, min(200, (1 << 24) // n))
        t0 = time.perf_counter()
        for _ in range(reps):
            fn.normalize3(p, x, out=(r, u))
        dt = (time.perf_counter() - t0) / reps
        print(f"n=2^{n.bit_length() - 1:<3d} pinned={int(pinned)}: {n / dt / 1e9:.3f} Gvec/s", flush=True)
