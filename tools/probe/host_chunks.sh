# host path for 1M / 16M-row arrays per chunk size (pageable and pinned)
for mb in 4 8 16 48; do
  FASTNORM_B200_HOST_CHUNK_MB=$mb timeout 300 python - <<'PY'
import os, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1606_06508_b200 as fn
p = fn.preset("double")
for n in (1 << 20, 1 << 24):
    for pinned in (False, True):
        x = torch.randn(n, 3, dtype=torch.float64, pin_memory=pinned).numpy()
        r = torch.empty(n, dtype=torch.float64, pin_memory=pinned).numpy(); u = torch.empty(n, 3, dtype=torch.float64, pin_memory=pinned).numpy()
        r.fill(0); u.fill(0)
        fn.normalize3(p, x, out=(r, u))
        t0 = time.perf_counter()
        for _ in range(5):
            fn.normalize3(p, x, out=(r, u))
        dt = (time.perf_counter() - t0) / 5
        print(f"chunk={os.environ['FASTNORM_B200_HOST_CHUNK_MB']}MB n={n} pinned={pinned}: {n / dt / 1e9:.3f} Gvec/s", flush=True)
PY
done
