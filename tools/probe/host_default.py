"""Developer probe (GPU): the default host call fn.normalize3(p, X) -- pageable numpy
input, library-allocated (page-locked pool) outputs -- under several staging settings,
plus host memcpy rates pageable -> page-locked with 1..16 Python threads.
Usage: python tools/probe/host_default.py [log2_rows]"""

import json
import os
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def child(log2):
    sys.path.insert(0, REPO)
    import numpy as np

    import paper_1606_06508_b200 as fn
    from paper_1606_06508_b200 import workloads

    n = 1 << log2
    p = fn.preset("double")
    x = np.empty((n, 3))
    step = 1 << 24
    for lo in range(0, n, step):
        x[lo:lo + step] = workloads.host_rows(5, lo, min(step, n - lo))
    res = fn.normalize3(p, x)
    del res
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        res = fn.normalize3(p, x)
        ts.append(time.perf_counter() - t0)
        del res
    env = {k: v for k, v in os.environ.items() if k.startswith("FASTNORM_B200")}
    print(json.dumps({"env": env, "rows": n, "best_s": min(ts), "Gvec_s": n / min(ts) / 1e9}), flush=True)


def memcpy_rates(log2):
    sys.path.insert(0, REPO)
    import numpy as np

    import paper_1606_06508_b200 as fn

    n = 1 << log2
    src = np.random.default_rng(0).random(n * 3)
    dst = fn.host_empty(n * 3)
    dst2 = np.empty(n * 3)
    dst2.fill(0)
    out = {}
    for name, d in (("to_page_locked", dst), ("to_pageable", dst2)):
        for th in (1, 4, 8, 12, 16):
            def work(k):
                per = len(src) // th
                np.copyto(d[k * per:(k + 1) * per], src[k * per:(k + 1) * per])
            best = None
            for _ in range(3):
                ts = [threading.Thread(target=work, args=(k,)) for k in range(th)]
                t0 = time.perf_counter()
                for t in ts:
                    t.start()
                for t in ts:
                    t.join()
                dt = time.perf_counter() - t0
                best = dt if best is None else min(best, dt)
            out[f"{name}_{th}t_GBs"] = src.nbytes / best / 1e9
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "child":
        child(int(sys.argv[2]))
    elif len(sys.argv) > 2 and sys.argv[1] == "memcpy":
        memcpy_rates(int(sys.argv[2]))
    else:
        log2 = int(sys.argv[1]) if len(sys.argv) > 1 else 28
        subprocess.run([sys.executable, __file__, "memcpy", str(log2)])
        settings = [{}, {"FASTNORM_B200_HOST_CHUNK_MB": "32"}, {"FASTNORM_B200_HOST_CHUNK_MB": "64"},
                    {"FASTNORM_B200_HOST_CHUNK_MB": "8"}, {"FASTNORM_B200_COPY_THREADS": "16"},
                    {"FASTNORM_B200_COPY_THREADS": "8"}, {"FASTNORM_B200_HOST_PIPES": "4"},
                    {"FASTNORM_B200_HOST_PIPES": "4", "FASTNORM_B200_HOST_CHUNK_MB": "32"},
                    {"FASTNORM_B200_HOST_POOL_MB": "0"}]
        for st in settings:
            env = dict(os.environ, **st)
            subprocess.run([sys.executable, __file__, "child", str(log2)], env=env)
