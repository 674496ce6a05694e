"""A/B timing of two builds of libfastnorm_b200.so on the bench workload (dev tool).

python tools/ab_lib.py OLD.so NEW.so [--reps 20] [--rounds 5]
Both libraries run fn_run(FN_OP_NORMALIZE, 3, FN_F64) over the same 2^30 config-5 rows,
interleaved round by round, timed with CUDA events on one stream."""
import ctypes
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_1606_06508_b200 import workloads  # noqa: E402


def load(path):
    L = ctypes.CDLL(path)
    L.fn_run.restype = ctypes.c_int
    L.fn_run.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 5
    return L


def main():
    # one library per process (each .so carries its own static cudart)
    if len(sys.argv) > 2:
        import subprocess
        for rd in range(3):
            for path in sys.argv[1:3]:
                subprocess.run([sys.executable, __file__, path], check=True)
        return
    libs = [load(sys.argv[1])]
    reps, rounds = 20, 3
    n = 1 << 30
    x = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    workloads.generate_device(5, x)
    r = torch.empty(n, dtype=torch.float64, device="cuda")
    u = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    import numpy as np
    ka = np.array([2.0 ** -482, 2.0 ** 510, 2.0 ** 592, 2.0 ** -514, 2.0 ** -592, 2.0 ** 514])
    s = torch.cuda.current_stream().cuda_stream
    res = {0: []}
    for rd in range(rounds):
        for k, L in enumerate(libs):
            for _ in range(3):
                rc = L.fn_run(1, 3, 1, x.data_ptr(), n, r.data_ptr(), u.data_ptr(), None, ka.ctypes.data, s)
                assert rc == 0, rc
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                L.fn_run(1, 3, 1, x.data_ptr(), n, r.data_ptr(), u.data_ptr(), None, ka.ctypes.data, s)
            e1.record()
            torch.cuda.synchronize()
            res[k].append(e0.elapsed_time(e1) / reps)
    for k in (0,):
        ms = statistics.median(res[k])
        print(f"{sys.argv[1 + k]}: {ms:.4f} ms/launch, {n * 56 / ms / 1e6:.1f} GB/s, all={['%.3f' % v for v in res[k]]}")


if __name__ == "__main__":
    main()
