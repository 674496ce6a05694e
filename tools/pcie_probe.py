"""PCIe ceiling probe (developer tool): pinned H2D, D2H and both directions at once,
then the library's host path (fn_host_run) at several chunk sizes / pipe counts."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

GB = 1 << 30


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    n = 4 * GB
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    t = timed(lambda: d.copy_(h, non_blocking=True))
    print(f"H2D pinned: {n / t / 1e9:.1f} GB/s")
    t = timed(lambda: h.copy_(d, non_blocking=True))
    print(f"D2H pinned: {n / t / 1e9:.1f} GB/s")

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    t = timed(both)
    print(f"H2D+D2H concurrent: {2 * n / t / 1e9:.1f} GB/s total ({n / t / 1e9:.1f} each way)")

    import paper_1606_06508_b200 as fn
    p = fn.preset("double")
    rows = 1 << 28
    x = torch.empty((rows, 3), dtype=torch.float64, pin_memory=True)
    x.uniform_(-1, 1)
    r = torch.empty(rows, dtype=torch.float64, pin_memory=True)
    u = torch.empty((rows, 3), dtype=torch.float64, pin_memory=True)
    xn, rn, un = x.numpy(), r.numpy(), u.numpy()
    fn.normalize3(p, xn[:1000], out=(rn[:1000], un[:1000]))
    t = timed(lambda: fn.normalize3(p, xn, out=(rn, un)))
    print(f"fn_host_run normalize3 f64 2^28 rows: {rows / t / 1e9:.3f} Gvec/s, "
          f"{rows * 24 / t / 1e9:.1f} GB/s in + {rows * 32 / t / 1e9:.1f} GB/s out "
          f"(chunk={os.environ.get('FASTNORM_B200_HOST_CHUNK_MB', 'default')} MB, "
          f"pipes={os.environ.get('FASTNORM_B200_HOST_PIPES', 'default')})")


if __name__ == "__main__" and "--pageable" not in sys.argv:
    main()


def pageable():
    """The host path with ordinary (pageable) numpy arrays, as most callers pass them."""
    import numpy as np

    import paper_1606_06508_b200 as fn
    p = fn.preset("double")
    rows = 1 << 27
    x = np.random.default_rng(0).uniform(-1, 1, (rows, 3))
    r = np.empty(rows)
    u = np.empty((rows, 3))
    fn.normalize3(p, x[:1000], out=(r[:1000], u[:1000]))
    t = timed(lambda: fn.normalize3(p, x, out=(r, u)))
    print(f"fn_host_run normalize3 f64 2^27 rows PAGEABLE: {rows / t / 1e9:.3f} Gvec/s "
          f"({rows * 56 / t / 1e9:.1f} GB/s over PCIe)")


if __name__ == "__main__" and "--pageable" in sys.argv:
    pageable()
