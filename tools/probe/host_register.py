"""How fast can pageable numpy buffers be page-locked in place (cudaHostRegister)?
Input (touched) and output (fresh np.empty, untouched) buffers of a 2^27-row 3-D f64
batch, registered whole and in 64 MiB pieces; then the library's host path on them."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1606_06508_b200 as fn  # noqa: E402

cr = torch.cuda.cudart()
torch.cuda.init()
rows = 1 << 27


def reg(a, piece=None):
    ptr, nb = a.ctypes.data, a.nbytes
    t0 = time.perf_counter()
    if piece is None:
        assert int(cr.cudaHostRegister(ptr, nb, 0)) == 0
        spans = [(ptr, nb)]
    else:
        spans = []
        for off in range(0, nb, piece):
            ln = min(piece, nb - off)
            assert int(cr.cudaHostRegister(ptr + off, ln, 0)) == 0
            spans.append((ptr + off, ln))
    t1 = time.perf_counter()
    for p, _ in spans:
        assert int(cr.cudaHostUnregister(p)) == 0
    t2 = time.perf_counter()
    return nb / (t1 - t0) / 1e9, nb / (t2 - t1) / 1e9


x = np.random.default_rng(0).standard_normal((rows, 3))
for piece in (None, 64 << 20):
    print(f"piece={piece}: touched input  register {reg(x, piece)[0]:.1f} GB/s, unregister {reg(x, piece)[1]:.1f} GB/s")
    u = np.empty((rows, 3))
    print(f"piece={piece}: fresh np.empty register {reg(u, piece)[0]:.1f} GB/s")
p = fn.preset("double")
r, u = np.empty(rows), np.empty((rows, 3))
fn.normalize3(p, x[:1000])
for rep in range(2):
    t0 = time.perf_counter()
    fn.normalize3(p, x, out=(r, u))
    t1 = time.perf_counter()
    print(f"pageable host path (outputs {'fresh' if rep == 0 else 'touched'}): {rows / (t1 - t0) / 1e9:.3f} Gvec/s")
t0 = time.perf_counter()
o = fn.normalize3(p, x)
t1 = time.perf_counter()
print(f"pageable host path, library allocates outputs: {rows / (t1 - t0) / 1e9:.3f} Gvec/s")
print("cores", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
