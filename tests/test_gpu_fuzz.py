"""Large batches of arbitrary bit patterns through every binary64 and binary32 family,
against the oracle (the hypothesis suite's full-range strategy at a million rows per
call): random 64/32-bit words (NaN payloads, infinities, subnormals, zeros), rows whose
components share the bottom of the exponent range, and rows spread up to 1100 binades
below their largest component (every quotient lands on the subnormal grid or flushes to
zero somewhere).  The comparison variants' division sites see every operand class here."""

import numpy as np
import pytest

import oracle
import paper_1606_06508_b200 as fn
from paper_1606_06508_b200 import _cuda_kernels, _lib

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROWS = 1 << 20
OPS = {"scale": _lib.OP_SCALE, "normalize": _lib.OP_NORMALIZE, "norm": _lib.OP_NORM,
       "naive": _lib.OP_NAIVE, "quotient": _lib.OP_QUOTIENT, "quotient3_fast": _lib.OP_QUOTIENT3_FAST}


def _rows(rng, n, dim, kind, f64):
    if f64:
        w = rng.integers(0, 2 ** 64, size=(n, dim), dtype=np.uint64)
        keep, shift, emax = np.uint64(0x800FFFFFFFFFFFFF), np.uint64(52), 2046
    else:
        w = rng.integers(0, 2 ** 32, size=(n, dim), dtype=np.uint64).astype(np.uint32)
        keep, shift, emax = np.uint32(0x807FFFFF), np.uint32(23), 254
    ut = w.dtype.type
    if kind == "bottom":
        e = rng.integers(0, 70 if f64 else 12, size=(n, dim))
        w = (w & keep) | (e.astype(w.dtype) << shift)
    elif kind == "spread":
        top = rng.integers(0, emax + 1, size=(n, 1))
        e = np.clip(top - rng.integers(0, 1100 if f64 else 160, size=(n, dim)), 0, emax)
        w = (w & keep) | (e.astype(w.dtype) << ut(shift))
    return w.view(np.float64 if f64 else np.float32)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("kind", ["bits", "bottom", "spread"])
@pytest.mark.parametrize("dim", [2, 3, 4])
def test_fuzz_every_family(cuda_dev, prec, kind, dim):
    rng = np.random.default_rng(1000 * dim + {"bits": 0, "bottom": 1, "spread": 2}[kind] + (0 if prec == "f64" else 7))
    f64 = prec == "f64"
    x = _rows(rng, ROWS, dim, kind, f64)
    xd = torch.from_numpy(x).to(cuda_dev)
    ka = np.array(fn.kernel_args(fn.preset("double" if f64 else "single")))
    fams = ["scale", "normalize", "norm", "naive", "quotient"] + (["quotient3_fast"] if dim == 3 else [])
    for fam in fams:
        base = "quotient3_fast" if fam == "quotient3_fast" else f"{fam}{dim}"
        takes = fam in ("scale", "normalize", "norm")
        res = _cuda_kernels.batch_kernel(base, prec)(xd, ka if takes else None)
        h, b, _ = oracle.run(OPS[fam], x, ka if takes else None)
        gh = res.head.cpu().numpy()
        ok = oracle.same(gh, h)
        if b is not None:
            ok &= oracle.same(res.body.cpu().numpy(), b).all(axis=1)
        bad = np.flatnonzero(~ok)
        assert bad.size == 0, (base, prec, kind, bad.size, [hex(v) for v in x[bad[0]].view(
            np.uint64 if f64 else np.uint32)])
