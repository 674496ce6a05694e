"""Hypothesis-drawn batches through the GPU kernels, against the oracle: the reference's
property-test strategies (full-range bit patterns, tests/test_scale.py:23-28) used as
batch generators, so shrinking finds a minimal failing row if one exists."""

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from conftest import FAMILIES, SCALING

import oracle
import paper_1606_06508_b200 as fn
from paper_1606_06508_b200 import _cuda_kernels, _lib

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

OPS = {"scale": _lib.OP_SCALE, "normalize": _lib.OP_NORMALIZE, "norm": _lib.OP_NORM,
       "naive": _lib.OP_NAIVE, "quotient": _lib.OP_QUOTIENT, "quotient3_fast": _lib.OP_QUOTIENT3_FAST}
_bits = {"f64": st.integers(0, 2 ** 64 - 1), "f32": st.integers(0, 2 ** 32 - 1)}


@settings(max_examples=150, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])
@given(dim=st.sampled_from([2, 3, 4]), prec=st.sampled_from(["f64", "f32"]),
       offset=st.integers(0, 3), data=st.data())
def test_hypothesis_batches_vs_oracle(cuda_dev, dim, prec, offset, data):
    """Every family on a drawn batch (1-600 rows of arbitrary bit patterns, storage
    shifted by 0-3 elements so aligned and misaligned kernels both run) equals the oracle."""
    n = data.draw(st.integers(1, 600))
    words = data.draw(st.lists(_bits[prec], min_size=n * dim, max_size=n * dim))
    ut = np.uint64 if prec == "f64" else np.uint32
    x = np.array(words, dtype=ut).view(np.float64 if prec == "f64" else np.float32).reshape(n, dim)
    buf = torch.zeros(n * dim + offset, dtype=torch.float64 if prec == "f64" else torch.float32,
                      device=cuda_dev)
    xd = buf[offset:].view(n, dim)
    xd.copy_(torch.from_numpy(x))
    ka = np.array(fn.kernel_args(fn.preset("double" if prec == "f64" else "single")))
    for fam in FAMILIES[dim]:
        base = "quotient3_fast" if fam == "quotient3_fast" else f"{fam}{dim}"
        takes = fam in SCALING
        res = _cuda_kernels.batch_kernel(base, prec)(xd, ka if takes else None)
        h, b, _ = oracle.run(OPS[fam], x, ka if takes else None)
        assert oracle.same(res.head.cpu().numpy(), h).all(), (fam, prec, dim, offset)
        if b is not None:
            assert oracle.same(res.body.cpu().numpy(), b).all(), (fam, prec, dim, offset)
