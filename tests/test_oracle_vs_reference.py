"""Oracle vs the live reference (oracle/_ref, compiled from /root/reference by
`make -C oracle ref`).  Skipped where the reference build is absent.

Extends the golden pin to larger random sweeps (the test_backends.py:41-67 construction)
and to rows of every BASELINE workload, including the reference timing-loop checksum
over a workload sample (_kernels.pyx:646-789).
"""

import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import FAMILIES, SCALING, kernel_name, same_scalar

import oracle
from paper_1606_06508_b200 import workloads

REF = oracle.ref_module()
pytestmark = pytest.mark.skipif(REF is None, reason="oracle/_ref not built")

L = math.ldexp
KA = {
    "f64": (L(1, -482), L(1, 510), L(1, 592), L(1, -514), L(1, -592), L(1, 514)),
    "f32": (L(1, -49), L(1, 62), L(1, 100), L(1, -66), L(1, -100), L(1, 66)),
}


def _rows_vs_reference(x: np.ndarray, prec: str, dim: int, ka=None, families=None):
    ka = KA[prec] if ka is None else tuple(float(v) for v in ka)
    for fam in families or FAMILIES[dim]:
        fn = getattr(REF, kernel_name(fam, dim, prec))
        h, b, _ = oracle.run(oracle.BASE_OPS[fam], x, ka)
        for i, row in enumerate(x.astype(np.float64).tolist()):
            want = fn(*ka, *row) if fam in SCALING else fn(*row)
            want = want if isinstance(want, tuple) else (want,)
            got = (float(h[i]),) if b is None else (float(h[i]), *map(float, b[i]))
            assert all(same_scalar(p, q) for p, q in zip(got, want)), (fam, prec, row, got, want)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("dim", [2, 3, 4])
def test_random_sweep_vs_reference(prec, dim):
    rng = np.random.default_rng(7 + dim)
    single = prec == "f32"
    lo, hi = (-149, 127) if single else (-1074, 1023)
    m = 3000
    x = np.ldexp(1.0 + rng.random((m, dim)), rng.integers(lo, hi, (m, dim)))
    x *= rng.integers(0, 2, (m, dim)) * 2 - 1
    x = x.astype(np.float32) if single else x
    _rows_vs_reference(x, prec, dim)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_workload_rows_vs_reference(cfg):
    c = workloads.CONFIGS[cfg]
    prec = "f64" if c.dtype == "float64" else "f32"
    x = workloads.host_rows(cfg, 12345, 2000)
    if cfg in (4, 5):  # make sure the sample holds the rare special rows too
        rng = np.random.default_rng(cfg)
        pool = workloads.host_rows(cfg, 0, 400_000)
        sp = ~np.isfinite(pool).all(axis=1) | (np.abs(pool).max(axis=1) == 0)
        if cfg == 5:
            sp |= np.abs(pool).max(axis=1) > 2.0 ** 1022
            sp |= np.abs(pool).max(axis=1) < 2.0 ** -1022
        x = np.concatenate([x, pool[sp][:500]])
        assert sp.sum() > 100
        rng.shuffle(x)
    _rows_vs_reference(x, prec, c.dim)


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_loop_checksum_vs_reference(cfg):
    c = workloads.CONFIGS[cfg]
    x = workloads.host_rows(cfg, 0, 1 << 14)
    flat = np.ascontiguousarray(x.reshape(-1))
    ka = KA["f64"]
    fn = getattr(REF, f"loop_scaling{c.dim}_f64")
    want = fn(flat, 1 << 14, (1 << 14) - 1, *ka)
    got = oracle.loop(oracle.ALGO_SCALING, x, 1 << 14, (1 << 14) - 1, ka)
    assert got == want


# Non-preset constants: valid sets (non-power-of-two tau_min, a lower tau_max / sigma_max
# pair) and raw constants that fail validation but that the reference's kernels still
# take (non-power-of-two sigma).  The GPU side of the same sets is
# tests/test_gpu_parity.py::test_custom_parameter_sets.
CUSTOM_KA = {
    "f64": [(3 * L(1, -484), L(1, 510), L(1, 592), L(1, -514), L(1, -592), L(1, 514)),
            (L(1, -482), L(1, 500), L(1, 592), L(1, -530), L(1, -592), L(1, 530)),
            (L(1, -482), L(1, 510), 3 * L(1, 592), L(1, -514), L(1, -592) / 3, L(1, 514))],
    "f32": [(L(1, -49), L(1, 60), L(1, 100), L(1, -70), L(1, -100), L(1, 70)),
            (L(1, -49), L(1, 62), L(1, 100), 1.5 * L(1, -66), L(1, -100), L(1, 66) / 1.5)],
}


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_custom_constants_vs_reference(prec):
    rng = np.random.default_rng(99)
    single = prec == "f32"
    lo, hi = (-149, 127) if single else (-1074, 1023)
    for ka in CUSTOM_KA[prec]:
        for dim in (3, 4):
            m = 1500
            x = np.ldexp(1.0 + rng.random((m, dim)), rng.integers(lo, hi, (m, dim)))
            x *= rng.integers(0, 2, (m, dim)) * 2 - 1
            x = x.astype(np.float32) if single else x
            _rows_vs_reference(x, prec, dim, ka=ka, families=["scale", "normalize", "norm"])


# Full-range bit patterns, the strategies of the reference's property tests
# (tests/test_scale.py:23-28): every finite, subnormal, zero, infinite and NaN value of the
# format can come up, in any position of a row.
_f64 = st.integers(0, 2 ** 64 - 1).map(lambda b: float(np.array(b, np.uint64).view(np.float64)))
_f32 = st.integers(0, 2 ** 32 - 1).map(lambda b: float(np.array(b, np.uint32).view(np.float32)))


@settings(max_examples=300, deadline=None)
@given(dim=st.sampled_from([2, 3, 4]), prec=st.sampled_from(["f64", "f32"]), data=st.data())
def test_hypothesis_rows_vs_reference(dim, prec, data):
    """Hypothesis-drawn rows: the oracle equals the reference's compiled kernels on every
    family (the reference's _same rule)."""
    vals = data.draw(st.lists(st.lists(_f64 if prec == "f64" else _f32, min_size=dim, max_size=dim),
                              min_size=1, max_size=8))
    x = np.array(vals, dtype=np.float64 if prec == "f64" else np.float32)
    _rows_vs_reference(x, prec, dim)


def _sample_vs_reference(x: np.ndarray, prec: str, dim: int, fam: str):
    """Vectorised form of _rows_vs_reference for large samples: the reference's compiled
    export called row by row, compared with the oracle as arrays (the _same rule)."""
    ka = KA[prec]
    f = getattr(REF, kernel_name(fam, dim, prec))
    rows = x.astype(np.float64).tolist()
    want = np.array([f(*ka, *row) for row in rows] if fam in SCALING else [f(*row) for row in rows],
                    dtype=np.float64).reshape(len(rows), -1)
    h, b, _ = oracle.run(oracle.BASE_OPS[fam], x, ka if fam in SCALING else None)
    got = h[:, None].astype(np.float64) if b is None else np.concatenate([h[:, None], b], axis=1).astype(np.float64)
    both_nan = np.isnan(got) & np.isnan(want)
    same = both_nan | ((got == want) & (np.signbit(got) == np.signbit(want)))
    bad = np.flatnonzero(~same.all(axis=1))
    assert bad.size == 0, (fam, prec, bad[:5], x[bad[:5]], got[bad[:5]], want[bad[:5]])


@pytest.mark.parametrize("cfg,rows", [(1, 1 << 20), (2, 1 << 20), (3, 1 << 20), (4, 1 << 22), (5, 1 << 22)])
def test_workload_sample_vs_reference(cfg, rows):
    """A 4-million-row sample of configs 4 and 5 (whose full-size parity reaches the
    reference only through the oracle: their NaN / infinity / overflowing rows make the
    reference's loop checksums uninformative) and 2^20 rows of configs 1-3, normalize
    family, plus the quotient variant the config runs: the oracle equals the reference's
    compiled exports on every row."""
    c = workloads.CONFIGS[cfg]
    prec = "f64" if c.dtype == "float64" else "f32"
    x = workloads.host_rows(cfg, 777 * cfg, rows)
    _sample_vs_reference(x, prec, c.dim, "normalize")
    if cfg in (2, 4):
        _sample_vs_reference(x[: rows // 4], prec, c.dim, "quotient")
