"""Synthetic workloads (BASELINE.json configs): determinism, shard independence and the
advertised row-class frequencies, on the host restatement of the CUDA generator."""

import numpy as np
import pytest

from paper_1606_06508_b200 import workloads
from paper_1606_06508_b200.scale import kernel_args
from paper_1606_06508_b200.params import preset


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_shard_independence(cfg):
    full = workloads.host_rows(cfg, 1000, 4000)
    a = workloads.host_rows(cfg, 1000, 1500)
    b = workloads.host_rows(cfg, 2500, 2500)
    both = np.concatenate([a, b])
    assert both.dtype == full.dtype
    assert (both.view(np.uint8) == full.view(np.uint8)).all()
    c = workloads.CONFIGS[cfg]
    assert full.shape == (4000, c.dim) and str(full.dtype) == c.dtype


def test_cfg1_uniform():
    x = workloads.host_rows(1, 0, 200_000)
    assert x.min() >= -1.0 and x.max() < 1.0
    assert abs(x.mean()) < 0.01 and abs(x.var() - 1 / 3) < 0.01


def test_cfg2_classes():
    x = workloads.host_rows(2, 0, 400_000)
    zero = (x == 0).all(axis=1)
    assert abs(zero.mean() - 0.01) < 0.002
    e = np.frexp(np.abs(x[~zero]))[1] - 1
    assert e.min() >= -1000 and e.max() <= 1000
    assert np.signbit(x).mean() > 0.45


def test_cfg3_normal():
    x = workloads.host_rows(3, 0, 200_000)
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1.0) < 0.01


def test_cfg4_classes():
    x = workloads.host_rows(4, 0, 2_000_000)
    assert x.dtype == np.float32
    zero = (x == 0).all(axis=1)
    special = ~np.isfinite(x).any(axis=1) | ~np.isfinite(x).all(axis=1)
    assert abs(zero.mean() - 0.001) < 0.0003
    assert abs(special.mean() - 0.0001) < 0.00005
    finite = x[np.isfinite(x).all(axis=1) & ~zero]
    sub = (np.abs(finite) < np.finfo(np.float32).tiny) & (finite != 0)
    assert sub.any()
    assert np.abs(finite).max() > 1e37


def test_cfg5_classes():
    x = workloads.host_rows(5, 0, 1_000_000)
    m = np.abs(x).max(axis=1)
    nearmax = m >= 2.0 ** 1023
    subn = m < 2.0 ** -1022
    assert abs(nearmax.mean() - 0.005) < 0.0005
    assert abs(subn.mean() - 0.005) < 0.0005
    assert (x[subn] != 0).all()


@pytest.mark.parametrize("cfg", [2, 4, 5])
def test_row_stats_host(cfg):
    x = workloads.host_rows(cfg, 0, 100_000)
    prec = "single" if x.dtype == np.float32 else "double"
    c = workloads.row_stats_host(x, kernel_args(preset(prec)))
    assert int(c.sum()) == len(x)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("dim", [2, 3, 4])
def test_reference_regime_ranges(dtype, dim):
    """Regime contracts of the reference harness (bench.py:151-158, test_bench.py)."""
    p = preset("double" if dtype == "float64" else "single")
    n = 20000
    x = workloads.regime_rows("normal", dim, dtype, 0, n).astype(np.float64)
    assert (np.abs(x) >= p.tau_min).all() and (np.abs(x) <= p.tau_max).all()
    x = workloads.regime_rows("subnormal", dim, dtype, 0, n).astype(np.float64)
    assert (np.abs(x) >= p.alpha).all() and (np.abs(x) < p.nu).all()
    x = workloads.regime_rows("huge", dim, dtype, 0, n).astype(np.float64)
    assert (np.abs(x) > p.tau_max).all() and np.isfinite(x).all()
    x = workloads.regime_rows("mixed", dim, dtype, 0, n).astype(np.float64)
    assert np.isfinite(x).all() and (x != 0).all()
    assert (np.abs(x) < p.nu).any() and (np.abs(x) > p.tau_max).any()
    x = workloads.regime_rows("unit-ish", dim, dtype, 0, n).astype(np.float64)
    norms = np.sqrt((x * x).sum(axis=1))
    assert (np.abs(norms - 1.0) <= 2.0 ** -10 + 1e-6).all()
    a = workloads.regime_rows("mixed", dim, dtype, 100, 50)
    b = workloads.regime_rows("mixed", dim, dtype, 0, 200)[100:150]
    assert (a.view(np.uint8) == b.view(np.uint8)).all()
