"""GPU error-bound sweep (reference oracle.py:151-290, acceptance criteria 2-3): the
paper's bounds hold for every row of every reference regime and config, the double-
double metrics agree with exact rational arithmetic, and violations are detected."""

import math
from fractions import Fraction

import pytest

import paper_1606_06508_b200 as fn
from paper_1606_06508_b200 import workloads
from paper_1606_06508_b200.bounds import sweep_bounds

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _rows(regime, dim, prec, n, dev, seed=21):
    dt = torch.float64 if prec == "double" else torch.float32
    x = torch.empty((n, dim), dtype=dt, device=dev)
    workloads.generate_regime_device(regime, x, seed=seed)
    return x


@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("regime", ["normal", "subnormal", "huge", "mixed", "unit-ish"])
def test_bounds_hold_on_reference_regimes(cuda_dev, prec, regime):
    p = fn.preset(prec)
    for dim in (2, 3, 4):
        n = 1 << 22
        s = sweep_bounds(p, _rows(regime, dim, prec, n, cuda_dev))
        assert s.samples + s.skipped == n and s.skipped == 0
        assert s.violation_count == 0, (regime, prec, dim, s.violation_ids, s.first_violation_row)
        assert s.max_metrics["dir_err"] <= 3.001 + dim / 2
        if dim < 4:
            assert s.max_metrics["sin_phi"] <= 1.001


def test_bounds_hold_on_cfg5_and_cfg4(cuda_dev):
    for cfg, prec in ((5, "double"), (4, "single")):
        c = workloads.CONFIGS[cfg]
        n = 1 << 24
        x = torch.empty((n, c.dim), dtype=torch.float64 if prec == "double" else torch.float32,
                        device=cuda_dev)
        workloads.generate_device(cfg, x)
        s = sweep_bounds(fn.preset(prec), x)
        assert s.violation_count == 0, (cfg, s.violation_ids)
        assert s.skipped > 0 if cfg == 4 else s.skipped == 0  # NaN/Inf/zero rows are skipped


def _exact_metrics(xs, r_hat, unit):
    q = [Fraction(v) for v in xs]
    s = sum(v * v for v in q)
    # direction error^2 = sum (u_k - x_k / r)^2, evaluated with r from a 200-bit isqrt
    bits = 200
    r_fx = Fraction(math.isqrt((s.numerator * s.denominator) << (2 * bits)), s.denominator << bits)
    d2 = sum((Fraction(uk) - xk / r_fx) ** 2 for uk, xk in zip(unit, q))
    rel = abs(Fraction(r_hat) - r_fx) / r_fx
    return float(rel), math.sqrt(float(d2))


def test_metrics_match_exact_rationals(cuda_dev):
    p = fn.preset("double")
    for regime in ("mixed", "normal"):
        x = _rows(regime, 3, "double", 400, cuda_dev, seed=5)
        out = fn.normalize3(p, x)
        s = sweep_bounds(p, x, out)
        xh, rh, uh = x.cpu().numpy(), out.length.cpu().numpy(), out.unit.cpu().numpy()
        rels, dirs = [], []
        for i in range(len(xh)):
            rel, d = _exact_metrics(xh[i].tolist(), float(rh[i]), uh[i].tolist())
            rels.append(rel)
            dirs.append(d)
        assert s.max_metrics["rel_length_err"] == pytest.approx(max(rels) / p.u, rel=1e-9, abs=1e-9)
        assert s.max_metrics["dir_err"] == pytest.approx(max(dirs) / p.u, rel=1e-9, abs=1e-9)


def test_violations_are_detected(cuda_dev):
    p = fn.preset("double")
    x = _rows("normal", 3, "double", 10000, cuda_dev, seed=9)
    out = fn.normalize3(p, x)
    bad_r = out.length.clone()
    bad_r[::100] *= 1.0 + 8 * p.u          # 100 rows with a length error > 2.5u
    s = sweep_bounds(p, x, fn.NormalizeOutcome(bad_r, out.unit))
    assert s.violation_ids.get("length-in-range") == 100 and s.first_violation_row == 0
    bad_u = out.unit.clone()
    bad_u[5, 0] += 64 * p.u
    s = sweep_bounds(p, x, fn.NormalizeOutcome(out.length, bad_u))
    assert s.violation_count == 1 and s.first_violation_row == 5
    nan_u = out.unit.clone()
    nan_u[7, 1] = float("nan")
    s = sweep_bounds(p, x, fn.NormalizeOutcome(out.length, nan_u))
    assert s.violation_ids == {"nan-output": 1}
