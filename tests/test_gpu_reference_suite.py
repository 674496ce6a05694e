"""The reference's example-based and contract tests for the normalization kernels,
restated as batched GPU tests.

Each test names the reference test it restates (pkg/tests/...).  The reference checks
one row per scalar call; here the rows of a test go to the device as one [N, n] batch
through the public API, and each row is then checked with the reference's rule:
exact values, a tolerance in units of u, or a contract such as NaN in -> NaN out.
Exact comparison values come from 400-bit mpmath arithmetic.  This replaces the
reference's gmpy2 `oracle.ref_normalize`, which is not installed here.  Bit parity
with the reference kernels on these rows is covered separately by the golden
fixtures (test_gpu_parity.py).
"""

import math

import numpy as np
import pytest

import paper_1606_06508_b200 as fn
from paper_1606_06508_b200 import workloads
from paper_1606_06508_b200.bounds import sweep_bounds

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
mpmath = pytest.importorskip("mpmath")

L = math.ldexp
U64, U32 = 2.0 ** -53, 2.0 ** -24
DT = {"double": torch.float64, "single": torch.float32}


def _run(f, rows, prec="double", p=None):
    """One batched launch of public function f over `rows`; (length [N], unit [N, n])."""
    x = torch.tensor(rows, dtype=DT[prec], device="cuda")
    out = f(p, x) if p is not None else f(x)
    return out.length.double().cpu().numpy(), out.unit.double().cpu().numpy()


def _exact(xs):
    """Correctly rounded length and unit vector of a finite nonzero row."""
    with mpmath.workprec(400):
        v = [mpmath.mpf(float(c)) for c in xs]
        r = mpmath.sqrt(mpmath.fsum(c * c for c in v))
        return float(r), [float(c / r) for c in v]


def _bits_equal(a, b):
    return (np.asarray(a, np.float64).view(np.int64) == np.asarray(b, np.float64).view(np.int64)).all()


# --- pkg/tests/test_normalize.py -------------------------------------------------------

def test_normalize_examples():
    """TestExamples (test_normalize.py:23-74)."""
    d, s = fn.preset("double"), fn.preset("single")
    r, u = _run(fn.normalize2, [[3.0, 4.0], [0.0, 0.0], [L(1, -1074), 0.0]], p=d)
    assert r[0] == 5.0 and abs(u[0, 0] - 0.6) <= 4 * d.u and abs(u[0, 1] - 0.8) <= 4 * d.u
    assert r[1] == 0.0 and _bits_equal(u[1], [0.0, 0.0])
    assert r[2] == L(1, -1074) and _bits_equal(u[2], [1.0, 0.0])

    big = [L(1, 600)] * 3
    r, u = _run(fn.normalize3, [[0.0, 0.0, 0.0], [2.0, 10.0, 11.0], big], p=d)
    assert r[0] == 0.0 and _bits_equal(u[0], [0.0, 0.0, 0.0])
    assert r[1] == 15.0
    assert all(abs(g - w) <= 5 * d.u for g, w in zip(u[1], (2 / 15, 10 / 15, 11 / 15)))
    r_ref, _ = _exact(big)
    assert r[2] == r_ref  # correctly rounded 2^600 * sqrt(3)

    upscale = [3 * L(1, -520), 0.0, 4 * L(1, -520), 0.0]
    r, u = _run(fn.normalize4, [[0.0] * 4, [1.0] * 4, upscale], p=d)
    assert r[0] == 0.0 and _bits_equal(u[0], [0.0, 0.0, 0.0, 1.0])
    assert r[1] == 2.0 and _bits_equal(u[1], [0.5] * 4)
    assert r[2] == 5 * L(1, -520)
    assert abs(u[2, 0] - 0.6) <= 8 * d.u and abs(u[2, 2] - 0.8) <= 8 * d.u

    r, u = _run(fn.normalize4, [[0.0] * 4], "single", p=s)
    assert r[0] == 0.0 and _bits_equal(u[0], [0.0, 0.0, 0.0, 1.0])
    r, u = _run(fn.normalize2, [[3.0, 4.0]], "single", p=s)
    assert r[0] == 5.0


def test_normalize_examples_meet_error_bounds():
    """The oracle.measure(...).bound_violations == () checks of test_normalize.py:29,
    :48, :55-57, :69, :74 and :122-125, through the GPU bound sweep."""
    d, s = fn.preset("double"), fn.preset("single")
    cases = {2: [[3.0, 4.0]], 3: [[2.0, 10.0, 11.0], [L(1, 600)] * 3,
                                  [L(1, -1060), -L(3, -1070), L(1, -1074)]],
             4: [[3 * L(1, -520), 0.0, 4 * L(1, -520), 0.0]]}
    for n, rows in cases.items():
        x = torch.tensor(rows, dtype=torch.float64, device="cuda")
        summary = sweep_bounds(d, x)
        assert summary.violation_count == 0 and summary.samples == len(rows), (n, summary)
    summary = sweep_bounds(s, torch.tensor([[3.0, 4.0]], dtype=torch.float32, device="cuda"))
    assert summary.violation_count == 0 and summary.samples == 1
    # the huge equilateral row: relative length error <= 2.5u (test_normalize.py:57)
    x = torch.tensor([[L(1, 600)] * 3], dtype=torch.float64, device="cuda")
    assert sweep_bounds(d, x).max_metrics["rel_length_err"] <= 2.5


def test_norm_examples():
    """TestNormOnly.test_examples (test_normalize.py:78-81)."""
    d = fn.preset("double")
    assert fn.norm2(d, torch.tensor([[3.0, 4.0]], dtype=torch.float64, device="cuda")).item() == 5.0
    assert fn.norm3(d, torch.zeros((1, 3), dtype=torch.float64, device="cuda")).item() == 0.0
    x4 = torch.tensor([[L(1, -1074), 0.0, 0.0, 0.0]], dtype=torch.float64, device="cuda")
    assert fn.norm4(d, x4).item() == L(1, -1074)


def test_warranted_overflow():
    """TestBounds.test_warranted_overflow (test_normalize.py:115-120)."""
    d = fn.preset("double")
    r, u = _run(fn.normalize3, [[d.omega] * 3], p=d)
    assert math.isinf(r[0]) and all(abs(v - 1 / math.sqrt(3)) <= 8 * d.u for v in u[0])


@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("n", [2, 3, 4])
def test_normalize_nan_contracts(n, prec):
    """TestNaN (test_normalize.py:128-145): NaN anywhere -> NaN out; clean rows never
    give NaN."""
    p = fn.preset(prec)
    f = getattr(fn, f"normalize{n}")
    rows = []
    for i in range(n):
        for fill in (0.0, 1.0, L(1, -600 if prec == "double" else -100)):
            row = [fill] * n
            row[i] = math.nan
            rows.append(row)
    r, u = _run(f, rows, prec, p=p)
    assert (np.isnan(r) | np.isnan(u).any(axis=1)).all()
    if prec == "double":
        r, u = _run(f, [[v] * n for v in (0.0, 1.0, L(1, 500), L(1, -1074))], p=p)
        assert not np.isnan(r).any() and not np.isnan(u).any()


# --- pkg/tests/test_baselines.py -------------------------------------------------------

def test_naive_examples():
    """TestNaive (test_baselines.py:24-52)."""
    r, u = _run(fn.naive_normalize2, [[3.0, 4.0], [L(1, -600), 0.0], [0.0, 0.0]])
    assert r[0] == 5.0 and abs(u[0, 0] - 0.6) <= 4 * U64
    assert r[1] == 0.0 and u[1, 0] == math.inf and math.isnan(u[1, 1])
    assert r[2] == 0.0 and np.isnan(u[2]).all()
    r, u = _run(fn.naive_normalize3, [[L(1, 600), 0.0, 0.0]])
    assert r[0] == math.inf and _bits_equal(u[0], [0.0, 0.0, 0.0])
    r, u = _run(fn.naive_normalize3, [[L(1, 70), 0.0, 0.0]], "single")
    assert r[0] == math.inf and _bits_equal(u[0], [0.0, 0.0, 0.0])


def test_quotient_robust_examples():
    """TestQuotientRobust (test_baselines.py:55-75)."""
    half = fn.preset("double").omega / 2
    r, u = _run(fn.quotient3_robust, [[3.0, 4.0, 12.0], [0.0] * 3, [L(1, -1074), 0.0, 0.0], [half] * 3])
    assert abs(r[0] - 13.0) <= 13 * 4 * U64
    assert all(abs(g - w) <= 4 * U64 for g, w in zip(u[0], (3 / 13, 4 / 13, 12 / 13)))
    assert r[1] == 0.0 and _bits_equal(u[1], [0.0] * 3)
    assert r[2] == L(1, -1074) and _bits_equal(u[2], [1.0, 0.0, 0.0])
    assert math.isfinite(r[3]) and all(abs(v - 1 / math.sqrt(3)) <= 8 * U64 for v in u[3])


PIVOT_ROWS = [(12.0, 4.0, 3.0), (4.0, 12.0, 3.0), (4.0, 3.0, 12.0), (3.0, 4.0, 12.0),
              (-12.0, 4.0, -3.0)]


def test_quotient_fast_examples_and_pivot_paths():
    """TestQuotientFast (test_baselines.py:78-109): zero, (3,4,12), NaN in x1, and every
    pivot branch against the exact result."""
    r, u = _run(fn.quotient3_fast, [[0.0] * 3, [math.nan, 1.0, 0.0]] + [list(v) for v in PIVOT_ROWS])
    assert r[0] == 0.0 and _bits_equal(u[0], [0.0] * 3)
    assert math.isnan(r[1]) and np.isnan(u[1]).all()
    for k, xs in enumerate(PIVOT_ROWS, start=2):
        r_ref, u_ref = _exact(xs)
        assert abs(r[k] - r_ref) <= 13 * 4 * U64
        assert all(abs(g - w) <= 4 * U64 for g, w in zip(u[k], u_ref))


def _full_range(n, dim, seed):
    """The st_f64 strategy of test_scale.py:23-25 (uniform over the positive finite bit
    patterns, random sign), as a batch."""
    rng = np.random.default_rng(seed)
    x = rng.integers(1, 0x7FEFFFFFFFFFFFFF, (n, dim), dtype=np.uint64).view(np.float64)
    return x * np.where(rng.random((n, dim)) < 0.5, -1.0, 1.0)


def test_quotient_fast_agrees_with_robust():
    """TestQuotientFast.test_agrees_with_robust (test_baselines.py:111-121), on 2^20
    full-range rows: units within 8u, lengths within 8u relative above the subnormal
    grid."""
    x = torch.from_numpy(_full_range(1 << 20, 3, seed=113)).cuda()
    a, b = fn.quotient3_fast(x), fn.quotient3_robust(x)
    assert ((a.unit - b.unit).abs() <= 8 * U64).all()
    la, lb = a.length, b.length
    m = torch.isfinite(la) & torch.isfinite(lb) & (lb >= 2.0 ** -1022)
    assert m.float().mean().item() > 0.99
    assert ((la - lb).abs()[m] <= 8 * U64 * torch.maximum(la.abs(), lb.abs())[m]).all()


def test_quotient2_quotient4_examples():
    """TestQuotient24 (test_baselines.py:124-131): n = 4 zero gives five zeros, no
    identity quaternion."""
    r, u = _run(fn.quotient2, [[3.0, 4.0], [0.0, 0.0]])
    assert r[0] == 5.0 and abs(u[0, 0] - 0.6) <= 4 * U64
    assert r[1] == 0.0 and _bits_equal(u[1], [0.0, 0.0])
    r, u = _run(fn.quotient4, [[1.0] * 4, [0.0] * 4])
    assert r[0] == 2.0 and _bits_equal(u[0], [0.5] * 4)
    assert r[1] == 0.0 and _bits_equal(u[1], [0.0] * 4)


@pytest.mark.parametrize("n", [2, 3, 4])
def test_baseline_nan_contracts(n):
    """TestNaNContracts (test_baselines.py:141-159)."""
    quotients = {2: [fn.quotient2], 3: [fn.quotient3_robust, fn.quotient3_fast], 4: [fn.quotient4]}[n]
    rows = []
    for i in range(n):
        for fill in (0.0, 1.0, L(1, -1074), L(1, 600)):
            row = [fill] * n
            row[i] = math.nan
            rows.append(row)
    for f in quotients:
        r, u = _run(f, rows)
        assert (np.isnan(r) | np.isnan(u).any(axis=1)).all(), f.__name__
    naive = getattr(fn, f"naive_normalize{n}")
    rows = []
    for i in range(n):
        row = [1.0] * n
        row[i] = math.nan
        rows.append(row)
    r, _ = _run(naive, rows)
    assert np.isnan(r).all()


@pytest.mark.parametrize("n", [2, 3, 4])
def test_in_band_agreement_with_exact(n):
    """TestInBandAgreementWithOracle (test_baselines.py:162-181): inside the safe band,
    scaling, naive and the quotients all track the exact result (length within 3u
    relative, unit within (3.001 + n/2)u)."""
    d = fn.preset("double")
    rows = workloads.regime_rows("normal", n, "float64", 0, 300, seed=5)
    x = torch.from_numpy(rows).cuda()
    quotients = {2: [fn.quotient2], 3: [fn.quotient3_robust, fn.quotient3_fast], 4: [fn.quotient4]}[n]
    outs = [getattr(fn, f"normalize{n}")(d, x), getattr(fn, f"naive_normalize{n}")(x)]
    outs += [f(x) for f in quotients]
    exact = [_exact(row) for row in rows.tolist()]
    r_ref = np.array([e[0] for e in exact])
    u_ref = np.array([e[1] for e in exact])
    for o in outs:
        r, u = o.length.cpu().numpy(), o.unit.cpu().numpy()
        assert (np.abs(r - r_ref) <= 3 * U64 * r_ref).all()
        assert (np.abs(u - u_ref) <= (3.001 + n / 2) * U64).all()


# --- pkg/tests/test_acceptance.py ------------------------------------------------------

def test_acceptance_4_robustness_differential():
    """Criterion 4 (test_acceptance.py:180-203): naive overflows / underflows where the
    scaling algorithm stays within 2.5u of the exact length."""
    d = fn.preset("double")
    rn3, _ = _run(fn.naive_normalize3, [[L(1, 600), 0.0, 0.0]])
    rn2, _ = _run(fn.naive_normalize2, [[L(1, -600), 0.0]])
    assert rn3[0] == math.inf and rn2[0] == 0.0
    r3, _ = _run(fn.normalize3, [[L(1, 600), 0.0, 0.0]], p=d)
    r2, _ = _run(fn.normalize2, [[L(1, -600), 0.0]], p=d)
    assert abs(r3[0] - L(1, 600)) <= 2.5 * U64 * L(1, 600)
    assert abs(r2[0] - L(1, -600)) <= 2.5 * U64 * L(1, -600)


ACCEPT5_FILLS = {
    "double": [0.0, 1.0, -1.0, L(1, -1074), L(1, -482), L(1, 600), -L(1, -600)],
    "single": [0.0, 1.0, -1.0, L(1, -149), L(1, -49), L(1, 70), -L(1, -70)],
}


@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("n", [2, 3, 4])
def test_acceptance_5_zero_and_nan_contracts(n, prec):
    """Criterion 5 (test_acceptance.py:210-244): the zero outcome of scale / normalize /
    norm, and NaN at every position for every fill value."""
    p = fn.preset(prec)
    dt = DT[prec]
    zero = torch.zeros((1, n), dtype=dt, device="cuda")
    s = getattr(fn, f"scale{n}")(p, zero)
    assert s.inv_sigma.item() == 0.0 and (s.scaled == 0).all()
    nz = getattr(fn, f"normalize{n}")(p, zero)
    want = [0.0, 0.0, 0.0, 1.0] if n == 4 else [0.0] * n
    assert nz.length.item() == 0.0 and _bits_equal(nz.unit.double().cpu().numpy()[0], want)
    assert getattr(fn, f"norm{n}")(p, zero).item() == 0.0
    rows = []
    for i in range(n):
        for fill in ACCEPT5_FILLS[prec]:
            row = [fill] * n
            row[i] = math.nan
            rows.append(row)
    x = torch.tensor(rows, dtype=dt, device="cuda")
    assert torch.isnan(getattr(fn, f"scale{n}")(p, x).scaled).any(dim=1).all()
    o = getattr(fn, f"normalize{n}")(p, x)
    assert (torch.isnan(o.length) | torch.isnan(o.unit).any(dim=1)).all()
    assert torch.isnan(getattr(fn, f"norm{n}")(p, x)).all()


@pytest.mark.parametrize("prec", ["double", "single"])
def test_acceptance_8_cross_algorithm_agreement(prec):
    """Criterion 8 (test_acceptance.py:326-360): scaling, quotient and naive agree
    pairwise inside the safe band (length within 4u relative, unit within 8u).  The
    reference checks a tenth of its sample count per n; here 2^20 rows per n, generated
    on the device."""
    p = fn.preset(prec)
    u = p.u
    quotient = {2: fn.quotient2, 3: fn.quotient3_robust, 4: fn.quotient4}
    for n in (2, 3, 4):
        x = torch.empty((1 << 20, n), dtype=DT[prec], device="cuda")
        workloads.generate_regime_device("normal", x, seed=88 + n)
        outs = [getattr(fn, f"normalize{n}")(p, x), quotient[n](x), getattr(fn, f"naive_normalize{n}")(x)]
        for a in range(3):
            for b in range(a + 1, 3):
                la, lb = outs[a].length.double(), outs[b].length.double()
                assert ((la - lb).abs() <= 4 * u * torch.maximum(la, lb)).all(), (n, a, b)
                du = (outs[a].unit.double() - outs[b].unit.double()).abs()
                assert (du <= 8 * u).all(), (n, a, b)


# --- pkg/tests/test_rotation.py / acceptance criterion 6 -------------------------------

def test_rotation_cross_validation():
    """TestCrossValidation (test_rotation.py:103-123) and criterion 6
    (test_acceptance.py:247-269) on 2^20 'mixed' quaternions normalized on the GPU: the
    unit and general forms agree within 16u per entry, and R^T R - I and det R - 1 stay
    within 64u.  The reference evaluates both budgets exactly with Fractions; here they
    use 64-bit-mantissa long doubles, whose own error (< 2^-60) is far below 64u."""
    d = fn.preset("double")
    x = torch.empty((1 << 20, 4), dtype=torch.float64, device="cuda")
    workloads.generate_regime_device("mixed", x, seed=66)
    q = fn.normalize4(d, x).unit
    Ru, Rg = fn.rotation_unit(q), fn.rotation_general(q)
    assert ((Ru - Rg).abs() <= 16 * U64).all()
    R = Ru.cpu().numpy().astype(np.longdouble)
    gram = np.einsum("nki,nkj->nij", R, R) - np.eye(3, dtype=np.longdouble)
    assert np.abs(gram).max() <= 64 * U64
    det = (R[:, 0, 0] * (R[:, 1, 1] * R[:, 2, 2] - R[:, 1, 2] * R[:, 2, 1])
           - R[:, 0, 1] * (R[:, 1, 0] * R[:, 2, 2] - R[:, 1, 2] * R[:, 2, 0])
           + R[:, 0, 2] * (R[:, 1, 0] * R[:, 2, 1] - R[:, 1, 1] * R[:, 2, 0]))
    assert np.abs(det - 1).max() <= 64 * U64
