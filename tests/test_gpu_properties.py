"""Property tests of the reference suite (tests/test_scale.py:82-186,
tests/test_normalize.py:77-145), evaluated on 2^20-row batches through the GPU kernels
instead of a few hundred hypothesis examples through scalar calls."""

import math

import numpy as np
import pytest

import paper_1606_06508_b200 as fn

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

N = 1 << 20


def _full_range(n, dim, single, seed):
    """Nonzero finite values, log-uniform over the whole format incl. subnormals (the
    st_f64 / st_f32 bit-pattern strategies of test_scale.py:23-28), random signs."""
    rng = np.random.default_rng(seed)
    if single:
        bits = rng.integers(1, 0x7F7FFFFF, (n, dim), dtype=np.uint32)
        x = bits.view(np.float32)
    else:
        bits = rng.integers(1, 0x7FEFFFFFFFFFFFFF, (n, dim), dtype=np.uint64)
        x = bits.view(np.float64)
    return x * np.where(rng.random((n, dim)) < 0.5, -1, 1).astype(x.dtype)


@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("dim", [2, 3, 4])
def test_scale_range_and_inverse(cuda_dev, prec, dim):
    """max |scaled| lands in [tau_min, tau_max]; inv is 1, 1/sigma_min or 1/sigma_max,
    a power of two (test_scale.py:82-98, :133-138)."""
    p = fn.preset(prec)
    x = torch.from_numpy(_full_range(N, dim, prec == "single", seed=dim)).to(cuda_dev)
    out = getattr(fn, f"scale{dim}")(p, x)
    top = out.scaled.abs().amax(dim=1).double().cpu().numpy()
    inv = out.inv_sigma.double().cpu().numpy()
    assert (top >= p.tau_min).all() and (top <= p.tau_max).all()
    allowed = np.array([1.0, 1.0 / p.sigma_min, 1.0 / p.sigma_max])
    assert np.isin(inv, allowed).all()
    m, _ = np.frexp(inv)
    assert (m == 0.5).all()


@pytest.mark.parametrize("prec", ["double", "single"])
@pytest.mark.parametrize("dim", [2, 3, 4])
def test_scale_idempotent(cuda_dev, prec, dim):
    """Scaling scaled rows is the identity with inv 1 (test_scale.py:100-106)."""
    p = fn.preset(prec)
    x = torch.from_numpy(_full_range(N, dim, prec == "single", seed=10 + dim)).to(cuda_dev)
    first = getattr(fn, f"scale{dim}")(p, x)
    again = getattr(fn, f"scale{dim}")(p, first.scaled.contiguous())
    torch.cuda.synchronize()
    assert bool((again.inv_sigma == 1).all())
    w = torch.int64 if prec == "double" else torch.int32
    assert bool((again.scaled.view(w) == first.scaled.view(w)).all())


def test_scale_exact_for_normal_results(cuda_dev):
    """sigma*x is exact wherever the exact product is normal (test_scale.py:108-122)."""
    p = fn.preset("double")
    xh = _full_range(N, 3, False, seed=31)
    out = fn.scale3(p, torch.from_numpy(xh).to(cuda_dev))
    s = out.scaled.cpu().numpy()
    sigma = 1.0 / out.inv_sigma.cpu().numpy()
    ex = np.frexp(np.abs(xh))[1] - 1 + np.round(np.log2(sigma))[:, None].astype(int)
    normal = (ex >= -1022) & (ex <= 1023)
    # in the normal range the product is a pure exponent shift: s == ldexp(x, log2 sigma)
    want = np.ldexp(xh, np.round(np.log2(sigma)).astype(int)[:, None])
    assert normal.mean() > 0.8
    assert (s[normal] == want[normal]).all()


def test_downscaled_component_can_flush_to_zero(cuda_dev):
    """A min-normal next to a just-over-tau_max component (test_scale.py:124-131)."""
    p = fn.preset("double")
    big = math.nextafter(p.tau_max, math.inf)
    out = fn.scale2(p, torch.tensor([[p.nu, big]], dtype=torch.float64, device=cuda_dev))
    assert out.inv_sigma.item() == 1.0 / p.sigma_max
    assert out.scaled[0, 0].item() == 0.0 and out.scaled[0, 1].item() == p.sigma_max * big


@pytest.mark.parametrize("dim", [2, 3, 4])
@pytest.mark.parametrize("prec", ["double", "single"])
def test_nan_contracts(cuda_dev, dim, prec):
    """NaN in any position: scale keeps a NaN component and never takes the zero branch;
    normalize returns NaN length and unit; clean rows never produce NaN
    (test_scale.py:144-169, test_normalize.py:128-145)."""
    p = fn.preset(prec)
    dt = torch.float64 if prec == "double" else torch.float32
    fills = [0.0, -0.0, 1.0, -2.5, 2.0 ** -1074 if prec == "double" else 2.0 ** -149,
             p.tau_min, 2.0 ** 600 if prec == "double" else 2.0 ** 70]
    rows = []
    for i in range(dim):
        for f in fills:
            r = [f] * dim
            r[i] = math.nan
            rows.append(r)
    x = torch.tensor(rows, dtype=dt, device=cuda_dev)
    sc = getattr(fn, f"scale{dim}")(p, x)
    assert bool(torch.isnan(sc.scaled).any(dim=1).all()) and bool((sc.inv_sigma != 0).all())
    nz = getattr(fn, f"normalize{dim}")(p, x)
    assert bool(torch.isnan(nz.length).all()) and bool(torch.isnan(nz.unit).all())
    clean = torch.tensor([[f] * dim for f in fills], dtype=dt, device=cuda_dev)
    nc = getattr(fn, f"normalize{dim}")(p, clean)
    assert not bool(torch.isnan(nc.length).any()) and not bool(torch.isnan(nc.unit).any())


def test_inf_pass_through_and_signed_zeros(cuda_dev):
    """Inf input: sigma_max branch, r = inf (test_scale.py:172-176); all -0 rows give +0
    outputs (:178-181); a zero component keeps its sign."""
    p = fn.preset("double")
    x = torch.tensor([[math.inf, 1.0, -2.0], [-0.0, -0.0, -0.0], [-3.0, 0.0, -0.0]],
                     dtype=torch.float64, device=cuda_dev)
    s = fn.scale3(p, x)
    assert s.inv_sigma[0].item() == 1.0 / p.sigma_max and s.scaled[0, 0].item() == math.inf
    assert s.inv_sigma[1].item() == 0.0
    out = fn.normalize3(p, x)
    u = out.unit.cpu().numpy()
    assert out.length[0].item() == math.inf and math.isnan(u[0, 0]) and u[0, 1] == 0.0
    assert np.signbit(u[0, 2])
    assert out.length[1].item() == 0.0 and not np.signbit(u[1]).any()
    assert u[2].tolist() == [-1.0, 0.0, -0.0] and np.signbit(u[2, 2]) and not np.signbit(u[2, 1])
