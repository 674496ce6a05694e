"""GPU parity at the BASELINE.json configs' full sizes.

Every config is generated in HBM by the seeded generator, run through the batched C ABI,
and compared bit for bit with the oracle over EVERY row (chunked).  Size-independent
properties are checked on the device as well: the device generator equals the host
restatement, the row-class counters match the advertised frequencies, norm == length,
and for the NaN/Inf-free configs the reference timing-loop checksum over the GPU outputs
equals the oracle (and, where built, the reference's own compiled loop).
"""

import numpy as np
import pytest

from gpu_helpers import compare_chunked, to_np

import oracle
import paper_1606_06508_b200 as fn
from paper_1606_06508_b200 import _lib, workloads

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _gen(cfg, dev, n=None):
    c = workloads.CONFIGS[cfg]
    n = c.rows if n is None else n
    dt = torch.float64 if c.dtype == "float64" else torch.float32
    x = torch.empty((n, c.dim), dtype=dt, device=dev)
    workloads.generate_device(cfg, x)
    return x


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_device_generator_matches_host(cuda_dev, cfg):
    c = workloads.CONFIGS[cfg]
    x = _gen(cfg, cuda_dev, n=1 << 20)
    lo = 777
    dev_rows = to_np(x[lo:lo + 100_000])
    host_rows = workloads.host_rows(cfg, lo, 100_000)
    if cfg == 3:  # libm vs CUDA transcendental: same distribution, not same bits
        assert np.allclose(dev_rows, host_rows, rtol=1e-12, atol=1e-12)
    else:
        assert (dev_rows.view(np.uint8) == host_rows.view(np.uint8)).all()
    # a shard generated at an offset equals the same rows of the full array
    y = torch.empty((1000, c.dim), dtype=x.dtype, device=cuda_dev)
    workloads.generate_device(cfg, y, row0=5000)
    assert (to_np(y).view(np.uint8) == to_np(x[5000:6000]).view(np.uint8)).all()


def _stats(x, prec):
    counts = torch.zeros(6, dtype=torch.uint64, device=x.device)
    workloads.row_stats_device(x, fn.kernel_args(fn.preset(prec)), counts)
    return to_np(counts.to(torch.int64))


def test_cfg1_scaling_full(cuda_dev):
    p = fn.preset("double")
    ka = np.array(fn.kernel_args(p))
    x = _gen(1, cuda_dev)
    res = fn.normalize3(p, x)
    torch.cuda.synchronize()
    bad, first = compare_chunked(_lib.OP_NORMALIZE, x, res.length, res.unit, None, ka)
    assert bad == 0, first
    st = _stats(x, "double")
    assert st[5] == x.shape[0]  # every row of U[-1,1]^3 is in the sigma = 1 band


def _loop_checksum_from_outputs(head, body) -> float:
    """acc += ((r + u1) + u2) + ... in the reference loop's order (_kernels.pyx:666-670)."""
    term = to_np(head).astype(np.float64)
    b = to_np(body).astype(np.float64)
    for k in range(b.shape[1]):
        term = term + b[:, k]
    return float(np.add.accumulate(np.concatenate(([0.0], term)))[-1])


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_loop_checksum_full_size(cuda_dev, cfg):
    """GPU outputs summed in the reference loop's order == the reference loop itself."""
    c = workloads.CONFIGS[cfg]
    p = fn.preset("double")
    ka = fn.kernel_args(p)
    x = _gen(cfg, cuda_dev)
    res = {2: fn.normalize2, 3: fn.normalize3, 4: fn.normalize4}[c.dim](p, x)
    torch.cuda.synchronize()
    got = _loop_checksum_from_outputs(res.length, res.unit)
    xh = to_np(x)
    n = xh.shape[0]
    mask = (1 << int(np.ceil(np.log2(n)))) - 1
    want = oracle.loop(oracle.ALGO_SCALING, xh, n, mask, ka)
    assert got == want
    ref = oracle.ref_module()
    if ref is not None:
        loop = getattr(ref, f"loop_scaling{c.dim}_f64")
        assert got == loop(np.ascontiguousarray(xh.reshape(-1)), n, mask, *ka)


def test_cfg2_scaling_and_quotient_full(cuda_dev):
    p = fn.preset("double")
    ka = np.array(fn.kernel_args(p))
    x = _gen(2, cuda_dev)
    res = fn.normalize2(p, x)
    torch.cuda.synchronize()
    bad, first = compare_chunked(_lib.OP_NORMALIZE, x, res.length, res.unit, None, ka)
    assert bad == 0, first
    del res
    q = fn.quotient2(x)
    torch.cuda.synchronize()
    bad, first = compare_chunked(_lib.OP_QUOTIENT, x, q.length, q.unit)
    assert bad == 0, first
    st = _stats(x, "double")
    assert abs(st[2] / x.shape[0] - 0.01) < 0.0005      # 1 % zero rows
    assert st[3] > 0 and st[4] > 0 and st[5] > 0        # all three scaling classes occur


def _two_prod_sq(a):
    """a*a as hi + lo exactly (Dekker's split; |a| far from overflow)."""
    p = a * a
    c = 134217729.0 * a
    ah = c - (c - a)
    al = a - ah
    return p, ((ah * ah - p) + 2.0 * ah * al) + al * al


def _two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def _dd_sum_squares(x):
    """Double-double sum of squares of each row of x (float64 [n, k])."""
    hi, lo = _two_prod_sq(x[:, 0])
    for k in range(1, x.shape[1]):
        p, e = _two_prod_sq(x[:, k])
        hi, t = _two_sum(hi, p)
        lo = lo + t + e
    return _two_sum(hi, lo)


def test_cfg3_quaternion_sq_full(cuda_dev):
    p = fn.preset("double")
    ka = np.array(fn.kernel_args(p))
    x = _gen(3, cuda_dev)
    res = fn.normalize4_sq(p, x)
    torch.cuda.synchronize()
    bad, first = compare_chunked(_lib.OP_NORMALIZE_SQ, x, res.length, res.unit,
                                 res.squared_length, ka)
    assert bad == 0, first
    # squared length vs exact rational sum of squares on a sample: relative error
    # <= (n + 1) u (n - 1 additions + n squarings, each <= u, one exact ldexp)
    from fractions import Fraction

    idx = np.random.default_rng(3).integers(0, x.shape[0], 2000)
    xs = to_np(x[torch.from_numpy(idx).to(cuda_dev)])
    sq = to_np(res.squared_length[torch.from_numpy(idx).to(cuda_dev)])
    u = Fraction(1, 2 ** 53)
    for row, s in zip(xs.tolist(), sq.tolist()):
        exact = sum(Fraction(v) ** 2 for v in row)
        assert abs(Fraction(s) - exact) <= 5 * u * exact
    # ... and on every row of the config (2^27) against a double-double sum of squares
    # (Dekker products, two-sum accumulation: relative error ~2^-100, far inside 5u)
    worst = 0.0
    for lo in range(0, x.shape[0], 1 << 23):
        xr = to_np(x[lo:lo + (1 << 23)])
        sr = to_np(res.squared_length[lo:lo + (1 << 23)])
        hi_s, lo_s = _dd_sum_squares(xr)
        d = (sr - hi_s) - lo_s  # sr - hi_s is exact (Sterbenz)
        rel = np.abs(d) / hi_s
        worst = max(worst, float(rel.max()))
    assert worst <= 5 * 2.0 ** -53 * (1 + 2.0 ** -40), worst


def test_cfg4_f32_full(cuda_dev):
    p = fn.preset("single")
    ka = np.array(fn.kernel_args(p))
    x = _gen(4, cuda_dev)
    res = fn.normalize3(p, x)
    torch.cuda.synchronize()
    bad, first = compare_chunked(_lib.OP_NORMALIZE, x, res.length, res.unit, None, ka)
    assert bad == 0, first
    st = _stats(x, "single")
    n = x.shape[0]
    assert abs(st[2] / n - 0.001) < 0.0001          # zero rows
    assert abs((st[0] + st[1]) / n - 0.0001) < 0.00002  # NaN / Inf rows
    nan_rows = to_np(torch.isnan(res.length)).sum()
    assert nan_rows == st[0]                         # exact NaN classification
    inf_rows = to_np(torch.isinf(res.length)).sum()
    assert inf_rows >= st[1]                         # inf rows -> r = inf (and warranted overflow)


def test_cfg5_full_2pow30(cuda_dev):
    p = fn.preset("double")
    ka = np.array(fn.kernel_args(p))
    x = _gen(5, cuda_dev)
    res = fn.normalize3(p, x)
    torch.cuda.synchronize()
    bad, first = compare_chunked(_lib.OP_NORMALIZE, x, res.length, res.unit, None, ka,
                                 chunk=1 << 26)
    assert bad == 0, first
    r = fn.norm3(p, x)
    torch.cuda.synchronize()
    assert bool((r.view(torch.int64) == res.length.view(torch.int64)).all())
    st = _stats(x, "double")
    n = x.shape[0]
    assert st[0] == 0 and st[1] == 0 and st[2] == 0
    # sigma_min path: all-subnormal rows (0.5 %) plus normal rows whose three exponents
    # all fall below -482: 0.99 * (538/2041)^3 = 1.813 %
    assert abs(st[3] / n - (0.005 + 0.99 * (538 / 2041) ** 3)) < 0.0005
    assert st[4] > 0.005 * n                           # near-DBL_MAX rows are sigma_max rows
