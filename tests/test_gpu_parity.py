"""GPU parity: every kernel family, both precisions, through the C ABI, bit for bit
against the reference's golden vectors and the pinned oracle (reference rule: NaN
matches NaN, everything else bit-equal including the sign of zero)."""

import math

import numpy as np
import pytest

from conftest import FAMILIES, SCALING, kernel_name, same_scalar
from gpu_helpers import compare_chunked

import oracle
import paper_1606_06508_b200 as fn
from paper_1606_06508_b200 import _backend, _cuda_kernels, _lib

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

OPS = {"scale": _lib.OP_SCALE, "normalize": _lib.OP_NORMALIZE, "norm": _lib.OP_NORM,
       "naive": _lib.OP_NAIVE, "quotient": _lib.OP_QUOTIENT,
       "quotient3_fast": _lib.OP_QUOTIENT3_FAST}
PREC = {"f64": "double", "f32": "single"}


def _base(fam, dim):
    return "quotient3_fast" if fam == "quotient3_fast" else f"{fam}{dim}"


def _golden_rows(golden, prec, dim):
    x = golden[f"{prec}_{dim}_x"]
    return x.astype(np.float32) if prec == "f32" else x


def _as_table(res):
    h = res.head.cpu().numpy() if hasattr(res.head, "cpu") else res.head
    if res.body is None:
        return h[:, None].astype(np.float64)
    b = res.body.cpu().numpy() if hasattr(res.body, "cpu") else res.body
    return np.concatenate([h[:, None], b], axis=1).astype(np.float64)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("dim", [2, 3, 4])
@pytest.mark.parametrize("where", ["device", "device_unaligned", "host"])
def test_golden_vectors(golden, cuda_dev, prec, dim, where):
    x = _golden_rows(golden, prec, dim)
    ka = golden[f"{prec}_ka"]
    for fam in FAMILIES[dim]:
        k = _cuda_kernels.batch_kernel(_base(fam, dim), prec)
        if where == "host":
            res = k(x, ka if fam in SCALING else None)
        elif where == "device":
            res = k(torch.from_numpy(x).to(cuda_dev), ka if fam in SCALING else None)
        else:  # one-row offset: 8/16/24/32-byte aligned rows -> per-row kernel path
            big = torch.from_numpy(np.concatenate([x[:1], x])).to(cuda_dev)
            res = k(big[1:], ka if fam in SCALING else None)
        torch.cuda.synchronize()
        got = _as_table(res)
        ref = golden[f"{prec}_{kernel_name(fam, dim, prec)}"]
        ok = oracle.same(got, ref)
        bad = np.argwhere(~ok)
        assert ok.all(), (fam, where, x[bad[0][0]], got[bad[0][0]], ref[bad[0][0]])


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_scalar_registry_calls(golden, cuda_dev, prec):
    """The reference's scalar signatures, resolved through the registry, on the GPU."""
    ka = tuple(golden[f"{prec}_ka"])
    for dim in (2, 3, 4):
        x = golden[f"{prec}_{dim}_x"]
        idx = np.linspace(0, len(x) - 1, 12).astype(int)
        for fam in FAMILIES[dim]:
            k = _backend.scalar_kernel(_base(fam, dim), PREC[prec])
            ref = golden[f"{prec}_{kernel_name(fam, dim, prec)}"]
            for i in idx:
                row = [float(v) for v in x[i]]
                out = k(*ka, *row) if fam in SCALING else k(*row)
                out = out if isinstance(out, tuple) else (out,)
                assert all(same_scalar(a, b) for a, b in zip(out, ref[i])), (fam, row, out, ref[i])


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("dim", [2, 3, 4])
def test_loop_checksums_through_gpu(golden, cuda_dev, prec, dim):
    ka = tuple(golden[f"{prec}_ka"])
    x = _golden_rows(golden, prec, dim)[:8]
    flat = np.ascontiguousarray(x.reshape(-1))
    algos = ["scaling", "quotient", "naive"] + (["quotient_fast"] if dim == 3 else [])
    for algo in algos:
        loop = _backend.loop_kernel(_backend.loop_base(algo, dim), PREC[prec])
        got = loop(flat, 37, 7, *ka)
        want = golden[f"{prec}_{dim}_loop_{algo}"][0]
        assert got == want or (np.isnan(got) and np.isnan(want)), (algo, got, want)
    got = _backend.loop_kernel(f"loop_empty{dim}", PREC[prec])(flat, 37, 7)
    assert got == golden[f"{prec}_{dim}_loop_empty"][0]


def _random_rows(n, dim, single, seed):
    rng = np.random.default_rng(seed)
    lo, hi = (-149, 128) if single else (-1074, 1024)
    x = np.ldexp(1.0 + rng.random((n, dim)), rng.integers(lo, hi, (n, dim)))
    x *= rng.integers(0, 2, (n, dim)) * 2 - 1
    # sprinkle specials: zeros, signed zeros, inf, nan, in every position
    sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan])
    mask = rng.random((n, dim)) < 0.02
    x[mask] = rng.choice(sp, mask.sum())
    zero_rows = rng.random(n) < 0.01
    x[zero_rows] = rng.choice([0.0, -0.0], (zero_rows.sum(), dim))
    with np.errstate(over="ignore"):
        return x.astype(np.float32) if single else x


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("dim", [2, 3, 4])
@pytest.mark.parametrize("aligned", [True, False])
def test_random_full_range_vs_oracle(cuda_dev, prec, dim, aligned):
    n = (1 << 20) + 37
    x = _random_rows(n + 1, dim, prec == "f32", seed=dim * 10 + (prec == "f32"))
    xd = torch.from_numpy(x).to(cuda_dev)
    xd = xd[:n] if aligned else xd[1:]
    ka = np.array(fn.kernel_args(fn.preset(PREC[prec])))
    for fam in FAMILIES[dim] + ["normalize_sq"]:
        base = f"normalize{dim}_sq" if fam == "normalize_sq" else _base(fam, dim)
        op = _lib.OP_NORMALIZE_SQ if fam == "normalize_sq" else OPS[fam]
        takes = fam in SCALING or fam == "normalize_sq"
        res = _cuda_kernels.batch_kernel(base, prec)(xd, ka if takes else None)
        torch.cuda.synchronize()
        bad, first = compare_chunked(op, xd, res.head, res.body, res.sq, ka if takes else None)
        assert bad == 0, (fam, prec, dim, aligned, bad, first)


@pytest.mark.parametrize("n", [1, 2, 3, 15, 16, 17, 255, 256, 257, 511, 512, 513, 1023, 4097, 100_003])
def test_tail_sizes(cuda_dev, n):
    p = fn.preset("double")
    ka = np.array(fn.kernel_args(p))
    x = torch.from_numpy(_random_rows(n, 3, False, seed=n)).to(cuda_dev)
    res = fn.normalize3(p, x)
    torch.cuda.synchronize()
    bad, first = compare_chunked(_lib.OP_NORMALIZE, x, res.length, res.unit, None, ka)
    assert bad == 0, first
    ps = fn.preset("single")
    x32 = torch.from_numpy(_random_rows(n, 2, True, seed=n + 1)).to(cuda_dev)
    r = fn.norm2(ps, x32)
    torch.cuda.synchronize()
    bad, first = compare_chunked(_lib.OP_NORM, x32, r, None, None, np.array(fn.kernel_args(ps)))
    assert bad == 0, first


def test_out_buffers_and_noncontiguous(cuda_dev):
    p = fn.preset("double")
    x = torch.from_numpy(_random_rows(5000, 4, False, seed=3)).to(cuda_dev)
    r = torch.empty(5000, dtype=torch.float64, device=cuda_dev)
    u = torch.empty((5000, 4), dtype=torch.float64, device=cuda_dev)
    res = fn.normalize4(p, x, out=(r, u))
    assert res.length.data_ptr() == r.data_ptr() and res.unit.data_ptr() == u.data_ptr()
    ref = fn.normalize4(p, x.cpu().numpy())
    torch.cuda.synchronize()
    assert oracle.same(r.cpu().numpy(), ref.length).all()
    assert oracle.same(u.cpu().numpy(), ref.unit).all()
    # a strided view (every other row) is made contiguous internally
    xs = x[::2]
    res2 = fn.normalize4(p, xs)
    torch.cuda.synchronize()
    assert oracle.same(res2.unit.cpu().numpy(), ref.unit[::2]).all()
    with pytest.raises(ValueError):
        fn.normalize4(p, x, out=(r[:10], u))


def _padded(x_np, ldx, dev, fill=np.nan, offset=0):
    """Rows of x as a [N, dim] view into [N, ldx] records (extra elements = fill), the
    storage shifted by `offset` elements."""
    n, dim = x_np.shape
    buf = torch.full((offset + n * ldx,), fill, dtype=torch.from_numpy(x_np).dtype, device=dev)
    rec = buf[offset:].view(n, ldx)
    rec[:, :dim] = torch.from_numpy(x_np).to(dev)
    return rec[:, :dim]


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("n", [1, 255, 256, 257, 513, 4099, (1 << 20) + 3])
def test_padded_records_xyz_in_xyzw(cuda_dev, prec, n):
    """xyz out of xyzw records (fn_run_ld, ldx 4): the bulk-copy kernel stages whole
    records; every family, bit for bit against the oracle; padding never read into a row."""
    single = prec == "f32"
    x = _random_rows(n, 3, single, seed=n + single)
    xv = _padded(x, 4, cuda_dev)
    assert n == 1 or not xv.is_contiguous()  # torch calls one row contiguous whatever its stride
    ka = np.array(fn.kernel_args(fn.preset(PREC[prec])))
    for fam in FAMILIES[3] + ["normalize_sq"]:
        base = "normalize3_sq" if fam == "normalize_sq" else _base(fam, 3)
        op = _lib.OP_NORMALIZE_SQ if fam == "normalize_sq" else OPS[fam]
        takes = fam in SCALING or fam == "normalize_sq"
        res = _cuda_kernels.batch_kernel(base, prec)(xv, ka if takes else None)
        torch.cuda.synchronize()
        bad, first = compare_chunked(op, xv, res.head, res.body, res.sq, ka if takes else None)
        assert bad == 0, (fam, prec, n, bad, first)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("offset_rows", [1, 2, 3])
def test_misaligned_rows_bulk_path(cuda_dev, prec, offset_rows):
    """Rows whose storage starts off a 16-byte boundary (x[k:] of a dense array) run the
    bulk-copy kernel from the boundary below each tile: every family, sizes around the
    tile and the end-of-array reach, bit for bit against the oracle."""
    single = prec == "f32"
    tr = 512 if single else 256
    ka = np.array(fn.kernel_args(fn.preset(PREC[prec])))
    for n in (tr - 1, tr, tr + 1, 2 * tr - 1, 2 * tr + 5, 100_003):
        x = _random_rows(n + offset_rows, 3, single, seed=n * 7 + offset_rows + single)
        xd = torch.from_numpy(x).to(cuda_dev)[offset_rows:]
        for fam in FAMILIES[3] + ["normalize_sq"]:
            base = "normalize3_sq" if fam == "normalize_sq" else _base(fam, 3)
            op = _lib.OP_NORMALIZE_SQ if fam == "normalize_sq" else OPS[fam]
            takes = fam in SCALING or fam == "normalize_sq"
            res = _cuda_kernels.batch_kernel(base, prec)(xd, ka if takes else None)
            torch.cuda.synchronize()
            bad, first = compare_chunked(op, xd, res.head, res.body, res.sq, ka if takes else None)
            assert bad == 0, (fam, prec, offset_rows, n, first)


def test_strided_rows_other_layouts(cuda_dev):
    """Other row strides (per-row kernel), a misaligned padded view, a last record that
    ends at its third element, rotation apply on padded vectors, and outputs overlapping
    strided input (gathered first)."""
    p = fn.preset("double")
    ka = np.array(fn.kernel_args(p))
    n = 5003
    for dim, ldx in ((2, 3), (3, 5), (4, 6), (3, 4)):
        x = _random_rows(n, dim, False, seed=ldx * 7 + dim)
        for offset in (0, 1):
            xv = _padded(x, ldx, cuda_dev, offset=offset)
            res = _cuda_kernels.batch_kernel(f"normalize{dim}", "f64")(xv, ka)
            torch.cuda.synchronize()
            bad, first = compare_chunked(_lib.OP_NORMALIZE, xv, res.head, res.body, None, ka)
            assert bad == 0, (dim, ldx, offset, first)
    # storage ends right after the last row's z: the last row must not ride in a tile
    x = _random_rows(4 * 256 + 1, 3, False, seed=77)
    m = x.shape[0]
    buf = torch.full(((m - 1) * 4 + 3,), np.nan, dtype=torch.float64, device=cuda_dev)
    xv = buf.as_strided((m, 3), (4, 1))
    xv.copy_(torch.from_numpy(x))
    res = fn.normalize3(p, xv)
    torch.cuda.synchronize()
    bad, first = compare_chunked(_lib.OP_NORMALIZE, xv, res.length, res.unit, None, ka)
    assert bad == 0, first
    # RotationMatrix.apply over padded vectors
    R = fn.rotation_unit((0.5, 0.5, 0.5, 0.5))
    v = _random_rows(3001, 3, False, seed=5)
    v[~np.isfinite(v)] = 1.0
    got = R.apply(_padded(v, 4, cuda_dev))
    want = R.apply(torch.from_numpy(v).to(cuda_dev))
    torch.cuda.synchronize()
    assert oracle.same(got.cpu().numpy(), want.cpu().numpy()).all()
    # outputs overlapping the strided rows: gathered before the launch
    x = _random_rows(4096, 3, False, seed=8)
    rec = torch.zeros((4096, 4), dtype=torch.float64, device=cuda_dev)
    rec[:, :3] = torch.from_numpy(x).to(cuda_dev)
    u = rec.view(-1)[: 4096 * 3].view(4096, 3)
    r = torch.empty(4096, dtype=torch.float64, device=cuda_dev)
    fn.normalize3(p, rec[:, :3], out=(r, u))
    torch.cuda.synchronize()
    h, b, _ = oracle.run(_lib.OP_NORMALIZE, x, ka)
    assert oracle.same(r.cpu().numpy(), h).all() and oracle.same(u.cpu().numpy(), b).all()


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("n", [1, 300, 4099, 3_000_001])
@pytest.mark.parametrize("pinned", [False, True])
def test_host_padded_records(cuda_dev, prec, n, pinned):
    """Host (numpy) xyz-of-xyzw rows through fn_host_run_ld: records cross PCIe as they
    are (small zero-copy path, staged pipeline, page-locked caller buffers), every
    family bit for bit against the oracle; 3e6 rows span several pipeline chunks."""
    single = prec == "f32"
    x = _random_rows(n, 3, single, seed=n * 3 + single)
    rec = fn.host_empty((n, 4), dtype=x.dtype) if pinned else np.empty((n, 4), dtype=x.dtype)
    rec[:, 3] = np.nan
    rec[:, :3] = x
    xv = rec[:, :3]
    ka = np.array(fn.kernel_args(fn.preset(PREC[prec])))
    for fam in FAMILIES[3] + ["normalize_sq"]:
        base = "normalize3_sq" if fam == "normalize_sq" else _base(fam, 3)
        op = _lib.OP_NORMALIZE_SQ if fam == "normalize_sq" else OPS[fam]
        takes = fam in SCALING or fam == "normalize_sq"
        res = _cuda_kernels.batch_kernel(base, prec)(xv, ka if takes else None)
        h, b, q = oracle.run(op, x, ka if takes else None, threads=8)
        assert oracle.same(res.head, h).all(), (fam, prec, n)
        if b is not None:
            assert oracle.same(res.body, b).all(), (fam, prec, n)
        if q is not None:
            assert oracle.same(res.sq, q).all(), (fam, prec, n)
    # other strides and a CPU tensor view
    x2 = _random_rows(5000, 2, False, seed=4)
    r5 = np.zeros((5000, 5))
    r5[:, 1:3] = x2
    got = fn.normalize2(fn.preset("double"), r5[:, 1:3])
    h, b, _ = oracle.run(_lib.OP_NORMALIZE, x2, np.array(fn.kernel_args(fn.preset("double"))))
    assert oracle.same(got.length, h).all() and oracle.same(got.unit, b).all()
    t = torch.from_numpy(r5)[:, 1:3]
    got = fn.normalize2(fn.preset("double"), t)
    assert oracle.same(got.length.numpy(), h).all() and oracle.same(got.unit.numpy(), b).all()


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_run_many_segments(cuda_dev, prec):
    """fn_run_many: every family over a list of arrays of mixed sizes (empty, one row,
    around the tile, large), one of them off the 16-byte grid (launched on its own), and
    60 arrays (two launches of at most 48) equals one call per array bit for bit."""
    from paper_1606_06508_b200 import batch

    single = prec == "f32"
    ka = np.array(fn.kernel_args(fn.preset(PREC[prec])))
    sizes = [0, 1, 255, 256, 257, 511, 513, 5000, 100_003]
    for dim in (2, 3, 4):
        xs = [torch.from_numpy(_random_rows(n, dim, single, seed=n + dim)).to(cuda_dev) for n in sizes]
        big = torch.from_numpy(_random_rows(3001, dim, single, seed=99)).to(cuda_dev)
        xs.append(big[1:])  # off the 16-byte grid for dim 3 (and f32 dim 2)
        ops = [OPS[f] for f in FAMILIES[dim]] + [_lib.OP_NORMALIZE_SQ]
        for op in ops:
            k = ka if op in (_lib.OP_SCALE, _lib.OP_NORMALIZE, _lib.OP_NORM, _lib.OP_NORMALIZE_SQ) else None
            got = batch.run_many(op, dim, xs, k)
            for x, g in zip(xs, got):
                want = batch.run(op, dim, x, k)
                for a, b in ((g.head, want.head), (g.body, want.body), (g.sq, want.sq)):
                    if b is not None:
                        assert oracle.same(a.cpu().numpy(), b.cpu().numpy()).all(), (prec, dim, op, x.shape)
    # more arrays than one launch holds, through the public API
    p = fn.preset(PREC[prec])
    xs = [torch.from_numpy(_random_rows(300 + 37 * j, 3, single, seed=j)).to(cuda_dev) for j in range(60)]
    outs = fn.normalize_many(p, xs)
    lens = fn.norm_many(p, xs)
    for x, o, r in zip(xs, outs, lens):
        w = fn.normalize3(p, x)
        assert oracle.same(o.length.cpu().numpy(), w.length.cpu().numpy()).all()
        assert oracle.same(o.unit.cpu().numpy(), w.unit.cpu().numpy()).all()
        assert oracle.same(r.cpu().numpy(), w.length.cpu().numpy()).all()
    # host arrays fall back to one host-path call each
    hs = [x.cpu().numpy() for x in xs[:3]]
    for h, o in zip(hs, fn.normalize_many(p, hs)):
        assert oracle.same(o.unit, fn.normalize3(p, h).unit).all()


def test_norm_equals_normalize_length(cuda_dev):
    for prec, dt in (("double", torch.float64), ("single", torch.float32)):
        p = fn.preset(prec)
        x = torch.from_numpy(_random_rows(1 << 20, 3, prec == "single", seed=9)).to(cuda_dev)
        a = fn.norm3(p, x)
        b = fn.normalize3(p, x).length
        torch.cuda.synchronize()
        assert oracle.same(a.cpu().numpy(), b.cpu().numpy()).all()


def test_public_api_examples(cuda_dev):
    """Known answers of the reference tests, through the batched device path."""
    d = fn.preset("double")
    x = torch.tensor([[3.0, 4.0, 0.0, 0.0], [1.0, 1.0, 1.0, 1.0], [0.0, 0.0, 0.0, 0.0],
                      [2.0 ** -1074, 0.0, 0.0, 0.0]], dtype=torch.float64, device=cuda_dev)
    res = fn.normalize4(d, x)
    torch.cuda.synchronize()
    assert res.length.tolist() == [5.0, 2.0, 0.0, 2.0 ** -1074]
    assert res.unit[1].tolist() == [0.5] * 4
    assert res.unit[2].tolist() == [0.0, 0.0, 0.0, 1.0]
    q = fn.quotient4(x)
    torch.cuda.synchronize()
    assert q.unit[2].tolist() == [0.0] * 4 and q.length[1].item() == 2.0
    nv = fn.naive_normalize2(torch.tensor([[2.0 ** -600, 0.0]], dtype=torch.float64, device=cuda_dev))
    torch.cuda.synchronize()
    assert nv.length.item() == 0.0 and nv.unit[0, 0].item() == float("inf")
    # scalar signatures keep working (one launch per call)
    assert fn.normalize2(d, 3.0, 4.0).length == 5.0
    assert fn.norm3(d, 2.0, 10.0, 11.0) == 15.0
    assert fn.quotient3_robust(0.0, 0.0, 0.0) == (0.0, (0.0, 0.0, 0.0))
    assert fn.scale2(d, 2.0 ** -500, 0.0) == (2.0 ** -592, (2.0 ** 92, 0.0))


@pytest.mark.parametrize("dtype", [_lib.F64, _lib.F32])
def test_division_selftest(cuda_dev, dtype):
    """The shared-divisor division equals IEEE division bit for bit on 2^28 pairs."""
    out = torch.zeros(3, dtype=torch.int64, device=cuda_dev)
    for seed in (1, 2):
        out.zero_()
        rc = _lib.lib().fn_selftest_div(dtype, seed, 1 << 27, out.data_ptr(),
                                        torch.cuda.current_stream().cuda_stream)
        _lib.check(rc, "fn_selftest_div")
        torch.cuda.synchronize()
        bad, a, b = out.tolist()
        assert bad == 0, (dtype, seed, bad, hex(a & (2**64 - 1)), hex(b & (2**64 - 1)))


@pytest.mark.parametrize("regime", ["normal", "subnormal", "huge", "mixed", "unit-ish"])
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_reference_regimes(cuda_dev, regime, prec):
    """The reference harness's input regimes (bench.py:146-207), every family, 2^20 rows."""
    from paper_1606_06508_b200 import workloads

    dt = torch.float64 if prec == "f64" else torch.float32
    dtype = "float64" if prec == "f64" else "float32"
    ka = np.array(fn.kernel_args(fn.preset(PREC[prec])))
    for dim in (2, 3, 4):
        n = (1 << 20) + 3
        x = torch.empty((n, dim), dtype=dt, device=cuda_dev)
        workloads.generate_regime_device(regime, x, seed=11)
        host = workloads.regime_rows(regime, dim, dtype, 1000, 5000, seed=11)
        dev = x[1000:6000].cpu().numpy()
        if regime == "unit-ish":
            assert np.allclose(dev, host, rtol=1e-6, atol=1e-7)
        else:
            assert (dev.view(np.uint8) == host.view(np.uint8)).all(), (regime, prec, dim)
        for fam in FAMILIES[dim] + ["normalize_sq"]:
            base = f"normalize{dim}_sq" if fam == "normalize_sq" else _base(fam, dim)
            op = _lib.OP_NORMALIZE_SQ if fam == "normalize_sq" else OPS[fam]
            takes = fam in SCALING or fam == "normalize_sq"
            res = _cuda_kernels.batch_kernel(base, prec)(x, ka if takes else None)
            torch.cuda.synchronize()
            bad, first = compare_chunked(op, x, res.head, res.body, res.sq, ka if takes else None)
            assert bad == 0, (regime, fam, prec, dim, bad, first)


def test_host_run_multi_device_sharding(cuda_dev):
    """fn_host_run_multi: shards over a device list (here device 0 three times, three
    host threads) give the same bits as the single-device host path."""
    from paper_1606_06508_b200.multigpu import host_devices

    p = fn.preset("double")
    x = _random_rows(300_001, 3, False, seed=77)
    ref = fn.normalize3(p, x)
    with host_devices([0, 0, 0]):
        got = fn.normalize3(p, x)
        q = fn.quotient2(x[:, :2].copy())
    assert oracle.same(got.length, ref.length).all() and oracle.same(got.unit, ref.unit).all()
    qr = fn.quotient2(x[:, :2].copy())
    assert oracle.same(q.unit, qr.unit).all()
    # strided rows (fn_host_run_multi_ld): xyz of xyzw records and a view of a wider array
    rec = np.full((x.shape[0], 4), np.nan)
    rec[:, :3] = x
    with host_devices([0, 0, 0]):
        got = fn.normalize3(p, rec[:, :3])
        q = fn.quotient2(x[:, :2])
    assert oracle.same(got.length, ref.length).all() and oracle.same(got.unit, ref.unit).all()
    assert oracle.same(q.unit, qr.unit).all()


@pytest.mark.parametrize("x_pinned,out_pinned", [(False, False), (True, False), (False, True), (True, True)])
def test_host_path_pageable_and_pinned(cuda_dev, x_pinned, out_pinned):
    """Host path across several 48 MiB chunks with every pinned / pageable combination
    (pageable sides go through the page-locked staging + parallel copier)."""
    p = fn.preset("double")
    n = 5_000_003  # 120 MB of input -> 3 chunks, ragged last chunk
    xn = _random_rows(n, 3, False, seed=123)
    x = torch.from_numpy(xn).pin_memory().numpy() if x_pinned else xn
    r = torch.empty(n, dtype=torch.float64, pin_memory=out_pinned).numpy()
    u = torch.empty((n, 3), dtype=torch.float64, pin_memory=out_pinned).numpy()
    fn.normalize3(p, x, out=(r, u))
    h, b, _ = oracle.run(_lib.OP_NORMALIZE, xn, np.array(fn.kernel_args(p)), threads=8)
    assert oracle.same(r, h).all() and oracle.same(u, b).all()


@pytest.mark.parametrize("graph", [False, True])
def test_back_to_back_launch_ordering(cuda_dev, graph):
    """The streaming kernels are launched with programmatic dependent launch.  Stream
    order must still hold for read-after-write (launch k+1 consumes launch k's unit
    vectors) and write-after-read (launch k+1 overwrites launch k's input), eagerly and
    inside a CUDA graph.  Buffers start as NaN so a stale read cannot pass."""
    n, chain = 1 << 21, 12
    x0 = torch.from_numpy(_random_rows(n, 3, False, seed=77)).to(cuda_dev)
    p = fn.preset("double")
    want = [x0]
    for _ in range(chain):
        want.append(fn.normalize3(p, want[-1]).unit)
    torch.cuda.synchronize()
    bufs = [x0.clone()] + [torch.full_like(x0, float("nan")) for _ in range(chain)]
    lens = [torch.full((n,), float("nan"), dtype=torch.float64, device=cuda_dev) for _ in range(chain)]
    spare = torch.full_like(x0, float("nan"))

    def run():
        for k in range(chain):
            fn.normalize3(p, bufs[k], out=(lens[k], bufs[k + 1]))
        # write-after-read: the next launch overwrites the input of the one before it
        fn.normalize3(p, bufs[chain - 1], out=(lens[0], spare))
        fn.normalize3(p, bufs[chain], out=(lens[1], bufs[chain - 1]))

    if graph:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(device=cuda_dev)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                run()
        torch.cuda.synchronize()
        for b in bufs[1:] + [spare]:
            b.fill_(float("nan"))
        bufs[0].copy_(x0)
        torch.cuda.synchronize()
        g.replay()
    else:
        run()
    torch.cuda.synchronize()
    bits = lambda t: t.view(torch.int64)  # noqa: E731
    for k in range(1, chain - 1):
        assert torch.equal(bits(bufs[k]), bits(want[k])), k
    assert torch.equal(bits(bufs[chain]), bits(want[chain]))
    assert torch.equal(bits(spare), bits(want[chain]))  # read before the overwrite
    assert torch.equal(bits(bufs[chain - 1]), bits(fn.normalize3(p, want[chain]).unit))


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_scalar_path_equals_batched_on_every_golden_row(golden, cuda_dev, prec):
    """Every golden row (random, special-value products, KATs) through the scalar
    signatures (CPython fast path -> fn_scalar, row in the kernel parameters) equals the
    batched kernels bit for bit, for every family incl. normalize{n}_sq (squared length
    first in the scalar tuple)."""
    ka = tuple(float(v) for v in golden[f"{prec}_ka"])
    for dim in (2, 3, 4):
        x = _golden_rows(golden, prec, dim)
        xd = torch.from_numpy(x).to(cuda_dev)
        for base in [_base(f, dim) for f in FAMILIES[dim]] + [f"normalize{dim}_sq"]:
            scaling = base.startswith(("scale", "normalize", "norm"))
            res = _cuda_kernels.batch_kernel(base, prec)(xd, np.array(ka) if scaling else None)
            torch.cuda.synchronize()
            table = _as_table(res)
            if base.endswith("_sq"):
                table = np.concatenate([res.sq.cpu().numpy().astype(np.float64)[:, None], table], axis=1)
            k = getattr(_cuda_kernels, f"{base}_{prec}")
            for i in range(len(x)):
                row = [float(v) for v in x[i]]
                out = k(*ka, *row) if scaling else k(*row)
                out = out if isinstance(out, tuple) else (out,)
                assert len(out) == table.shape[1]
                assert all(same_scalar(a, b) for a, b in zip(out, table[i])), (base, row, out, table[i])


def test_host_empty_buffers_exact_and_released(cuda_dev):
    """host_empty arrays (page-locked, DMA'd without staging) go through the host path and
    give the same bits as device inputs; the memory is freed with the last view."""
    import gc
    import weakref

    n = (1 << 20) + 7
    x = fn.host_empty((n, 3))
    x[:] = _random_rows(n, 3, False, seed=21)
    r, u = fn.host_empty(n), fn.host_empty((n, 3))
    p = fn.preset("double")
    fn.normalize3(p, x, out=(r, u))
    want = fn.normalize3(p, torch.from_numpy(np.array(x)).to(cuda_dev))
    assert np.array_equal(r.view(np.int64), want.length.cpu().numpy().view(np.int64))
    assert np.array_equal(u.view(np.int64), want.unit.cpu().numpy().view(np.int64))
    owner = x
    while isinstance(owner, np.ndarray):
        owner = owner.base
    alive = weakref.ref(owner)  # the ctypes block whose finalizer calls fn_host_free
    del x, owner
    gc.collect()
    assert alive() is None


def test_concurrent_calls_from_threads(cuda_dev):
    """The ABI is reentrant: host-path calls (per-device staging behind a mutex), scalar
    calls (per-thread mapped buffers) and device-path calls on per-thread streams, all
    from 6 Python threads at once, each checked against a serial run."""
    import threading

    p = fn.preset("double")
    ka = fn.kernel_args(p)
    rows = [_random_rows(200_003 + 17 * t, 3, False, seed=40 + t) for t in range(6)]
    want = [fn.normalize3(p, torch.from_numpy(x).to(cuda_dev)) for x in rows]
    want = [(w.length.cpu().numpy(), w.unit.cpu().numpy()) for w in want]
    k = _backend.scalar_kernel("normalize3", "double")
    errors = []

    def work(t):
        try:
            x = rows[t]
            for _ in range(3):
                res = fn.normalize3(p, x)  # host path
                assert np.array_equal(res.length.view(np.int64), want[t][0].view(np.int64))
                assert np.array_equal(res.unit.view(np.int64), want[t][1].view(np.int64))
                s = torch.cuda.Stream(device=cuda_dev)
                with torch.cuda.stream(s):
                    xd = torch.from_numpy(x).to(cuda_dev, non_blocking=False)
                    rd = fn.normalize3(p, xd)
                    s.synchronize()
                assert np.array_equal(rd.unit.cpu().numpy().view(np.int64), want[t][1].view(np.int64))
                for i in range(0, len(x), 20_011):
                    out = k(*ka, *x[i].tolist())
                    assert same_scalar(out[0], want[t][0][i])
                    assert all(same_scalar(a, b) for a, b in zip(out[1:], want[t][1][i]))
        except Exception as exc:  # noqa: BLE001 -- reported below
            errors.append((t, repr(exc)))

    threads = [threading.Thread(target=work, args=(t,)) for t in range(6)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors


@pytest.mark.parametrize("pinned", [False, True])
def test_host_path_every_family_small_chunks(cuda_dev, pinned, monkeypatch):
    """Every kernel family and both precisions through the host pipeline with 1 MiB
    chunks (FASTNORM_B200_HOST_CHUNK_MB is read per call): many chunks, a ragged last
    chunk, one to three output arrays of every width, page-locked or pageable buffers.
    The device path (parity-tested above) is the reference."""
    monkeypatch.setenv("FASTNORM_B200_HOST_CHUNK_MB", "1")

    def host(a):
        return torch.from_numpy(a).pin_memory().numpy() if pinned else a

    for prec, single in (("f64", False), ("f32", True)):
        for dim in (2, 3, 4):
            x = host(_random_rows(3 * (1 << 20) // (dim * (4 if single else 8)) + 4099, dim, single, seed=dim))
            xd = torch.from_numpy(np.array(x)).to(cuda_dev)
            ka = np.array(fn.kernel_args(fn.preset("single" if single else "double")))
            bases = [_base(f, dim) for f in FAMILIES[dim]] + [f"normalize{dim}_sq"]
            for base in bases:
                scaling = base.startswith(("scale", "normalize", "norm"))
                k = _cuda_kernels.batch_kernel(base, prec)
                got, want = k(x, ka if scaling else None), k(xd, ka if scaling else None)
                torch.cuda.synchronize()
                for g, w in zip(got, want):
                    if g is None:
                        continue
                    assert oracle.same(np.asarray(g), w.cpu().numpy()).all(), (base, prec)
    q = host(_random_rows(200_000, 4, False, seed=9))
    qd = torch.from_numpy(np.array(q)).to(cuda_dev)
    for f in (fn.rotation_unit, fn.rotation_general):
        assert oracle.same(f(q, strict=False), f(qd, strict=False).cpu().numpy()).all()
    res, resd = fn.normalize4_rotation(fn.preset("double"), q), fn.normalize4_rotation(fn.preset("double"), qd)
    for g, w in zip(res, resd):
        assert oracle.same(np.asarray(g), w.cpu().numpy()).all()
    v = host(_random_rows(300_001, 3, False, seed=10))
    m = fn.rotation_unit((0.1, 0.2, 0.3, 0.9))
    assert oracle.same(m.apply(v), m.apply(torch.from_numpy(np.array(v)).to(cuda_dev)).cpu().numpy()).all()


def test_in_place_outputs(cuda_dev):
    """unit (or scaled) may alias the input rows: every row is read into the tile before
    its own outputs are written, and rows belong to one tile only (device TMA path, the
    unaligned per-row path and the host pipeline)."""
    p = fn.preset("double")
    for n in (1_000_003, 777):
        xh = _random_rows(n, 3, False, seed=n)
        want = fn.normalize3(p, torch.from_numpy(xh).to(cuda_dev))
        x = torch.from_numpy(xh.copy()).to(cuda_dev)
        r = torch.empty(n, dtype=torch.float64, device=cuda_dev)
        fn.normalize3(p, x, out=(r, x))
        assert torch.equal(x.view(torch.int64), want.unit.view(torch.int64))
        assert torch.equal(r.view(torch.int64), want.length.view(torch.int64))
        big = torch.from_numpy(np.concatenate([xh[:1], xh])).to(cuda_dev)
        xu = big[1:]
        fn.normalize3(p, xu, out=(r, xu))  # 8-byte aligned rows: per-row kernel
        assert torch.equal(xu.view(torch.int64), want.unit.view(torch.int64))
        hx = xh.copy()
        hr = np.empty(n)
        fn.normalize3(p, hx, out=(hr, hx))
        assert np.array_equal(hx.view(np.int64), want.unit.cpu().numpy().view(np.int64))
        s = torch.from_numpy(xh.copy()).to(cuda_dev)
        inv = torch.empty(n, dtype=torch.float64, device=cuda_dev)
        ws = fn.scale3(p, torch.from_numpy(xh).to(cuda_dev))
        fn.scale3(p, s, out=(inv, s))
        assert torch.equal(s.view(torch.int64), ws.scaled.view(torch.int64))


def _custom_sets():
    """Valid non-preset parameter sets (validate_conditions passes), and raw constants
    that fail validation but that the kernels -- like the reference's -- still take."""
    L = math.ldexp
    d, s = fn.preset("double"), fn.preset("single")
    valid = [d.with_field("tau_min", 3 * L(1, -484)),                      # non-power-of-two tau
             d.with_field("tau_max", L(1, 500)).with_field("sigma_max", L(1, -530)),
             s.with_field("tau_max", L(1, 60)).with_field("sigma_max", L(1, -70))]
    for p in valid:
        assert fn.validate_conditions(p) == (), p
    raw = [(np.array(fn.kernel_args(d)) * np.array([1, 1, 3, 1, 1 / 3, 1]), False),   # sigma_min = 3 2^592
           (np.array(fn.kernel_args(s)) * np.array([1, 1, 1, 1.5, 1, 1 / 1.5]), True)]
    return valid, raw


def test_custom_parameter_sets(cuda_dev):
    """Any parameter set runs on the GPU bit-identically to the oracle: valid non-preset
    sets through the public API, and raw constants (non-power-of-two sigma, which
    disables exponent insertion) through the registry's batched kernels."""
    valid, raw = _custom_sets()
    for p in valid:
        single = p.precision == "single"
        ka = np.array(fn.kernel_args(p))
        x = _random_rows(1 << 18, 3, single, seed=5)
        xd = torch.from_numpy(x).to(cuda_dev)
        for op, f in ((_lib.OP_NORMALIZE, fn.normalize3), (_lib.OP_SCALE, fn.scale3), (_lib.OP_NORM, fn.norm3)):
            res = f(p, xd)
            torch.cuda.synchronize()
            h, b, _ = oracle.run(op, x, ka, threads=8)
            got = [res] if op == _lib.OP_NORM else list(res)
            want = [h] if op == _lib.OP_NORM else [h, b]
            for g, w in zip(got, want):
                assert oracle.same(g.cpu().numpy(), w).all(), (p, op)
    for ka, single in raw:
        prec = "f32" if single else "f64"
        x = _random_rows(1 << 18, 4, single, seed=6)
        xd = torch.from_numpy(x).to(cuda_dev)
        for base, op in (("normalize4", _lib.OP_NORMALIZE), ("scale4", _lib.OP_SCALE)):
            res = _cuda_kernels.batch_kernel(base, prec)(xd, ka)
            torch.cuda.synchronize()
            h, b, _ = oracle.run(op, x, ka, threads=8)
            assert oracle.same(res.head.cpu().numpy(), h).all() and oracle.same(res.body.cpu().numpy(), b).all()


@pytest.mark.parametrize("small", ["1", "0"])
def test_host_path_small_batches(cuda_dev, small, monkeypatch):
    """Host arrays up to 256 KiB of traffic take the zero-copy path (rows in mapped
    page-locked memory, per-row kernel in place); FASTNORM_B200_HOST_SMALL=0 forces the
    staged pipeline.  Both equal the device path for every family, precision and the
    two-input rotation, at sizes around the path boundary and a tile."""
    monkeypatch.setenv("FASTNORM_B200_HOST_SMALL", small)
    for prec, single in (("f64", False), ("f32", True)):
        ka = np.array(fn.kernel_args(fn.preset("single" if single else "double")))
        for dim in (2, 3, 4):
            for n in (1, 7, 255, 256, 1000, 4681):
                x = _random_rows(n, dim, single, seed=n + dim)
                xd = torch.from_numpy(x).to(cuda_dev)
                for base in [_base(f, dim) for f in FAMILIES[dim]] + [f"normalize{dim}_sq"]:
                    scaling = base.startswith(("scale", "normalize", "norm"))
                    k = _cuda_kernels.batch_kernel(base, prec)
                    got, want = k(x, ka if scaling else None), k(xd, ka if scaling else None)
                    for g, w in zip(got, want):
                        if g is not None:
                            assert oracle.same(np.asarray(g), w.cpu().numpy()).all(), (base, prec, n)
    q, v = _random_rows(300, 4, False, seed=3), _random_rows(300, 3, False, seed=4)
    got = fn.normalize4_rotate(fn.preset("double"), q, v, strict=False)
    want = fn.normalize4_rotate(fn.preset("double"), torch.from_numpy(q).to(cuda_dev),
                                torch.from_numpy(v).to(cuda_dev), strict=False)
    assert oracle.same(got, want.cpu().numpy()).all()


@pytest.mark.parametrize("home", ["device", "numpy"])
def test_structure_of_arrays_calls(cuda_dev, home):
    """The reference's scalar signatures called with one array per component
    (normalize3(p, x1[], x2[], x3[]) and friends) run the SoA kernel and equal the AoS
    batched results bit for bit, for every family, dimension and precision."""
    for prec, single in (("double", False), ("single", True)):
        p = fn.preset(prec)
        for dim in (2, 3, 4):
            x = _random_rows(100_003, dim, single, seed=17 + dim)
            xd = torch.from_numpy(x).to(cuda_dev)
            comps = [xd[:, k].contiguous() for k in range(dim)] if home == "device" else \
                [np.ascontiguousarray(x[:, k]) for k in range(dim)]
            as_np = (lambda t: t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t))  # noqa: E731

            def same(a, b):
                return oracle.same(as_np(a), as_np(b)).all()

            soa, aos = getattr(fn, f"normalize{dim}")(p, *comps), getattr(fn, f"normalize{dim}")(p, xd)
            assert same(soa.length, aos.length)
            assert all(same(soa.unit[k], aos.unit[:, k]) for k in range(dim))
            soa, aos = getattr(fn, f"normalize{dim}_sq")(p, *comps), getattr(fn, f"normalize{dim}_sq")(p, xd)
            assert same(soa.squared_length, aos.squared_length) and same(soa.length, aos.length)
            assert same(getattr(fn, f"norm{dim}")(p, *comps), getattr(fn, f"norm{dim}")(p, xd))
            soa, aos = getattr(fn, f"scale{dim}")(p, *comps), getattr(fn, f"scale{dim}")(p, xd)
            assert same(soa.inv_sigma, aos.inv_sigma)
            assert all(same(soa.scaled[k], aos.scaled[:, k]) for k in range(dim))
            bases = [getattr(fn, f"naive_normalize{dim}"), {2: fn.quotient2, 3: fn.quotient3_robust,
                                                            4: fn.quotient4}[dim]]
            if dim == 3:
                bases.append(fn.quotient3_fast)
            for f in bases:
                soa, aos = f(*comps), f(xd)
                assert same(soa.length, aos.length), f.__name__
                assert all(same(soa.unit[k], aos.unit[:, k]) for k in range(dim)), f.__name__


@pytest.mark.parametrize("home", ["device", "host"])
def test_structure_of_arrays_columns_of_records(cuda_dev, home):
    """Component arrays that are the columns of one record array (X[:, 0], X[:, 1], ...,
    dense or padded records) run the AoS kernels on the records in place; the results
    equal the AoS call bit for bit.  Columns out of order take the SoA kernels."""
    for prec, single in (("double", False), ("single", True)):
        p = fn.preset(prec)
        for dim, width in ((3, 3), (3, 4), (2, 2), (4, 4), (2, 5)):
            x = _random_rows(70_001, dim, single, seed=dim * 31 + width)
            rec = np.full((x.shape[0], width), np.nan, dtype=x.dtype)
            rec[:, :dim] = x
            if home == "device":
                rec = torch.from_numpy(rec).to(cuda_dev)
            comps = [rec[:, k] for k in range(dim)]
            as_np = (lambda t: t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t))  # noqa: E731
            for order in (list(range(dim)), list(range(dim))[::-1]):
                want = getattr(fn, f"normalize{dim}")(p, torch.from_numpy(np.ascontiguousarray(x[:, order])).to(cuda_dev))
                got = getattr(fn, f"normalize{dim}")(p, *[comps[k] for k in order])
                assert oracle.same(as_np(got.length), as_np(want.length)).all(), (prec, dim, width, order)
                for j in range(dim):
                    assert oracle.same(as_np(got.unit[j]), as_np(want.unit[:, j])).all(), (prec, dim, width, order)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_structure_of_arrays_misaligned_bulk_path(cuda_dev, prec):
    """Component arrays off the 16-byte grid by different amounts (one each of 0, 1, 2, 3
    elements) through the bulk-copy SoA kernel, sizes around the run length and the end
    reach: every scaling family equals the AoS call bit for bit."""
    single = prec == "f32"
    p = fn.preset(PREC[prec])
    run = 1024 if single else 512  # rows per 4 KiB run
    for dim in (2, 3, 4):
        for n in (run, run + 1, 2 * run - 1, 3 * run + 3, 100_003):
            x = _random_rows(n, dim, single, seed=n + dim + single)
            xd = torch.from_numpy(x).to(cuda_dev)
            comps = []
            for k in range(dim):  # array k starts k elements past an aligned allocation
                buf = torch.zeros(n + k, dtype=xd.dtype, device=cuda_dev)
                buf[k:] = xd[:, k]
                comps.append(buf[k:])
            for name in (f"normalize{dim}", f"normalize{dim}_sq", f"norm{dim}", f"scale{dim}"):
                got, want = getattr(fn, name)(p, *comps), getattr(fn, name)(p, xd)
                pairs = zip(got, want) if hasattr(got, "_fields") else [(got, want)]
                for a, b in pairs:
                    if isinstance(a, tuple):  # per-component arrays vs the AoS columns
                        assert all(oracle.same(a[k].cpu().numpy(), b[:, k].cpu().numpy()).all()
                                   for k in range(dim)), (prec, dim, n, name)
                    else:
                        assert oracle.same(a.cpu().numpy(), b.cpu().numpy()).all(), (prec, dim, n, name)


@pytest.mark.parametrize("pinned", [False, True])
def test_structure_of_arrays_host_pipeline(cuda_dev, pinned):
    """Host component arrays through fn_host_run_soa (several pipeline chunks, pageable or
    page-locked, numpy and CPU tensors, both precisions): the AoS results bit for bit."""
    for prec, single in (("double", False), ("single", True)):
        p = fn.preset(prec)
        n = 3_000_001
        x = _random_rows(n, 3, single, seed=31 + single)
        comps = []
        for k in range(3):
            a = fn.host_empty((n,), dtype=x.dtype) if pinned else np.empty(n, dtype=x.dtype)
            a[:] = x[:, k]
            comps.append(a)
        want = fn.normalize3(p, torch.from_numpy(x).to(cuda_dev))
        wl, wu = want.length.cpu().numpy(), want.unit.cpu().numpy()
        got = fn.normalize3(p, *comps)
        assert oracle.same(got.length, wl).all()
        assert all(oracle.same(got.unit[k], wu[:, k]).all() for k in range(3))
        sq = fn.normalize3_sq(p, *comps)
        assert oracle.same(sq.length, wl).all()
        assert oracle.same(fn.norm3(p, *comps), wl).all()
        sc = fn.scale3(p, *comps)
        wsc = fn.scale3(p, torch.from_numpy(x).to(cuda_dev))
        assert oracle.same(sc.inv_sigma, wsc.inv_sigma.cpu().numpy()).all()
        t = fn.normalize3(p, *[torch.from_numpy(c) for c in comps])  # CPU tensors
        assert isinstance(t.length, torch.Tensor) and oracle.same(t.length.numpy(), wl).all()
        for m in (1, 100, 5000):  # the zero-copy route for small batches
            sub = [np.ascontiguousarray(c[:m]) for c in comps]
            got = fn.normalize3(p, *sub)
            assert oracle.same(got.length, wl[:m]).all()
            assert all(oracle.same(got.unit[k], wu[:m, k]).all() for k in range(3))
            q = fn.normalize3_sq(p, *sub)
            assert oracle.same(q.length, wl[:m]).all() and oracle.same(q.squared_length, sq.squared_length[:m]).all()


def test_structure_of_arrays_unaligned_and_tails(cuda_dev):
    """Component arrays at an 8-byte offset (scalar SoA kernel) and lengths that leave a
    partial 16-byte vector (vector kernel + scalar tail) give the AoS results."""
    p = fn.preset("double")
    for n in (1, 2, 3, 5, 1001):
        x = _random_rows(n, 3, False, seed=n)
        xd = torch.from_numpy(x).to(cuda_dev)
        want = fn.normalize3(p, xd)
        big = [torch.from_numpy(np.concatenate([[0.0], x[:, k]])).to(cuda_dev)[1:] for k in range(3)]
        for comps in (big, [xd[:, k].contiguous() for k in range(3)]):
            got = fn.normalize3(p, *comps)
            assert oracle.same(got.length.cpu().numpy(), want.length.cpu().numpy()).all()
            for k in range(3):
                assert oracle.same(got.unit[k].cpu().numpy(), want.unit[:, k].cpu().numpy()).all()
    x32 = _random_rows(4099, 3, True, seed=1)
    comps = [torch.from_numpy(np.ascontiguousarray(x32[:, k])).to(cuda_dev) for k in range(3)]
    got, want = fn.normalize3(fn.preset("single"), *comps), fn.normalize3(fn.preset("single"), torch.from_numpy(x32).to(cuda_dev))
    assert all(oracle.same(got.unit[k].cpu().numpy(), want.unit[:, k].cpu().numpy()).all() for k in range(3))
