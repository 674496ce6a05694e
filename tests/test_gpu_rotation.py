"""Batched rotations on the GPU (reference rotation.py:53-111), bit for bit against the
reference's own outputs (golden) and the oracle, including the fused normalize4 ->
rotation_unit kernel, at the config-3 size (2^27 quaternions)."""

import numpy as np
import pytest

from gpu_helpers import to_np

import oracle
import paper_1606_06508_b200 as fn
from paper_1606_06508_b200 import workloads

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("where", ["device", "device_unaligned", "host"])
def test_rotation_golden(golden, cuda_dev, where):
    q = golden["rot_q"]
    if where == "device":
        qd = torch.from_numpy(q).to(cuda_dev)
    elif where == "device_unaligned":
        qd = torch.from_numpy(np.concatenate([q[:1], q])).to(cuda_dev)[1:]
    else:
        qd = q
    g = fn.rotation_general(qd, strict=False)
    u = fn.rotation_unit(qd, strict=False)
    torch.cuda.synchronize()
    g = to_np(g) if hasattr(g, "cpu") else g
    u = to_np(u) if hasattr(u, "cpu") else u
    assert oracle.same(g.reshape(-1, 9), golden["rot_general"]).all()
    assert oracle.same(u.reshape(-1, 9), golden["rot_unit"]).all()
    res = fn.normalize4_rotation(fn.preset("double"), qd)
    torch.cuda.synchronize()
    R = to_np(res.rotation) if hasattr(res.rotation, "cpu") else res.rotation
    assert oracle.same(R.reshape(-1, 9), golden["rot_unit_of_normalized"]).all()


def test_rotation_errors_and_kats(cuda_dev):
    with pytest.raises(ValueError):
        fn.rotation_general((0.0, 0.0, 0.0, 0.0))
    with pytest.raises(ValueError):
        fn.rotation_general((float("inf"), 0.0, 0.0, 1.0))
    with pytest.raises(ValueError):
        fn.rotation_unit((float("nan"), 0.0, 0.0, 1.0))
    assert fn.rotation_general((0.0, 0.0, 0.0, 2.0)).rows == ((1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0))
    assert fn.rotation_general((1.0, 0.0, 0.0, 0.0)).rows == ((1.0, 0.0, 0.0), (0.0, -1.0, 0.0), (0.0, 0.0, -1.0))
    assert fn.rotation_general((1.0, 1.0, 1.0, 1.0)).rows == ((0.0, 0.0, 1.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0))
    q = torch.tensor([[0.0, 0.0, 0.0, 1.0], [0.0, 0.0, 0.0, 0.0]], dtype=torch.float64, device=cuda_dev)
    with pytest.raises(ValueError):
        fn.rotation_general(q)
    R = fn.rotation_general(q, strict=False)
    torch.cuda.synchronize()
    assert torch.isnan(R[1]).all() and R[0].tolist() == [[1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]]
    fn.rotation_unit(q)  # the zero quaternion is finite: accepted by the unit form
    with pytest.raises(TypeError):
        fn.rotation_unit(q.float())


def test_rotations_cfg3_full(cuda_dev):
    """All 2^27 config-3 quaternions through the three rotation kernels vs the oracle."""
    ka = np.array(fn.kernel_args(fn.preset("double")))
    n = workloads.CONFIGS[3].rows
    q = torch.empty((n, 4), dtype=torch.float64, device=cuda_dev)
    workloads.generate_device(3, q)
    res = fn.normalize4_rotation(fn.preset("double"), q)
    G = fn.rotation_general(q)
    torch.cuda.synchronize()
    chunk = 1 << 24
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        qh = to_np(q[lo:hi])
        r, u, R, bad = oracle.rotation(oracle.OP_NORMALIZE_ROT, qh, ka)
        assert bad == 0
        assert oracle.same(to_np(res.length[lo:hi]), r).all()
        assert oracle.same(to_np(res.unit[lo:hi]), u).all()
        assert oracle.same(to_np(res.rotation[lo:hi]), R).all()
        Rg, bad = oracle.rotation(oracle.OP_ROT_GENERAL, qh, ka)
        assert bad == 0 and oracle.same(to_np(G[lo:hi]), Rg).all()
    U = fn.rotation_unit(res.unit)
    torch.cuda.synchronize()
    assert bool((U.view(torch.int64) == res.rotation.view(torch.int64)).all())


@pytest.mark.parametrize("where", ["device", "device_unaligned", "host"])
def test_rotate_apply_golden(golden, cuda_dev, where):
    """RotationMatrix.apply over a batch (FN_OP_ROT_APPLY) == the reference's apply, row
    by row, for every golden matrix and vector (special values included)."""
    v = golden["rot_apply_v"]
    if where == "device":
        vd = torch.from_numpy(v).to(cuda_dev)
    elif where == "device_unaligned":
        vd = torch.from_numpy(np.concatenate([v[:1], v])).to(cuda_dev)[1:]
    else:
        vd = v
    for Rf, want in zip(golden["rot_apply_R"], golden["rot_apply_out"]):
        m = fn.RotationMatrix(tuple(tuple(Rf[3 * i:3 * i + 3].tolist()) for i in range(3)))
        got = m.apply(vd)
        got = to_np(got) if hasattr(got, "cpu") else got
        assert oracle.same(got, want).all()
        # the scalar form (the reference's own Python expression) agrees as well
        for k in range(0, len(v), 97):
            assert oracle.same(np.array(m.apply(tuple(v[k].tolist()))), want[k]).all()


def test_rotate_vectors_full_size(cuda_dev):
    """2^27 config-5-class vectors (wide exponent range, near-DBL_MAX and subnormal rows)
    rotated by one quaternion, unit and general forms, vs the oracle; the scalar matrix
    comes from the scalar rotation path."""
    n = 1 << 27
    v = torch.empty((n, 3), dtype=torch.float64, device=cuda_dev)
    workloads.generate_device(5, v)
    q = (0.3, -1.2, 2.5, 0.7)
    for method in ("unit", "general"):
        out = fn.rotate_vectors(q, v, method=method)
        m = fn.rotation_unit(q) if method == "unit" else fn.rotation_general(q)
        torch.cuda.synchronize()
        chunk = 1 << 24
        for lo in range(0, n, chunk):
            vh = to_np(v[lo:lo + chunk])
            assert oracle.same(to_np(out[lo:lo + chunk]), oracle.rotate_apply(m.flat(), vh)).all()
    with pytest.raises(TypeError):
        fn.rotation_unit(q).apply(v.float())


@pytest.mark.parametrize("where", ["device", "device_unaligned", "host", "host_pinned"])
def test_rotate_rows_golden(golden, cuda_dev, where):
    """Per-row rotation of vectors (two-input kernels) == the reference composition on every
    golden row: normalize4 -> rotation_unit -> apply, and per-row RotationMatrix.apply."""
    q, v, Rg = golden["rot_q"], golden["rot_rows_v"], golden["rot_general"]
    p = fn.preset("double")

    def home(a):
        if where == "device":
            return torch.from_numpy(a).to(cuda_dev)
        if where == "device_unaligned":
            return torch.from_numpy(np.concatenate([a[:1], a])).to(cuda_dev)[1:]
        if where == "host_pinned":
            return torch.from_numpy(a).pin_memory().numpy()
        return a

    got = fn.normalize4_rotate(p, home(q), home(v), strict=False)
    assert oracle.same(to_np(got) if hasattr(got, "cpu") else got, golden["rot_rows_quat_out"]).all()
    got = fn.apply_rotations(home(Rg), home(v))
    assert oracle.same(to_np(got) if hasattr(got, "cpu") else got, golden["rot_rows_mat_out"]).all()
    with pytest.raises(ValueError):
        fn.normalize4_rotate(p, home(q), home(v))  # three non-finite quaternions


@pytest.mark.parametrize("shift_q,shift_v", [(0, 1), (1, 0), (1, 1), (0, 2)])
def test_rotate_rows_misaligned_bulk_path(cuda_dev, shift_q, shift_v):
    """Two-input kernels with either input off the 16-byte grid (x[k:] views): both
    inputs are loaded from the boundary below each tile; equal to the aligned call."""
    n = 100_003
    p = fn.preset("double")
    q = torch.empty((n + 2, 4), dtype=torch.float64, device=cuda_dev)
    workloads.generate_device(3, q)
    v = torch.empty((n + 2, 3), dtype=torch.float64, device=cuda_dev)
    workloads.generate_device(5, v)
    qa, va = q[:n].clone(), v[:n].clone()
    qs = torch.empty((n + shift_q, 4), dtype=torch.float64, device=cuda_dev)[shift_q:]
    qs.copy_(qa)
    flat = torch.empty(n * 3 + shift_v, dtype=torch.float64, device=cuda_dev)  # shift by elements
    vs = flat[shift_v:].view(n, 3)
    vs.copy_(va)
    assert oracle.same(to_np(fn.normalize4_rotate(p, qs, vs)), to_np(fn.normalize4_rotate(p, qa, va))).all()
    R = fn.rotation_unit(qa)
    Rflat = torch.empty(n * 9 + shift_q, dtype=torch.float64, device=cuda_dev)
    Rs = Rflat[shift_q:].view(n, 3, 3)
    Rs.copy_(R)
    assert oracle.same(to_np(fn.apply_rotations(Rs, vs)), to_np(fn.apply_rotations(R, va))).all()


def test_rotate_rows_full_size(cuda_dev):
    """2^27 config-3 quaternions rotating 2^27 config-5-class vectors, vs the oracle, and
    the per-row matrix form on the rotation_unit matrices of the same quaternions."""
    n = workloads.CONFIGS[3].rows
    p = fn.preset("double")
    ka = np.array(fn.kernel_args(p))
    q = torch.empty((n, 4), dtype=torch.float64, device=cuda_dev)
    workloads.generate_device(3, q)
    v = torch.empty((n, 3), dtype=torch.float64, device=cuda_dev)
    workloads.generate_device(5, v)
    out = fn.normalize4_rotate(p, q, v)
    torch.cuda.synchronize()
    chunk = 1 << 24
    for lo in range(0, n, chunk):
        want, bad = oracle.rotate_rows(oracle.OP_QUAT_ROTATE, to_np(q[lo:lo + chunk]), to_np(v[lo:lo + chunk]), ka)
        assert bad == 0 and oracle.same(to_np(out[lo:lo + chunk]), want).all()
    sub = 1 << 22
    R = fn.rotation_unit(q[:sub])
    out2 = fn.apply_rotations(R, v[:sub])
    want2, _ = oracle.rotate_rows(oracle.OP_MAT_APPLY, to_np(R).reshape(sub, 9), to_np(v[:sub]))
    assert oracle.same(to_np(out2), want2).all()
    # the fused path equals the three-step composition on the device
    u = fn.normalize4(p, q[:sub]).unit
    assert oracle.same(to_np(out[:sub]), to_np(fn.apply_rotations(fn.rotation_unit(u), v[:sub]))).all()
