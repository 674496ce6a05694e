"""Single-process multi-GPU driver (fn_run_sharded, multigpu.DeviceShards): device-resident
row shards, one stream per shard, no collective.  On a one-GPU box the shards all live on
cuda:0 (independent kernels on separate streams); with two or more GPUs the distinct-device
case runs too.  The results must equal the one-launch call bit for bit (rows are
independent: /root/reference/pkg/src/fastnorm/_kernels.pyx:167-412)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _bits(t):
    import torch

    return t.cpu().contiguous().view(torch.int64 if t.dtype == torch.float64 else torch.int32)


def _device_lists():
    import torch

    lists = [[0], [0, 0], [0, 0, 0]]
    if torch.cuda.device_count() >= 2:
        lists.append(list(range(torch.cuda.device_count())))
    return lists


@pytest.mark.parametrize("cfg", [5, 4, 2, 3])
def test_generate_shards_equal_one_device_batch(cfg):
    import torch

    from paper_1606_06508_b200 import multigpu, workloads

    rows = (1 << 18) + 37
    c = workloads.CONFIGS[cfg]
    dt = torch.float64 if c.dtype == "float64" else torch.float32
    whole = torch.empty((rows, c.dim), dtype=dt, device="cuda:0")
    workloads.generate_device(cfg, whole)
    for devs in _device_lists():
        sh = multigpu.DeviceShards.generate(cfg, rows, devs)
        assert sh.rows == rows and sh.devices == devs
        assert torch.equal(_bits(sh.gather()), _bits(whole))


@pytest.mark.parametrize("cfg", [5, 4, 2, 3])
def test_normalize_sharded_bit_exact(cfg):
    import torch

    import paper_1606_06508_b200 as fn
    from paper_1606_06508_b200 import multigpu, workloads

    rows = (1 << 20) + 1001
    c = workloads.CONFIGS[cfg]
    dt = torch.float64 if c.dtype == "float64" else torch.float32
    p = fn.preset("double" if dt == torch.float64 else "single")
    whole = torch.empty((rows, c.dim), dtype=dt, device="cuda:0")
    workloads.generate_device(cfg, whole)
    ref = getattr(fn, f"normalize{c.dim}")(p, whole)
    ref_norm = getattr(fn, f"norm{c.dim}")(p, whole)
    torch.cuda.synchronize()
    for devs in _device_lists():
        sh = multigpu.DeviceShards.generate(cfg, rows, devs)
        res = multigpu.normalize_sharded(p, sh)
        assert res.sq is None and len(res.elapsed_ms) == len(devs)
        assert all(ms > 0 for ms in res.elapsed_ms)
        assert torch.equal(_bits(res.head.gather()), _bits(ref.length))
        assert torch.equal(_bits(res.body.gather()), _bits(ref.unit))
        nr = multigpu.norm_sharded(p, sh)
        assert nr.body is None
        assert torch.equal(_bits(nr.head.gather()), _bits(ref_norm))


def test_every_family_through_the_sharded_entry():
    import torch

    from paper_1606_06508_b200 import _lib, batch, multigpu, workloads
    from paper_1606_06508_b200.params import preset
    from paper_1606_06508_b200.scale import kernel_args_array

    rows = 300_001
    ka = kernel_args_array(preset("double"))
    whole = torch.empty((rows, 3), dtype=torch.float64, device="cuda:0")
    workloads.generate_device(5, whole)
    sh = multigpu.DeviceShards.scatter(whole, [0, 0, 0])
    for op in (_lib.OP_SCALE, _lib.OP_NORMALIZE, _lib.OP_NORM, _lib.OP_NAIVE, _lib.OP_QUOTIENT,
               _lib.OP_QUOTIENT3_FAST, _lib.OP_NORMALIZE_SQ):
        needs_ka = op in (_lib.OP_SCALE, _lib.OP_NORMALIZE, _lib.OP_NORM, _lib.OP_NORMALIZE_SQ)
        ref = batch.run(op, 3, whole, ka if needs_ka else None)
        res = multigpu.run_sharded(op, 3, sh, ka if needs_ka else None)
        for got, want in zip((res.head, res.body, res.sq), ref):
            assert (got is None) == (want is None)
            if want is not None:
                assert torch.equal(_bits(got.gather()), _bits(want)), op


def test_sharded_out_reuse_and_producer_ordering():
    """Outputs are reused across calls, and each shard waits for the work already queued
    on torch's current stream of its device (the copy that fills its rows)."""
    import torch

    import paper_1606_06508_b200 as fn
    from paper_1606_06508_b200 import multigpu, workloads

    rows = 1 << 21
    p = fn.preset("double")
    devs = [0, 0]
    a = multigpu.DeviceShards.generate(5, rows, devs)
    b = multigpu.DeviceShards.generate(1, rows, devs)
    ra = multigpu.normalize_sharded(p, a)
    rb = multigpu.normalize_sharded(p, b)
    want = {0: (ra.head.gather(), ra.body.gather()), 1: (rb.head.gather(), rb.body.gather())}
    x = multigpu.DeviceShards.empty(rows, 3, torch.float64, devs)
    r = multigpu.DeviceShards.empty(rows, 0, torch.float64, devs)
    u = multigpu.DeviceShards.empty(rows, 3, torch.float64, devs)
    for it in range(8):
        src = (a, b)[it % 2]
        for t, s in zip(x.tensors, src.tensors):
            t.copy_(s, non_blocking=True)  # queued on the current stream, not waited for
        res = multigpu.normalize_sharded(p, x, out=(r, u))
        assert res.head is r and res.body is u
        assert torch.equal(_bits(r.gather()), _bits(want[it % 2][0]))
        assert torch.equal(_bits(u.gather()), _bits(want[it % 2][1]))


def test_sharded_empty_and_ragged_shards():
    import torch

    import paper_1606_06508_b200 as fn
    from paper_1606_06508_b200 import multigpu, workloads

    p = fn.preset("double")
    for rows in (0, 1, 2, 5):
        sh = multigpu.DeviceShards.generate(5, rows, [0, 0, 0])  # some shards are empty
        res = multigpu.normalize_sharded(p, sh)
        assert res.head.rows == rows
        if rows:
            whole = torch.empty((rows, 3), dtype=torch.float64, device="cuda:0")
            workloads.generate_device(5, whole)
            ref = fn.normalize3(p, whole)
            assert torch.equal(_bits(res.head.gather()), _bits(ref.length))
            assert torch.equal(_bits(res.body.gather()), _bits(ref.unit))


def test_sharded_errors():
    import ctypes

    import torch

    import paper_1606_06508_b200 as fn
    from paper_1606_06508_b200 import _lib, multigpu

    p = fn.preset("double")
    sh = multigpu.DeviceShards.generate(5, 1000, [0, 0])
    with pytest.raises(TypeError):
        multigpu.normalize_sharded(fn.preset("single"), sh)
    with pytest.raises(TypeError):
        multigpu.run_sharded(_lib.OP_NORMALIZE, 3, sh.tensors, None)
    bad = multigpu.DeviceShards.empty(999, 0, torch.float64, [0, 0])
    with pytest.raises(ValueError):
        multigpu.normalize_sharded(p, sh, out=(bad, None))
    # raw ABI: a device ordinal that does not exist, and a NULL output
    L = _lib.lib()
    n = (ctypes.c_int64 * 1)(10)
    x = torch.zeros((10, 3), dtype=torch.float64, device="cuda:0")
    r = torch.zeros(10, dtype=torch.float64, device="cuda:0")
    u = torch.zeros((10, 3), dtype=torch.float64, device="cuda:0")
    xp, rp, up = ((ctypes.c_void_p * 1)(t.data_ptr()) for t in (x, r, u))
    ka = np.array(fn.kernel_args(p), dtype=np.float64)
    nodev = (ctypes.c_int * 1)(torch.cuda.device_count())
    dev0 = (ctypes.c_int * 1)(0)

    def call(dev, body):
        return L.fn_run_sharded(_lib.OP_NORMALIZE, 3, _lib.F64, 1, ctypes.addressof(dev), ctypes.addressof(xp),
                                ctypes.addressof(n), ctypes.addressof(rp), body, None, ka.ctypes.data, None, None)

    assert call(nodev, ctypes.addressof(up)) == -1
    assert b"device index" in L.fn_last_error()
    assert call(dev0, None) == -1
    assert call(dev0, ctypes.addressof(up)) == 0
