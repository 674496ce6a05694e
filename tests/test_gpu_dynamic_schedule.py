"""tma_stream_kernel's dynamic tile schedule (small batches: more than S and at most 32
tiles per CTA; a {next, done} counter pair per stream, reset by the kernel's last CTA).

The schedule changes which CTA computes a tile, never what is computed: outputs must be
bit-identical to the oracle and to the static schedule (FASTNORM_B200_DYN=0), across
back-to-back launches on one stream (the counter is reset between them, PDL included),
on two streams at once (each stream has its own pair), and in CUDA graphs (a captured
launch owns a counter that its last CTA re-zeroes for the next replay)."""

import os
import subprocess
import sys

import numpy as np
import pytest

from gpu_helpers import compare_chunked

import oracle
import paper_1606_06508_b200 as fn
from paper_1606_06508_b200 import _lib, workloads

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

SIZES = [1_000_000, 600_001, (1 << 21) + 5, 3_000_017]  # config 1 and neighbours (dynamic range)


def _rows(n, cfg=5, dtype=torch.float64, dim=3):
    x = torch.empty((n, dim), dtype=dtype, device="cuda")
    workloads.generate_device(cfg, x)
    return x


@pytest.mark.parametrize("n", SIZES)
def test_dynamic_schedule_matches_oracle(cuda_dev, n):
    p = fn.preset("double")
    x = _rows(n)
    out = fn.normalize3(p, x)
    torch.cuda.synchronize()
    bad, first = compare_chunked(_lib.OP_NORMALIZE, x, out.length, out.unit, ka=np.array(fn.kernel_args(p)))
    assert bad == 0, first


@pytest.mark.parametrize("dtype,cfg,family", [(torch.float32, 4, "quotient3"), (torch.float32, 4, "normalize3"),
                                              (torch.float64, 1, "normalize3")])
def test_back_to_back_launches_reuse_the_counter(cuda_dev, dtype, cfg, family):
    p = fn.preset("single" if dtype == torch.float32 else "double")
    call = (lambda x, out=None: fn.quotient3_robust(x, out=out)) if family == "quotient3" else \
        (lambda x, out=None: fn.normalize3(p, x, out=out))
    xs = [_rows(n, cfg, dtype) for n in SIZES]
    want = [call(x) for x in xs]
    torch.cuda.synchronize()
    want = [(w.length.clone(), w.unit.clone()) for w in want]
    outs = [(torch.empty_like(w[0]), torch.empty_like(w[1])) for w in want]
    for _ in range(20):  # 80 launches on one stream, no synchronisation between them
        for x, o in zip(xs, outs):
            call(x, out=o)
    torch.cuda.synchronize()
    for w, o in zip(want, outs):
        assert torch.equal(w[0].view(torch.int64 if dtype == torch.float64 else torch.int32),
                           o[0].view(torch.int64 if dtype == torch.float64 else torch.int32))
        assert torch.equal(w[1].view(torch.int64 if dtype == torch.float64 else torch.int32),
                           o[1].view(torch.int64 if dtype == torch.float64 else torch.int32))


def test_two_streams_at_once(cuda_dev):
    p = fn.preset("double")
    xa, xb = _rows(1_000_000, 1), _rows(3_000_017, 5)
    wa, wb = fn.normalize3(p, xa), fn.normalize3(p, xb)
    torch.cuda.synchronize()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    oa = [(torch.empty_like(wa.length), torch.empty_like(wa.unit)) for _ in range(8)]
    ob = [(torch.empty_like(wb.length), torch.empty_like(wb.unit)) for _ in range(8)]
    for k in range(8):
        with torch.cuda.stream(sa):
            fn.normalize3(p, xa, out=oa[k])
        with torch.cuda.stream(sb):
            fn.normalize3(p, xb, out=ob[k])
    torch.cuda.synchronize()
    for k in range(8):
        assert torch.equal(oa[k][1].view(torch.int64), wa.unit.view(torch.int64))
        assert torch.equal(ob[k][1].view(torch.int64), wb.unit.view(torch.int64))
        assert torch.equal(ob[k][0].view(torch.int64), wb.length.view(torch.int64))


def _i64(t):
    return t.view(torch.int64 if t.dtype == torch.float64 else torch.int32)


def test_graph_capture_small_batch(cuda_dev):
    p = fn.preset("double")
    x = _rows(1_000_000, 1)
    want = fn.normalize3(p, x)
    r, u = torch.empty_like(want.length), torch.empty_like(want.unit)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn.normalize3(p, x, out=(r, u))
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(3):
                fn.normalize3(p, x, out=(r, u))
    for _ in range(3):
        r.zero_()
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(u.view(torch.int64), want.unit.view(torch.int64))
    assert torch.equal(r.view(torch.int64), want.length.view(torch.int64))


def test_graph_capture_dynamic_schedule_replays(cuda_dev):
    """Captured launches claim tiles from a counter of their own that the kernel's last CTA
    re-zeroes: a graph holding AoS, SoA and many-batch launches (back to back, PDL edges
    included) must give the eager results on every one of many replays, also when the
    replays alternate between two streams."""
    p = fn.preset("double")
    n = (1 << 23) + 12345  # well past S tiles per CTA: the dynamic part does most tiles
    x = _rows(n, 5)
    x2 = _rows(n, 2, dim=2)
    comps = [x[:, c].contiguous() for c in range(3)]
    many = [_rows(m, 1) for m in (1_000_000, 700_001, 1_300_000, 999_999, 1_000_000, 1_200_000, 2_000_003, 1_500_000)]
    w_aos, w_norm, w_2 = fn.normalize3(p, x), fn.norm3(p, x), fn.normalize2(p, x2)
    w_soa = fn.normalize3(p, *comps)
    w_many = fn.normalize_many(p, many)
    w_q = fn.quotient3_robust(x)
    torch.cuda.synchronize()
    o_aos = (torch.empty_like(w_aos.length), torch.empty_like(w_aos.unit))
    o_norm = torch.empty_like(w_norm)
    o_2 = (torch.empty_like(w_2.length), torch.empty_like(w_2.unit))
    o_q = (torch.empty_like(w_q.length), torch.empty_like(w_q.unit))
    o_many = [(torch.empty_like(w.length), torch.empty_like(w.unit)) for w in w_many]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    soa_out = {}
    with torch.cuda.stream(s):
        fn.normalize3(p, x, out=o_aos)  # eager warm-up on the capture stream (allocates the counter pool)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            fn.normalize3(p, x, out=o_aos)
            fn.norm3(p, x, out=o_norm)
            fn.normalize2(p, x2, out=o_2)
            soa_out["res"] = fn.normalize3(p, *comps)
            fn.normalize_many(p, many, out=o_many)
            fn.quotient3_robust(x, out=o_q)
            fn.normalize3(p, x, out=o_aos)  # the same node kind twice in one graph
    s2 = torch.cuda.Stream()
    for it in range(12):
        for t in (o_aos[0], o_aos[1], o_norm, o_2[0], o_2[1], o_q[0], o_q[1]):
            t.zero_()
        torch.cuda.synchronize()
        with torch.cuda.stream(s if it % 2 == 0 else s2):
            g.replay()
        torch.cuda.synchronize()
        assert torch.equal(_i64(o_aos[0]), _i64(w_aos.length)) and torch.equal(_i64(o_aos[1]), _i64(w_aos.unit)), it
        assert torch.equal(_i64(o_norm), _i64(w_norm)), it
        assert torch.equal(_i64(o_2[0]), _i64(w_2.length)) and torch.equal(_i64(o_2[1]), _i64(w_2.unit)), it
        assert torch.equal(_i64(o_q[0]), _i64(w_q.length)) and torch.equal(_i64(o_q[1]), _i64(w_q.unit)), it
        sr = soa_out["res"]
        assert torch.equal(_i64(sr.length), _i64(w_soa.length)), it
        for a, b in zip(sr.unit, w_soa.unit):
            assert torch.equal(_i64(a), _i64(b)), it
        for o, w in zip(o_many, w_many):
            assert torch.equal(_i64(o[0]), _i64(w.length)) and torch.equal(_i64(o[1]), _i64(w.unit)), it
    # eager launches still work after (and between) replays: the stream pair is untouched
    again = fn.normalize3(p, x)
    torch.cuda.synchronize()
    assert torch.equal(_i64(again.unit), _i64(w_aos.unit))


def test_static_and_dynamic_schedules_agree(cuda_dev, tmp_path):
    """The same batches under FASTNORM_B200_DYN=0 (static) and =1 (dynamic wherever a
    batch has more than S tiles per CTA, large ones included), in fresh processes."""
    code = ("import sys, numpy as np, torch, paper_1606_06508_b200 as fn\n"
            "from paper_1606_06508_b200 import workloads\n"
            "p = fn.preset('double'); outs = []\n"
            "for n in (1_000_000, 3_000_017, 1 << 25):\n"
            "    x = torch.empty((n, 3), dtype=torch.float64, device='cuda'); workloads.generate_device(5, x)\n"
            "    o = fn.normalize3(p, x); outs += [o.length.cpu().numpy(), o.unit.cpu().numpy().ravel()]\n"
            "    o = fn.normalize3(p, *[x[:, c].contiguous() for c in range(3)])\n"
            "    outs += [o.length.cpu().numpy()] + [c.cpu().numpy() for c in o.unit]\n"
            "    for o in fn.normalize_many(p, [x[: n // 3], x[n // 3:]]):\n"
            "        outs += [o.length.cpu().numpy(), o.unit.cpu().numpy().ravel()]\n"
            "np.save(sys.argv[1], np.concatenate(outs))\n")
    res = {}
    for mode in ("0", "1"):
        path = str(tmp_path / f"dyn{mode}.npy")
        env = dict(os.environ, FASTNORM_B200_DYN=mode)
        out = subprocess.run([sys.executable, "-c", code, path], env=env, capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        res[mode] = np.load(path)
    assert np.array_equal(res["0"].view(np.uint64), res["1"].view(np.uint64))
