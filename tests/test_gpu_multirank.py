"""Multi-rank and multi-device paths on whatever GPUs the box has (often one).

* bench.py with two ranks: launched by torchrun explicitly and by bench.py's own
  self-launch (``--gpus 2`` without a torchrun environment), both ranks on cuda:0 with
  the gloo backend (NCCL refuses two ranks on one GPU).  The ranks share no kernels and
  wait on nothing but host barriers, so this is the N = 2 control flow of the 8-GPU
  run: sharding, barriers, max-over-ranks timing, the counter reduce, the e2e legs.
* ``bench.py --gpus N`` with more NCCL ranks than GPUs exits non-zero instead of
  silently running one rank.
* fn_host_run_multi / fn_host_run_soa_multi over distinct ordinals (skipped with fewer
  than two GPUs) and over one ordinal repeated, bit-identical to the one-device call;
  repeated small sharded calls do not grow the zero-copy context pool.
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import paper_1606_06508_b200 as fn
from paper_1606_06508_b200 import _lib, workloads

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(REPO, "bench.py")
ROWS = 1 << 26
ARGS = ["--gpus", "2", "--rows", "2^26", "--dist-backend", "gloo", "--steps", "3", "--warmup", "3",
        "--e2e-steps", "1", "--no-configs", "--no-cpu-baseline"]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _json_line(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-3000:]
    return json.loads(lines[0])


def _check_two_rank_line(d):
    assert d["n_gpus"] == 2
    assert d["validation"]["rows_counted"] == ROWS
    assert "gloo" in d["validation"]["reduce"]
    assert d["config"]["rows_total"] == ROWS and d["config"]["rows_per_gpu"] == ROWS // 2
    assert np.isfinite(d["value"]) and d["value"] > 0
    assert d["e2e"]["value"] and d["e2e"]["value"] > 0 and d["e2e"]["gpu_launches"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == ROWS * 24
    assert d["e2e_default_api"]["value"] and d["e2e_default_api"]["value"] > 0


def test_bench_two_ranks_under_torchrun():
    env = dict(os.environ, OMP_NUM_THREADS="4")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), BENCH] + ARGS
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    _check_two_rank_line(_json_line(p.stdout))


def test_bench_self_launches_two_ranks():
    env = dict(os.environ, OMP_NUM_THREADS="4")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, BENCH] + ARGS, capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    _check_two_rank_line(_json_line(p.stdout))


def test_bench_refuses_more_nccl_ranks_than_gpus():
    n = torch.cuda.device_count() + 1
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, BENCH, "--gpus", str(n), "--steps", "3", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert p.returncode != 0 and "needs" in p.stderr
    assert not [ln for ln in p.stdout.splitlines() if ln.startswith("{")]


def _host_rows(n):
    x = workloads.host_rows(5, 0, n)
    x[:7] = [[0.0, 0.0, 0.0], [-0.0, 0.0, -0.0], [np.inf, 1.0, -2.0], [np.nan, 1.0, 0.0],
             [1.7976931348623157e308] * 3, [5e-324, -5e-324, 5e-324], [-3.0, 0.0, -0.0]]
    return x


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("devices", ["distinct", "repeated"])
def test_host_run_multi_devices(devices):
    ndev = torch.cuda.device_count()
    if devices == "distinct":
        if ndev < 2:
            pytest.skip("needs two GPUs")
        devs = list(range(min(ndev, 4)))
    else:
        devs = [0, 0, 0]
    p = fn.preset("double")
    x = _host_rows(3_000_017)
    want = fn.normalize3(p, x)
    with fn.batch.host_devices(devs):
        got = fn.normalize3(p, x)
        got_soa = fn.normalize3(p, *(np.ascontiguousarray(x[:, k]) for k in range(3)))
    assert _same(got.length, want.length) and _same(got.unit, want.unit)
    assert _same(got_soa.length, want.length)
    for k in range(3):
        assert _same(got_soa.unit[k], want.unit[:, k])


def test_small_sharded_calls_reuse_contexts():
    """every sharded small call used to leak a mapped page-locked
    buffer and a stream per device (thread_local contexts on short-lived threads)."""
    L = _lib.lib()
    p = fn.preset("double")
    x = _host_rows(1000)
    want = fn.normalize3(p, x)
    with fn.batch.host_devices([0, 0]):
        fn.normalize3(p, x)
        before = L.fn_small_contexts()
        for _ in range(200):
            got = fn.normalize3(p, x)
        after = L.fn_small_contexts()
    assert _same(got.length, want.length) and _same(got.unit, want.unit)
    assert after - before <= 2, (before, after)
