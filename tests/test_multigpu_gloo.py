"""N > 1 host logic on CPU: world-size-2 gloo process group (127.0.0.1).

Sharding covers every row exactly once, the validation counters reduced over ranks equal
the single-process counters, and max-over-ranks returns the slowest rank's time -- the
same code bench.py runs over NCCL on the B200 box.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1606_06508_b200 import multigpu, workloads
from paper_1606_06508_b200.params import preset
from paper_1606_06508_b200.scale import kernel_args


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = multigpu.shard_range(n, rank, world)
        x = workloads.host_rows(cfg, lo, hi - lo)
        prec = "single" if x.dtype == np.float32 else "double"
        c = torch.from_numpy(workloads.row_stats_host(x, kernel_args(preset(prec))).astype(np.int64))
        total = multigpu.reduce_counts(c)
        t = multigpu.max_over_ranks(0.25 * (rank + 1))
        q.put((rank, lo, hi, total, t))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,n", [(2, 100_003), (4, 200_001), (5, 150_000)])
def test_two_rank_shard_and_reduce(cfg, n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # shards are contiguous, disjoint and cover [0, n)
    assert res[0][1] == 0 and res[0][2] == res[1][1] and res[1][2] == n
    # reduced counters equal the single-process counters of the whole batch
    x = workloads.host_rows(cfg, 0, n)
    prec = "single" if x.dtype == np.float32 else "double"
    want = workloads.row_stats_host(x, kernel_args(preset(prec))).astype(np.int64).tolist()
    assert res[0][3] == want and res[1][3] == want
    assert sum(want) == n
    # max over ranks
    assert res[0][4] == 0.5 and res[1][4] == 0.5


@pytest.mark.parametrize("n,world", [(0, 3), (1, 2), (7, 8), (1 << 30, 8), (1000003, 7)])
def test_shard_range_properties(n, world):
    spans = [multigpu.shard_range(n, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        multigpu.shard_range(n, world, world)
