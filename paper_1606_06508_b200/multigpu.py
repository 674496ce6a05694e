"""Multi-GPU host logic: row sharding, max-over-ranks timing and the validation reduce.

Rows are independent (no cross-row arithmetic anywhere in _kernels.pyx:167-412), so the
batch shards into contiguous row ranges, one per rank (one process per GPU), with no
collective on the data path.  The only collectives are two tiny all-reduces after the
timed region: MAX of the elapsed time (the job takes as long as its slowest rank) and
SUM of six row-class counters (validation statistics).  Works with any
torch.distributed backend: NCCL on the B200 box, gloo for the CPU tests.

For a single process driving several GPUs with host arrays, ``host_devices([...])``
shards every host-array call over those devices (fn_host_run_multi: one host thread
and one PCIe link per device).
"""

from __future__ import annotations

from paper_1606_06508_b200.batch import host_devices  # noqa: F401  (re-export)

COUNTER_NAMES = ("nan", "inf", "zero", "below_tau_min", "above_tau_max", "in_band")


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced shard [lo, hi) of rank; the first n % world ranks get one more."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    if n_total < 0:
        raise ValueError("n_total must be >= 0")
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device=None) -> float:
    """MAX of a per-rank scalar over the default process group (identity without one)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_counts(counts):
    """In-place SUM all-reduce of an int64 counter tensor; returns it as a list of ints."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(counts)
    return [int(v) for v in counts.cpu().tolist()]


def shard_counts_device(x, ka):
    """Six row-class counters of a device shard (CUDA kernel fn_row_stats), as int64."""
    import torch

    from paper_1606_06508_b200 import workloads

    counts = torch.zeros(6, dtype=torch.int64, device=x.device)
    workloads.row_stats_device(x, ka, counts.view(torch.uint64))
    return counts


def gpu_local_cpus(device_index: int) -> set[int] | None:
    """CPUs of the NUMA node the GPU's PCIe link hangs off (sysfs), or None if unknown."""
    import os

    import torch

    try:
        prop = torch.cuda.get_device_properties(device_index)
        bus = f"{prop.pci_domain_id:04x}:{prop.pci_bus_id:02x}:{prop.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
            node = int(f.read().strip())
        if node < 0:
            return None
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            spec = f.read().strip()
    except Exception:
        return None
    cpus: set[int] = set()
    for part in spec.split(","):
        lo, _, hi = part.partition("-")
        cpus.update(range(int(lo), int(hi or lo) + 1))
    allowed = os.sched_getaffinity(0)
    return (cpus & allowed) or None


class numa_local:
    """Context manager: run (and first-touch page-locked host buffers) on the CPUs local
    to the GPU, so host <-> device copies do not cross the socket interconnect; the
    previous affinity is restored on exit.  A no-op where the topology is unknown."""

    def __init__(self, device_index: int):
        self.device_index = device_index
        self.saved = None
        self.cpus = None

    def __enter__(self):
        import os

        self.cpus = gpu_local_cpus(self.device_index)
        if self.cpus:
            self.saved = os.sched_getaffinity(0)
            os.sched_setaffinity(0, self.cpus)
        return self

    def __exit__(self, *exc):
        import os

        if self.saved is not None:
            os.sched_setaffinity(0, self.saved)
