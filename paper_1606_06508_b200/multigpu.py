"""Multi-GPU host logic: row sharding, max-over-ranks timing and the validation reduce.

Rows are independent (no cross-row arithmetic anywhere in _kernels.pyx:167-412), so the
batch shards into contiguous row ranges, one per rank (one process per GPU), with no
collective on the data path.  The only collectives are two tiny all-reduces after the
timed region: MAX of the elapsed time (the job takes as long as its slowest rank) and
SUM of six row-class counters (validation statistics).  Works with any
torch.distributed backend: NCCL on the B200 box, gloo for the CPU tests.

For a single process driving several GPUs there are two routes.  Host arrays:
``host_devices([...])`` shards every host-array call over those devices
(fn_host_run_multi: one host thread and one PCIe link per device).  Device-resident
rows: :class:`DeviceShards` keeps one contiguous row shard per GPU, and
``normalize_sharded`` / ``norm_sharded`` / ``run_sharded`` run every shard on a stream
of its own device from one host thread (fn_run_sharded; BASELINE.json north star (c):
"device-resident inputs, one stream per device and no collective on the data path").
"""

from __future__ import annotations

from typing import NamedTuple

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


# --------------------------------------------------------------------------------------
# one process, several GPUs, device-resident shards
# --------------------------------------------------------------------------------------
class DeviceShards:
    """One ``[N, w]`` (or ``[N]``) array as contiguous row shards, shard k resident on GPU
    ``devices[k]`` of this process (balanced like ``shard_range``).  A device may appear
    more than once (two shards on ``cuda:0`` exercise the driver on a one-GPU box)."""

    def __init__(self, tensors):
        tensors = list(tensors)
        if not tensors:
            raise ValueError("need at least one shard")
        t0 = tensors[0]
        for t in tensors:
            if not t.is_cuda:
                raise TypeError("shards must be CUDA tensors")
            if t.dtype != t0.dtype or t.shape[1:] != t0.shape[1:]:
                raise TypeError("shards must share dtype and row shape")
        self.tensors = tensors

    # -- constructors ------------------------------------------------------------------
    @staticmethod
    def _devices(devices):
        import torch

        devs = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d) for d in devices]
        if not devs:
            raise ValueError("need at least one device")
        return devs

    @classmethod
    def empty(cls, rows: int, width: int, dtype, devices) -> "DeviceShards":
        """Uninitialised shards of a ``[rows, width]`` array (``width`` 0: ``[rows]``)."""
        import torch

        devs = cls._devices(devices)
        out = []
        for k, d in enumerate(devs):
            lo, hi = shard_range(rows, k, len(devs))
            shape = (hi - lo, width) if width else (hi - lo,)
            out.append(torch.empty(shape, dtype=dtype, device=d))
        return cls(out)

    @classmethod
    def generate(cls, cfg: int, rows: int, devices, seed: int | None = None) -> "DeviceShards":
        """Rows [0, rows) of a BASELINE.json config, each shard generated in its own
        GPU's HBM from the global row index (workloads.generate_device, row0 = shard
        start), so the shards together equal the one-device batch bit for bit."""
        import torch

        from paper_1606_06508_b200 import workloads

        c = workloads.CONFIGS[cfg]
        dt = torch.float64 if c.dtype == "float64" else torch.float32
        sh = cls.empty(rows, c.dim, dt, devices)
        for k, t in enumerate(sh.tensors):
            lo, _ = shard_range(rows, k, len(sh.tensors))
            with torch.cuda.device(t.device):
                workloads.generate_device(cfg, t, row0=lo, seed=seed)
        return sh

    @classmethod
    def scatter(cls, x, devices) -> "DeviceShards":
        """Shards of a host (numpy / CPU tensor) or CUDA array, copied to the devices."""
        import numpy as np
        import torch

        if isinstance(x, np.ndarray):
            x = torch.from_numpy(x)
        devs = cls._devices(devices)
        out = []
        for k, d in enumerate(devs):
            lo, hi = shard_range(int(x.shape[0]), k, len(devs))
            out.append(x[lo:hi].to(d, copy=True).contiguous())
        return cls(out)

    # -- views -------------------------------------------------------------------------
    @property
    def rows(self) -> int:
        return sum(int(t.shape[0]) for t in self.tensors)

    @property
    def devices(self) -> list[int]:
        return [t.device.index for t in self.tensors]

    @property
    def dtype(self):
        return self.tensors[0].dtype

    def __len__(self) -> int:
        return len(self.tensors)

    def __getitem__(self, k):
        return self.tensors[k]

    def gather(self):
        """The whole array as one CPU tensor (tests and small results)."""
        import torch

        return torch.cat([t.cpu() for t in self.tensors], dim=0)


class ShardedOut(NamedTuple):
    head: DeviceShards            # r (inv for scale)
    body: DeviceShards | None     # unit (scaled for scale); None for norm
    sq: DeviceShards | None       # squared norm (normalize*_sq only)
    elapsed_ms: list              # device time of each shard's launch (CUDA events on its stream)


def run_sharded(op: int, dim: int, x: DeviceShards, ka_arr=None, out=None) -> ShardedOut:
    """Kernel family ``op`` over device-resident shards: one launch per shard, each on a
    library-owned stream of its device, all enqueued before any is waited for; returns
    when every shard has finished.  Each shard waits for torch's current stream on its
    device (the producer of its rows).  ``out``: (head[, body][, sq]) DeviceShards with
    the same row split, reused instead of allocating."""
    import ctypes

    import torch

    from paper_1606_06508_b200 import _lib, batch

    if not isinstance(x, DeviceShards):
        raise TypeError("x must be DeviceShards")
    m = len(x)
    for t in x.tensors:
        if t.ndim != 2 or t.shape[1] != dim:
            raise ValueError(f"expected shards of shape [n, {dim}], got {tuple(t.shape)}")
    xs = [t if t.is_contiguous() else t.contiguous() for t in x.tensors]
    w0, w1, w2 = batch.widths(op, dim)
    widths = [w0] + ([w1] if w1 else []) + ([w2] if w2 else [])
    if out is not None:
        out = tuple(out)
        if len(out) != len(widths):
            raise ValueError(f"out must hold {len(widths)} DeviceShards")
    results = []
    for j, w in enumerate(widths):
        if out is not None and out[j] is not None:
            o = out[j]
            if not isinstance(o, DeviceShards) or len(o) != m:
                raise TypeError("out entries must be DeviceShards with one shard per input shard")
            for t, xi in zip(o.tensors, xs):
                shape = batch._shape(int(xi.shape[0]), w)
                if t.device != xi.device or t.dtype != xi.dtype or tuple(t.shape) != shape or not t.is_contiguous():
                    raise ValueError("out shard does not match its input shard (device, dtype, shape, dense)")
            results.append(o)
        else:
            results.append(DeviceShards([xi.new_empty(batch._shape(int(xi.shape[0]), w)) for xi in xs]))
    head = results[0]
    body = results[1] if w1 else None
    sq = results[-1] if w2 else None
    dcode = _lib.F64 if x.dtype == torch.float64 else _lib.F32 if x.dtype == torch.float32 else None
    if dcode is None:
        raise TypeError(f"unsupported dtype {x.dtype}")
    arr = (lambda vals: (ctypes.c_void_p * m)(*vals))
    xp = arr([t.data_ptr() for t in xs])
    hp = arr([t.data_ptr() for t in head.tensors])
    bp = arr([t.data_ptr() for t in body.tensors]) if body is not None else None
    qp = arr([t.data_ptr() for t in sq.tensors]) if sq is not None else None
    ns = (ctypes.c_int64 * m)(*[int(t.shape[0]) for t in xs])
    devs = (ctypes.c_int * m)(*[t.device.index for t in xs])
    after = arr([torch.cuda.current_stream(t.device).cuda_stream for t in xs])
    ms = (ctypes.c_float * m)()
    addr = (lambda a: None if a is None else ctypes.addressof(a))
    rc = _lib.lib().fn_run_sharded(op, dim, dcode, m, addr(devs), addr(xp), addr(ns), addr(hp), addr(bp), addr(qp),
                                   None if ka_arr is None else ka_arr.ctypes.data, addr(after), addr(ms))
    _lib.check(rc, "fn_run_sharded")
    return ShardedOut(head, body, sq, [float(v) for v in ms])


def _ka_for(p, x: DeviceShards):
    from paper_1606_06508_b200.scale import check_precision, kernel_args_array

    for t in x.tensors:
        check_precision(p, t)
    return kernel_args_array(p)


def normalize_sharded(p, x: DeviceShards, out=None) -> ShardedOut:
    """normalize{n} (normalize.py:51-89 of the reference, one row per call there) over
    device-resident shards on several GPUs: r and unit come back as DeviceShards."""
    from paper_1606_06508_b200 import _lib

    return run_sharded(_lib.OP_NORMALIZE, int(x[0].shape[1]), x, _ka_for(p, x), out)


def norm_sharded(p, x: DeviceShards, out=None) -> ShardedOut:
    """norm{n} over device-resident shards (only r is written)."""
    from paper_1606_06508_b200 import _lib

    return run_sharded(_lib.OP_NORM, int(x[0].shape[1]), x, _ka_for(p, x), out)
