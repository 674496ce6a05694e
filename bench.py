#!/usr/bin/env python
"""Benchmark: normalized vectors/s and achieved HBM GB/s vs peak (3-D fp64) on 1-8 B200.

Workload (BASELINE.json configs[4], the config the headline metric is quoted on):
3-D float64 vectors, N = 2^30 rows in total (24 GiB of input), sharded evenly over the
ranks (strong scaling: the total is fixed, every rank owns N/world contiguous rows),
exponents uniform in [-1020, 1020], mantissas uniform in [1, 2), random signs, 0.5 %
rows with one component near DBL_MAX, 0.5 % rows of subnormals.  One step = one pass of
normalize3 (scaling algorithm: r[N] and unit[N, 3]) over every rank's shard.

* value  -- device-resident: inputs generated in HBM before timing; K back-to-back
            launches timed with CUDA events on the launching stream, barrier + sync on
            both sides, max over ranks.  Inputs (24 GiB/world) exceed L2 (126 MB), so no
            L2 flush is needed between steps.
* e2e    -- the same metric through the public API with HOST buffers
            (fn.normalize3(p, pinned_numpy, out=...) -> fn_host_run): every step copies
            the shard's input H2D and r + unit D2H inside the timed region.
* e2e_default_api -- the default drop-in call, fn.normalize3(p, numpy_rows): pageable
            input, no out= (outputs from the library's page-locked pool), each step's
            result dropped before the next, as a caller's loop over batches does.
* roofline -- algorithmic bytes per launch (56 B/row x rows) / mean launch duration,
            against MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline -- (rank 0, N = 1 only) the reference's own compiled timing loop
            (oracle/_ref, `loop_scaling3_f64`, checksum only) on all host cores over a
            bounded sample of the same workload; the oracle port if _ref is absent.

`--impl reference` times only that CPU reference path (rank 0; other ranks exit 0).
Run: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                     [--rows R] [--dist-backend nccl|gloo]
--gpus N > 1 without a torchrun environment launches N ranks itself (torch.distributed.run
on 127.0.0.1) and refuses to put two NCCL ranks on one GPU.  --rows changes the total
(default 2^30); --dist-backend gloo lets test ranks share a GPU.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "normalized vectors/sec and achieved HBM GB/s vs peak (3D fp64), 1/2/4/8 B200"
UNIT = "vectors/s"
CFG = 5
ROWS_TOTAL = 1 << 30
WORKLOAD = ("cfg5: 3D f64 normalize3 (scaling algorithm), N=2^30 rows total, "
            "exponents U[-1020,1020], 0.5% near-DBL_MAX rows, 0.5% all-subnormal rows")


def _workload(rows: int) -> str:
    if rows == ROWS_TOTAL:
        return WORKLOAD
    return WORKLOAD.replace("N=2^30 rows total", f"N={rows} rows total (--rows; BASELINE config 5 is 2^30)")


DIM = 3
BYTES_PER_ROW = 56  # 24 in + 8 (r) + 24 (unit)
NOMINAL_HBM_GBS = 7700.0  # B200_PROFILING.md hardware table (HGX figure)
CPU_SAMPLE_ROWS = 1 << 26


def _peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def _host_rows_that_fit(world: int) -> int:
    """Rows per rank whose pinned e2e buffers (56 B/row) fit in MemAvailable with 30 %
    to spare, all ranks of this host together (a multiple of 2^20, at least 2^20)."""
    try:
        with open("/proc/meminfo") as f:
            avail = next(int(ln.split()[1]) * 1024 for ln in f if ln.startswith("MemAvailable:"))
    except Exception:
        return ROWS_TOTAL
    rows = int(avail / 1.3 / BYTES_PER_ROW / max(1, world))
    return max(1 << 20, (rows >> 20) << 20)


def _traffic_per_row():
    """Per-row DRAM bytes of the top kernel from the committed ncu capture, if any."""
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["normalize3_f64"]["dram_bytes_per_row"]), d["normalize3_f64"].get("source")
    except Exception:
        return None, None


class ClockSampler:
    """SM clocks and throttle reasons sampled every 10 ms (NVML) during the timed region.

    Falls back to `nvidia-smi -lms 200` when pynvml is unavailable."""

    _REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int, period_s: float = 0.01):
        self.index = index
        self.period = period_s
        self.sm: list[float] = []
        self.smax = None
        self.reasons: set[str] = set()
        self._stop = threading.Event()
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self._nvml = (pynvml, h)
        except Exception:
            self._nvml = None
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _sample_nvml(self):
        pynvml, h = self._nvml
        self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
        try:
            bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            bits = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        for mask, name in self._REASONS.items():
            if bits & mask:
                self.reasons.add(name)

    def _run(self):
        if self._nvml is not None:
            while not self._stop.is_set():
                try:
                    self._sample_nvml()
                except Exception:
                    break
                self._stop.wait(self.period)
            return
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                     "--format=csv,noheader,nounits", "-lms", "200"],
                                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            return
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        while not self._stop.is_set():
            line = proc.stdout.readline()
            if not line:
                break
            parts = [p.strip() for p in line.split(",")]
            try:
                self.sm.append(float(parts[0]))
                self.smax = float(parts[1])
            except (ValueError, IndexError):
                continue
            for name, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    self.reasons.add(name)
        proc.terminate()

    def __exit__(self, *exc):
        if self._nvml is not None:
            try:  # one last sample so very short regions still get one
                self._sample_nvml()
            except Exception:
                pass
        self._stop.set()
        self._t.join(timeout=5)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.smax, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.smax,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


from paper_1606_06508_b200.multigpu import shard_range  # noqa: E402


def _lib_handle():
    from paper_1606_06508_b200 import _lib

    return _lib.lib()


# --------------------------------------------------------------------------------------
# CPU reference path (reference's compiled loop, all host cores)
# --------------------------------------------------------------------------------------
def cpu_reference_rate(x: np.ndarray, ka, reps: int = 3):
    """Best-of-reps vectors/s of the reference timing loop over x on all host cores."""
    import oracle

    threads = len(os.sched_getaffinity(0))
    ref = oracle.ref_module()
    n = x.shape[0]
    bounds = [shard_range(n, t, threads) for t in range(threads)]
    flat = np.ascontiguousarray(x.reshape(-1))
    if ref is not None:
        kind = "reference"
        loop = ref.loop_scaling3_f64

        def work(lo, hi, out, t):
            rows = hi - lo
            mask = (1 << max(0, (rows - 1).bit_length())) - 1
            out[t] = loop(flat[lo * 3: hi * 3], rows, mask, *ka)
    else:  # oracle port (same loop body, C restatement)
        kind = "port"

        def work(lo, hi, out, t):
            rows = hi - lo
            mask = (1 << max(0, (rows - 1).bit_length())) - 1
            out[t] = oracle.loop(oracle.ALGO_SCALING, x[lo:hi], rows, mask, ka)

    best = None
    for _ in range(reps):
        out = [0.0] * threads
        ts = [threading.Thread(target=work, args=(lo, hi, out, t)) for t, (lo, hi) in enumerate(bounds)]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return n / best, threads, kind, best


def cpu_detail(ka64, ka32, sample_rows: int = 1 << 22):
    """The CPU legs SURVEY §8(d) lists beside the T-thread reference loop (rank 0, N = 1):
    the same reference loop on one thread; the oracle restatement *with output stores*
    on all threads (a port, labelled so); and the reference loop on a sample of every
    other BASELINE config, to pair each GPU config with its CPU rate."""
    import oracle
    from paper_1606_06508_b200 import workloads

    ref = oracle.ref_module()
    threads = len(os.sched_getaffinity(0))
    out = {"cores_available": threads, "sample_rows": sample_rows}

    def best_time(fn, reps=3):
        best = None
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        return best

    x5 = workloads.host_rows(CFG, 0, sample_rows)
    if ref is not None:
        flat = np.ascontiguousarray(x5.reshape(-1))
        mask = (1 << (sample_rows - 1).bit_length()) - 1
        t = best_time(lambda: ref.loop_scaling3_f64(flat, sample_rows, mask, *ka64))
        out["reference_loop_1_thread"] = {"value": sample_rows / t, "unit": UNIT, "cores": 1,
                                          "kind": "reference", "sample": f"cfg5 rows [0, {sample_rows})"}
    t = best_time(lambda: oracle.run(oracle.OP_NORMALIZE, x5, np.array(ka64), threads=threads))
    out["port_with_stores"] = {"value": sample_rows / t, "unit": UNIT, "cores": threads, "kind": "port",
                               "sample": f"cfg5 rows [0, {sample_rows}), oracle normalize3 writing r and unit"}
    per_cfg = {}
    for cfg in (1, 2, 3, 4):
        c = workloads.CONFIGS[cfg]
        n = min(sample_rows, c.rows)
        xc = workloads.host_rows(cfg, 0, n)
        single = c.dtype == "float32"
        rate, thr, kind, _ = cpu_loop_rate(xc, c.dim, single, ka32 if single else ka64, ref, threads)
        per_cfg[str(cfg)] = {"value": rate, "unit": UNIT, "cores": thr, "kind": kind,
                             "sample": f"cfg{cfg} rows [0, {n}), loop_scaling{c.dim}_{'f32' if single else 'f64'}"}
    out["reference_loop_per_config"] = per_cfg
    return out


def cpu_loop_rate(x: np.ndarray, dim: int, single: bool, ka, ref, threads: int, reps: int = 3):
    """Best-of-reps vectors/s of the reference's scaling loop of any config on all cores."""
    import oracle

    n = x.shape[0]
    bounds = [shard_range(n, t, threads) for t in range(threads)]
    flat = np.ascontiguousarray(x.reshape(-1))
    loop = getattr(ref, f"loop_scaling{dim}_{'f32' if single else 'f64'}") if ref is not None else None

    def work(lo, hi):
        rows = hi - lo
        mask = (1 << max(0, (rows - 1).bit_length())) - 1
        if loop is not None:
            loop(flat[lo * dim: hi * dim], rows, mask, *ka)
        else:
            oracle.loop(oracle.ALGO_SCALING, x[lo:hi], rows, mask, ka)

    best = None
    for _ in range(reps):
        ts = [threading.Thread(target=work, args=b) for b in bounds]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return n / best, threads, "reference" if loop is not None else "port", best


def run_reference_arm(args):
    rank, world, _ = _dist_env()
    if rank != 0:
        return 0
    from paper_1606_06508_b200 import workloads
    from paper_1606_06508_b200.params import preset
    from paper_1606_06508_b200.scale import kernel_args

    ka = kernel_args(preset("double"))
    x = workloads.host_rows(CFG, 0, CPU_SAMPLE_ROWS)
    for _ in range(args.warmup):
        cpu_reference_rate(x, ka, reps=1)
    rates = []
    threads = kind = None
    t_total = 0.0
    for _ in range(args.steps):
        rate, threads, kind, dt = cpu_reference_rate(x, ka, reps=1)
        rates.append(rate)
        t_total += dt
    value = statistics.median(rates)
    sample = (f"cfg5 rows [0, {CPU_SAMPLE_ROWS}) ({CPU_SAMPLE_ROWS * 24 >> 20} MiB of input), "
              f"reference loop_scaling3_f64 (checksum, no output stores), "
              f"{threads} threads x contiguous shards, median of {args.steps} passes")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_total / max(1, args.steps),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded cfg5 generator, host restatement)",
        "config": {"workload": _workload(args.rows), "rows_total": args.rows,
                   "rows_sampled": CPU_SAMPLE_ROWS,
                   "sample": "each step: a bounded CPU sample of the workload (rows_sampled rows)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------------------
# the other BASELINE configs (informational, measured after the timed region)
# --------------------------------------------------------------------------------------
OTHER_CONFIGS = {  # config -> [(public API call, algorithmic bytes per row)]
    1: [("normalize3", 56)],
    2: [("normalize2", 40), ("quotient2", 40)],
    3: [("normalize4_sq", 80), ("normalize4_rotation", 144)],
    4: [("normalize3", 28), ("quotient3_robust", 28)],
    5: [("quotient3_robust", 56)],  # the headline's comparison variant (division-bound)
}


def _batch_stream_rate(fn, p, x, bytes_per_row, peak, reps, sets=8, per_set=4):
    """Config 1 as a stream of 1e6-row batches: a CUDA graph of sets x per_set launches
    that cycles over `sets` distinct input/output buffer sets (8 x 56 MB > the 126 MB
    L2, so every launch streams from HBM without a flush kernel).  Per-launch time =
    graph time / launches; the launch latency a lone launch pays is hidden."""
    import torch

    n = x.shape[0]
    bufs = []
    for _ in range(sets):
        xi = torch.empty_like(x)
        xi.copy_(x)
        bufs.append((xi, torch.empty(n, dtype=x.dtype, device=x.device), torch.empty_like(x)))
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream(device=x.device)
    s.wait_stream(torch.cuda.current_stream(x.device))
    with torch.cuda.stream(s):
        for xi, ri, ui in bufs:
            fn.normalize3(p, xi, out=(ri, ui))
        torch.cuda.synchronize(x.device)
        with torch.cuda.graph(g, stream=s):
            for _ in range(per_set):
                for xi, ri, ui in bufs:
                    fn.normalize3(p, xi, out=(ri, ui))
    torch.cuda.synchronize(x.device)
    launches = sets * per_set
    # the same launches issued eagerly through the public API (no graph): host cost per
    # call (~10 us) against ~10 us of kernel
    eager = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream(x.device)
        e0.record(cur)
        for _ in range(per_set):
            for xi, ri, ui in bufs:
                fn.normalize3(p, xi, out=(ri, ui))
        e1.record(cur)
        torch.cuda.synchronize(x.device)
        eager.append(e0.elapsed_time(e1) / 1e3 / launches)
    t_eager = statistics.median(eager)
    times = []
    for _ in range(max(reps, 3) + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream(x.device)
        e0.record(cur)
        g.replay()
        e1.record(cur)
        torch.cuda.synchronize(x.device)
        times.append(e0.elapsed_time(e1) / 1e3 / launches)
    t = statistics.median(times[1:])
    # the same 32 batches as one grouped call (normalize_many -> fn_run_many: one launch),
    # graph-replayed like the launches above and eagerly through the public API
    xs = [b[0] for _ in range(per_set) for b in bufs]
    outs = [(b[1], b[2]) for _ in range(per_set) for b in bufs]
    gm = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn.normalize_many(p, xs, out=outs)
        torch.cuda.synchronize(x.device)
        with torch.cuda.graph(gm, stream=s):
            fn.normalize_many(p, xs, out=outs)
    torch.cuda.synchronize(x.device)

    def per_batch(run):
        ts = []
        for _ in range(max(reps, 3) + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cur = torch.cuda.current_stream(x.device)
            e0.record(cur)
            run()
            e1.record(cur)
            torch.cuda.synchronize(x.device)
            ts.append(e0.elapsed_time(e1) / 1e3 / launches)
        return statistics.median(ts[1:])

    t_many = per_batch(gm.replay)
    t_many_eager = per_batch(lambda: fn.normalize_many(p, xs, out=outs))
    del g, gm, bufs, xs, outs
    many = {"api": "normalize_many(p, 32 batches) -> fn_run_many, one launch",
            "ms_per_batch": t_many * 1e3, "vectors_per_s": n / t_many,
            "frac": n * bytes_per_row / t_many / 1e9 / peak,
            "eager_public_api": {"ms_per_batch": t_many_eager * 1e3, "vectors_per_s": n / t_many_eager,
                                 "frac": n * bytes_per_row / t_many_eager / 1e9 / peak}}
    return {"launches_per_graph": launches, "buffer_sets": sets, "grouped_call": many,
            "bytes_cycled": sets * n * bytes_per_row, "ms_per_launch": t * 1e3,
            "vectors_per_s": n / t, "GB_per_s": n * bytes_per_row / t / 1e9,
            "frac": n * bytes_per_row / t / 1e9 / peak,
            "eager_public_api": {"ms_per_launch": t_eager * 1e3, "vectors_per_s": n / t_eager,
                                 "frac": n * bytes_per_row / t_eager / 1e9 / peak}}


_ISSUE_KEYS = {("quotient2", 2): "quotient2_f64_cfg2", ("normalize2", 2): "normalize2_f64_cfg2",
               ("quotient3_robust", 4): "quotient3_f32_cfg4", ("quotient3_robust", 5): "quotient3_f64_cfg5"}


def _issue_roofline(name: str, cfg: int, rows: int, t: float, clock_mhz):
    """Instruction-issue roofline of a kernel: warp instructions per row (from the
    committed ncu pass, profiles/ncu_issue.json, tools/ncu_issue.sh) x rows over the
    issue peak -- one warp instruction per SMSP per cycle, 4 SMSPs x 148 SMs at the SM
    clock sampled during this run -- against the measured launch time."""
    key = _ISSUE_KEYS.get((name, cfg))
    try:
        with open(os.path.join(REPO, "profiles", "ncu_issue.json")) as f:
            d = json.load(f)[key]
    except Exception:
        return None
    clk = (clock_mhz or 1965.0) * 1e6
    peak = 148 * 4 * clk  # warp instructions per second
    achieved = d["warp_inst_per_row"] * rows / t
    fp64 = d["fp64_warp_inst_per_row"] * rows / t
    return {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "warp inst/s", "frac": achieved / peak,
            "warp_inst_per_row": d["warp_inst_per_row"], "fp64_warp_inst_per_row": d["fp64_warp_inst_per_row"],
            "fp64_pipe_frac": fp64 / (peak / 2),  # the FP64 pipe takes a warp instruction every 2 cycles
            "clock_mhz": clk / 1e6, "source": d["source"]}


def measure_other_configs(dev, reps: int = 5, clocks_mhz=None):
    """Each BASELINE config's kernels through the public API: rows generated in HBM, L2
    evicted (a 512 MiB read) before every timed launch, CUDA events on the launching
    stream, median of `reps`."""
    import torch

    import paper_1606_06508_b200 as fn
    from paper_1606_06508_b200 import workloads

    peak, _ = _peaks()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    out = []
    for cfg, calls in OTHER_CONFIGS.items():
        c = workloads.CONFIGS[cfg]
        dt = torch.float64 if c.dtype == "float64" else torch.float32
        p = fn.preset("double" if dt == torch.float64 else "single")
        x = torch.empty((c.rows, c.dim), dtype=dt, device=dev)
        workloads.generate_device(cfg, x)
        for name, bpr in calls:
            f = getattr(fn, name)
            call = (lambda: f(x)) if name.startswith("quotient") else (lambda: f(p, x))
            for _ in range(3):
                call()
            times = []
            for _ in range(reps if c.rows > (1 << 24) else 6 * reps):  # ~10 us launches: more samples
                flush.sum(dtype=torch.int32)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                call()
                e1.record(stream)
                torch.cuda.synchronize(dev)
                times.append(e0.elapsed_time(e1) / 1e3)
            t = statistics.median(times)
            out.append({"config": cfg, "kernel": name, "rows": c.rows, "dtype": c.dtype,
                        "vectors_per_s": c.rows / t, "GB_per_s": c.rows * bpr / t / 1e9,
                        "frac": c.rows * bpr / t / 1e9 / peak, "ms": t * 1e3})
            issue = _issue_roofline(name, cfg, c.rows, t, clocks_mhz)
            if issue is not None:
                out[-1]["issue_roofline"] = issue
            if cfg == 1:
                out[-1]["stream_of_batches"] = _batch_stream_rate(fn, p, x, bpr, peak, reps)
        del x
        torch.cuda.empty_cache()
    return out


# --------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1606_06508_b200 as fn
    from paper_1606_06508_b200 import multigpu, workloads

    rank, world, local = _dist_env()
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    ndev = torch.cuda.device_count()
    if args.dist_backend == "nccl" and world > ndev:
        raise SystemExit(f"{world} NCCL ranks need {world} GPUs, {ndev} visible")
    torch.cuda.set_device(local % ndev)
    dev = torch.device("cuda", local % ndev)
    # under torchrun (RANK set) the process group is created even for a single rank, so
    # the same barrier / max-reduce / counter-reduce code runs at every N.  NCCL on the
    # B200 box; gloo (collectives on host tensors) when a test puts ranks on one GPU.
    distributed = "RANK" in os.environ and "MASTER_ADDR" in os.environ
    if distributed:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    cdev = dev if args.dist_backend == "nccl" else torch.device("cpu")  # collective tensors live here
    rows_total = args.rows

    def barrier():
        if distributed:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        return multigpu.max_over_ranks(v, device=cdev)

    p = fn.preset("double")
    ka = fn.kernel_args(p)
    lo, hi = shard_range(rows_total, rank, world)
    n = hi - lo

    x = torch.empty((n, DIM), dtype=torch.float64, device=dev)
    workloads.generate_device(CFG, x, row0=lo)
    r = torch.empty((n,), dtype=torch.float64, device=dev)
    u = torch.empty((n, DIM), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    # ---------------- device-resident throughput ----------------
    for _ in range(args.warmup):
        fn.normalize3(p, x, out=(r, u))
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            fn.normalize3(p, x, out=(r, u))
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    t_dev = max_over_ranks(ev0.elapsed_time(ev1) / 1e3)
    value = rows_total * args.steps / t_dev
    per_launch_s = t_dev / args.steps  # one kernel launch per step per rank
    achieved_gbs = (n * BYTES_PER_ROW) / per_launch_s / 1e9 if world == 1 else \
        (rows_total // world * BYTES_PER_ROW) / per_launch_s / 1e9

    # ---------------- validation counters: one small NCCL all-reduce ----------------
    counts_h = multigpu.reduce_counts(multigpu.shard_counts_device(x, ka).to(cdev))
    torch.cuda.synchronize(dev)

    # ---------------- single-process multi-GPU driver (informational, N = 1) ----------------
    # The same rows as two device-resident shards through fn_run_sharded, both on this
    # rank's GPU (the rows live here): this measures the driver's overhead against the
    # one-launch step above, not scaling.  Shards are views of x / r / u: nothing is allocated.
    sharded = None
    if world == 1 and not args.no_configs:
        try:
            devs = [local % ndev] * 2
            cuts = [shard_range(n, k, len(devs)) for k in range(len(devs))]
            xs_sh = multigpu.DeviceShards([x[lo:hi] for lo, hi in cuts])
            out_sh = (multigpu.DeviceShards([r[lo:hi] for lo, hi in cuts]),
                      multigpu.DeviceShards([u[lo:hi] for lo, hi in cuts]))
            for _ in range(2):
                multigpu.normalize_sharded(p, xs_sh, out=out_sh)
            k0 = _lib_handle().fn_launch_count()
            ms, wall = [], []
            for _ in range(5):
                torch.cuda.synchronize(dev)
                t0 = time.perf_counter()
                res = multigpu.normalize_sharded(p, xs_sh, out=out_sh)
                wall.append(time.perf_counter() - t0)
                ms.append(max(res.elapsed_ms))
            t_sh = statistics.median(ms) / 1e3
            sharded = {"api": "multigpu.normalize_sharded(p, DeviceShards) -> fn_run_sharded (one stream per shard)",
                       "devices": devs, "rows": n, "ms_device_max_over_shards": t_sh * 1e3,
                       "ms_host_wall": statistics.median(wall) * 1e3, "vectors_per_s": n / t_sh,
                       "GB_per_s": n * BYTES_PER_ROW / t_sh / 1e9,
                       "gpu_launches": int(_lib_handle().fn_launch_count() - k0)}
            del xs_sh, out_sh, res
        except Exception as exc:  # informational only: never lose the headline line
            sharded = {"error": str(exc)}

    # ---------------- end to end through the public API, host buffers ----------------
    # Every rank pins its shard's input and outputs (56 B/row).  If the host cannot hold
    # all ranks' shards with a 30 % margin, the e2e pass runs on the largest prefix of
    # each shard that fits (recorded as e2e.rows_per_gpu); the rate stays per row.
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    e2e_rows = min(n, _host_rows_that_fit(world))
    if distributed:
        t = torch.tensor([e2e_rows], dtype=torch.int64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        e2e_rows = int(t.item())
    e2e_error = None
    numa = multigpu.numa_local(local)  # pin + copy from the GPU's own socket
    numa.__enter__()
    try:  # page-locked through the library (released to the OS as soon as they are dropped)
        xn = fn.host_empty((e2e_rows, DIM))
        torch.from_numpy(xn).copy_(x[:e2e_rows])
        rn = fn.host_empty((e2e_rows,))
        un = fn.host_empty((e2e_rows, DIM))
    except Exception as exc:  # pragma: no cover - host-dependent
        e2e_error = f"pinned allocation failed: {exc}"
    if distributed:  # every rank skips the e2e pass if any rank could not pin
        flag = torch.tensor([0 if e2e_error is None else 1], dtype=torch.int64, device=cdev)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        if int(flag.item()) and e2e_error is None:
            e2e_error = "another rank could not pin its e2e buffers"
    del x, r, u
    torch.cuda.empty_cache()
    t_e2e = float("nan")
    L = _lib_handle()
    e2e_launches = None
    if e2e_error is None:
        w = min(e2e_rows, 1 << 20)
        fn.normalize3(p, xn[:w], out=(rn[:w], un[:w]))  # warm the staging pool
        barrier()
        k0 = L.fn_launch_count()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            fn.normalize3(p, xn, out=(rn, un))
        t1 = time.perf_counter()
        e2e_launches = int(L.fn_launch_count() - k0)  # counted by the library itself
        barrier()
        t_e2e = max_over_ranks(t1 - t0)
    # ---------------- end to end, the default call: fn.normalize3(p, numpy_rows) ----------------
    # Pageable numpy input, outputs allocated by the library (page-locked pool), the result
    # dropped after each step as a caller's loop over batches would.
    default_api = None
    if not args.no_default_api and e2e_error is None:
        try:
            del rn, un  # the caller-provided outputs go; the library allocates its own
            xp = np.empty((e2e_rows, DIM), dtype=np.float64)  # plain pageable numpy rows
            np.copyto(xp, xn)
            del xn
            res = fn.normalize3(p, xp)  # warm-up: pins the output blocks once
            del res
            barrier()
            k0 = L.fn_launch_count()
            pool0 = (fn.batch.pinned_pool.allocs, fn.batch.pinned_pool.reuses)
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                res = fn.normalize3(p, xp)
                del res
            t1 = time.perf_counter()
            launches_d = int(L.fn_launch_count() - k0)
            barrier()
            t_def = max_over_ranks(t1 - t0)
            default_api = {
                "value": e2e_rows * world * e2e_steps / t_def, "unit": UNIT,
                "h2d_bytes_per_step": e2e_rows * world * DIM * 8,
                "d2h_bytes_per_step": e2e_rows * world * (DIM + 1) * 8,
                "rows_per_gpu": e2e_rows, "steps": e2e_steps, "ms_per_step": 1e3 * t_def / e2e_steps,
                "api": "paper_1606_06508_b200.normalize3(p, numpy [N,3]) with pageable input and no out= "
                       "-> fn_host_run (outputs from the library's page-locked pool)",
                "gpu_launches": launches_d,
                "pool_blocks_pinned_in_timed_region": fn.batch.pinned_pool.allocs - pool0[0],
                "pool_blocks_reused_in_timed_region": fn.batch.pinned_pool.reuses - pool0[1],
            }
            del xp
        except Exception as exc:  # informational: never lose the headline line
            default_api = {"value": None, "error": str(exc)}
    else:
        xn = rn = un = None
    numa.__exit__(None, None, None)
    e2e_value = e2e_rows * world * e2e_steps / t_e2e if e2e_error is None else None

    if distributed:
        dist.destroy_process_group()
    if rank != 0:
        return 0

    peak, peak_src = _peaks()
    traffic_row, traffic_src = _traffic_per_row()
    rows_rank0 = n
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * t_dev / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded cfg5 generator in HBM; BASELINE.json configs[4])",
        "config": {
            "workload": _workload(rows_total),
            "rows_total": rows_total,
            "rows_per_gpu": rows_rank0,
            "bytes_per_row": BYTES_PER_ROW,
            "l2": "no flush: each step streams 24 GiB/world of input + 32 GiB/world of outputs >> 126 MB L2",
            "parallelism": f"dp{world} contiguous row shards, no data-path collective",
        },
        "achieved_gbs_per_gpu": achieved_gbs,
        "roofline": {
            "bound": "hbm",
            "achieved": achieved_gbs,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved_gbs / peak,
            "traffic": None if traffic_row is None else traffic_row * rows_rank0,
            "peak_source": peak_src,
            # the measured peak is a torch copy kernel, which this kernel can beat; the
            # nominal HBM3e figure bounds both
            "nominal_peak": NOMINAL_HBM_GBS,
            "frac_of_nominal": achieved_gbs / NOMINAL_HBM_GBS,
            "nominal_source": "B200_PROFILING.md: HBM3e 7.7 TB/s (HGX figure; 8 TB/s DGX)",
            "traffic_source": traffic_src,
            "kernel": "tma_stream_kernel<double,3,NORMALIZE> (one launch per step)",
        },
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
        "e2e": {
            "value": e2e_value,
            "unit": UNIT,
            "h2d_bytes_per_step": e2e_rows * world * DIM * 8,
            "d2h_bytes_per_step": e2e_rows * world * (DIM + 1) * 8,
            "rows_per_gpu": e2e_rows,
            "steps": e2e_steps,
            "ms_per_step": 1e3 * t_e2e / e2e_steps,
            "error": e2e_error,
            "api": "paper_1606_06508_b200.normalize3(p, pinned numpy [N,3], out=(r, unit)) -> fn_host_run",
            "gpu_launches": e2e_launches,
            "gpu_launches_source": "fn_launch_count() difference around the timed loop",
            "host_cpus": "NUMA-local to the GPU" if numa.cpus else "all (topology unknown)",
        },
        "e2e_default_api": default_api,
        "sharded_driver": sharded,
        "validation": {
            "row_classes": dict(zip(multigpu.COUNTER_NAMES, counts_h)),
            "rows_counted": int(sum(counts_h)),
            "reduce": f"{args.dist_backend} all_reduce(sum) of 6 counters over {world} rank(s)"
                      if distributed else "single process",
        },
    }
    if world == 1 and not args.no_configs:
        try:
            line["other_configs"] = measure_other_configs(dev, clocks_mhz=(line.get("clocks") or {}).get("sm_mhz"))
        except Exception as exc:  # informational only: never lose the headline line
            line["other_configs"] = {"error": str(exc)}
    if world == 1 and not args.no_cpu_baseline:
        try:
            from paper_1606_06508_b200 import workloads as wl

            xs = wl.host_rows(CFG, 0, CPU_SAMPLE_ROWS)
            rate, threads, kind, best = cpu_reference_rate(xs, ka, reps=12)
            line["cpu_baseline"] = {
                "value": rate, "unit": UNIT, "cores": threads, "kind": kind,
                "sample": (f"cfg5 rows [0, {CPU_SAMPLE_ROWS}): reference loop_scaling3_f64 "
                           f"(checksum only) on {threads} threads, best of 12 passes ({best:.3f} s "
                           f"each; ~{12 * best * threads:.0f} CPU-s in total)"),
            }
        except Exception as exc:  # never lose the headline line
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": None, "kind": None,
                                    "sample": f"failed: {exc}"}
        try:
            line["cpu_detail"] = cpu_detail(ka, fn.kernel_args(fn.preset("single")))
        except Exception as exc:  # informational only
            line["cpu_detail"] = {"error": str(exc)}
    print(json.dumps(line), flush=True)
    return 0


def _rows_arg(text: str) -> int:
    t = text.strip().replace(" ", "")
    if "^" in t:
        b, e = t.split("^")
        v = int(b) ** int(e)
    elif "<<" in t:
        b, e = t.split("<<")
        v = int(b) << int(e)
    else:
        v = int(float(t)) if "e" in t.lower() else int(t)
    if v < 1:
        raise argparse.ArgumentTypeError("--rows must be positive")
    return v


def _self_launch(args) -> int:
    """`bench.py --gpus N` (N > 1) run without torchrun: launch N ranks the way the driver
    does (torch.distributed.run, one process per GPU, 127.0.0.1) and return their exit
    code.  Refuses to share GPUs between NCCL ranks."""
    import socket

    import torch

    ndev = torch.cuda.device_count()
    if args.dist_backend == "nccl" and ndev < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices for NCCL ranks, "
              f"{ndev} visible (use --dist-backend gloo to share devices in a test)", file=sys.stderr)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the informational per-config measurements (configs 1-4)")
    ap.add_argument("--no-default-api", action="store_true",
                    help="skip the e2e_default_api leg (pageable numpy in, library-allocated outputs)")
    ap.add_argument("--rows", type=_rows_arg, default=ROWS_TOTAL,
                    help="total rows over all ranks (default 2^30, BASELINE config 5); e.g. 2^26")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="process-group backend for N > 1 (gloo lets several ranks share one GPU in tests)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _self_launch(args)
    if args.warmup < 3 and args.impl == "ours":
        print("note: --warmup raised to 3 (timing rule)", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
