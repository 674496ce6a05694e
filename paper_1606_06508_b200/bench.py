"""Algorithm-comparison harness on the GPU: per-vector times and the paper's ratio tables.

API mirror of the reference module ``fastnorm.bench`` (pkg/src/fastnorm/bench.py): the
same names (``REGIMES``, ``BenchConfig``, ``BenchConfigError``, ``BenchRow``,
``RatioRow``, ``BenchReport``, ``generate_inputs``, ``run_bench``) and the same two
ratio families:
- "T3" is quotient time over scaling time (bench.py:340-350);
- "T4" is scaling time over naive time.
Both are the quantities of the paper's Table 3 and of BASELINE.md §1.

What a "call" is differs, because the hot path here is batched:
- **Reference.** It times a CPU loop of scalar calls over an L1-resident 1024-row batch
  and subtracts an empty loop.
- **Here.** Each experiment generates ``rows`` vectors of the regime in HBM (a fresh
  seed per experiment). Each algorithm's batched kernel is timed with CUDA events over
  ``reps`` launches. The time per vector is the launch time over ``rows``; there is no
  loop overhead to subtract.
- **Ratios.** They are formed per experiment on shared inputs, as in the reference.

The rows are large enough to stream from HBM (2^24 rows is 256-512 MB per pass against
a 126 MB L2). So the ratios show whether an algorithm is memory-bound (ratio ~1) or
arithmetic-bound on that regime (quotient on wide-range data).
"""

from __future__ import annotations

import csv
import hashlib
import io
import json
import math
import platform
import statistics
from dataclasses import asdict, dataclass, field

import numpy as np

from paper_1606_06508_b200 import _backend, _lib, workloads
from paper_1606_06508_b200.params import preset
from paper_1606_06508_b200.scale import kernel_args_array

__all__ = ["REGIMES", "BenchConfig", "BenchConfigError", "BenchRow", "RatioRow", "BenchReport",
           "generate_inputs", "generate_regime_rows", "run_bench"]

REGIMES = workloads.REGIMES
_PREC_DTYPE = {"double": "float64", "single": "float32"}
_PREC_ID = {"double": 0, "single": 1}


class BenchConfigError(ValueError):
    """An unrunnable benchmark configuration."""


@dataclass(frozen=True)
class BenchConfig:
    """Workload of :func:`run_bench`.  ``rows`` vectors per experiment (in HBM), timed
    over ``reps`` launches per algorithm."""

    experiments: int = 10
    rows: int = 1 << 24
    reps: int = 5
    dimensions: tuple[int, ...] = (2, 3, 4)
    precisions: tuple[str, ...] = ("double",)
    algorithms: tuple[str, ...] = _backend.ALGORITHMS
    seed: int = 0
    regime: str = "normal"
    backend: str | None = None


@dataclass
class BenchRow:
    task: str
    precision: str
    algorithm: str
    backend: str
    mean_ns_per_vector: float
    std_ns_per_vector: float
    vectors_per_s: float
    checksum: float


@dataclass
class RatioRow:
    label: str          # "T3" quotient/scaling, "T4" scaling/naive
    task: str
    precision: str
    backend: str
    numerator: str
    denominator: str
    mean: float
    std: float
    experiments: int


@dataclass
class BenchReport:
    config: BenchConfig
    rows: list[BenchRow]
    ratios: list[RatioRow]
    environment: dict = field(default_factory=dict)

    def to_json(self) -> str:
        body = {"config": asdict(self.config), "rows": [asdict(r) for r in self.rows],
                "ratios": [asdict(r) for r in self.ratios], "environment": self.environment}
        return json.dumps(body, sort_keys=True, indent=2)

    def to_csv(self) -> str:
        buf = io.StringIO()
        out = csv.writer(buf)
        out.writerow(["kind", "label", "task", "precision", "backend", "algorithm_or_pair",
                      "mean", "std", "vectors_per_s", "checksum"])
        for r in self.rows:
            out.writerow(["time", "", r.task, r.precision, r.backend, r.algorithm,
                          f"{r.mean_ns_per_vector:.6g}", f"{r.std_ns_per_vector:.6g}",
                          f"{r.vectors_per_s:.6g}", repr(r.checksum)])
        for r in self.ratios:
            out.writerow(["ratio", r.label, r.task, r.precision, r.backend,
                          f"{r.numerator}/{r.denominator}", f"{r.mean:.6g}", f"{r.std:.6g}", "", ""])
        return buf.getvalue()


# Binade exponents per format: least subnormal, least normal, largest (bench.py:49).
_BINADES = {"double": (-1074, -1022, 1023), "single": (-149, -126, 127)}


def generate_inputs(regime: str, dimension: int, precision: str, count: int, seed) -> np.ndarray:
    """The reference's deterministic ``(count, dimension)`` host batch of nonzero finite
    vectors, bit for bit (bench.py:146-207): the same PCG64 stream seeded through
    ``SeedSequence(seed)`` (``seed``: an int or a tuple of ints), drawn in the same order
    (signs, mantissas, then the regime's exponents or normals).

    ``normal``: magnitudes in [tau_min, tau_max]; ``subnormal``: in [alpha, nu);
    ``huge``: above tau_max; ``mixed``: exponents uniform over the whole range,
    subnormals included; ``unit-ish``: norms within 2^-10 of one.

    The GPU ratio harness (:func:`run_bench`) draws its HBM-sized batches with the
    counter generator instead (:func:`generate_regime_rows`), which any shard or device
    reproduces without drawing the rows before it."""
    if regime not in REGIMES:
        raise ValueError(f"unknown regime {regime!r}; choices: {REGIMES}")
    if dimension not in (2, 3, 4):
        raise ValueError(f"dimension must be 2, 3 or 4, got {dimension}")
    if precision not in _PREC_DTYPE:
        raise ValueError(f"unknown precision {precision!r}")
    if count <= 0:
        raise ValueError("count must be positive")
    gen = np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed)))
    fmt = preset(precision)
    dtype = np.dtype(_PREC_DTYPE[precision])
    least_sub, least_normal, top = _BINADES[precision]
    lo_band, hi_band = int(math.log2(fmt.tau_min)), int(math.log2(fmt.tau_max))
    shape = (count, dimension)
    signs = 2.0 * gen.integers(0, 2, size=shape).astype(np.float64) - 1.0
    mantissas = gen.random(shape) + 1.0
    if regime == "unit-ish":
        g = gen.standard_normal(shape)
        lengths = np.sqrt(np.sum(g * g, axis=1, keepdims=True))
        g[:, 0] = np.where(lengths[:, 0] == 0.0, 1.0, g[:, 0])
        lengths = np.maximum(lengths, np.finfo(np.float64).tiny)
        stretch = 1.0 + (2.0 * gen.random((count, 1)) - 1.0) * 2.0 ** -10
        return np.ascontiguousarray(((g / lengths) * stretch).astype(dtype))
    exp_range = {"normal": (lo_band, hi_band), "subnormal": (least_sub, least_normal),
                 "huge": (hi_band + 1, top - 1), "mixed": (least_sub, top)}[regime]
    mags = np.ldexp(mantissas, gen.integers(*exp_range, size=shape))
    if regime == "subnormal":  # rounding can lift the top of the range onto nu
        mags = np.minimum(mags, fmt.nu - fmt.alpha)
    vals = (mags * signs).astype(dtype)
    if regime == "subnormal" and precision == "single":
        cap = np.float32(fmt.nu - fmt.alpha)
        np.clip(vals, -cap, cap, out=vals)
    return np.ascontiguousarray(vals)


def generate_regime_rows(regime: str, dimension: int, precision: str, count: int, seed=0) -> np.ndarray:
    """Rows of a reference regime from the counter generator the device uses
    (workloads.regime_rows): the same seed gives the same rows on the host and in HBM,
    and any row range can be drawn alone.  Not the reference's stream -- that is
    :func:`generate_inputs`."""
    if regime not in REGIMES:
        raise ValueError(f"unknown regime {regime!r}; choices: {REGIMES}")
    if dimension not in (2, 3, 4):
        raise ValueError(f"dimension must be 2, 3 or 4, got {dimension}")
    if precision not in _PREC_DTYPE:
        raise ValueError(f"unknown precision {precision!r}")
    if count <= 0:
        raise ValueError("count must be positive")
    return workloads.regime_rows(regime, dimension, _PREC_DTYPE[precision], 0, count, seed=_seed_int(seed))


def _seed_int(seed) -> int:
    """Fold an int or a tuple of ints into one 64-bit generator seed."""
    if isinstance(seed, (tuple, list)):
        h = hashlib.sha256(",".join(str(int(s)) for s in seed).encode()).digest()
        return int.from_bytes(h[:8], "little")
    return int(seed) & 0xFFFFFFFFFFFFFFFF


def _validate(c: BenchConfig) -> None:
    problems = []
    if c.experiments <= 0 or c.rows <= 0 or c.reps <= 0:
        problems.append("experiments, rows and reps must be positive")
    if not (c.dimensions and c.precisions and c.algorithms):
        problems.append("at least one dimension, precision and algorithm is required")
    problems += [f"unsupported dimension {d}" for d in c.dimensions if d not in (2, 3, 4)]
    problems += [f"unsupported precision {p!r}" for p in c.precisions if p not in _PREC_DTYPE]
    problems += [f"unsupported algorithm {a!r}" for a in c.algorithms if a not in _backend.ALGORITHMS]
    if c.regime not in REGIMES:
        problems.append(f"unsupported regime {c.regime!r}")
    if problems:
        raise BenchConfigError("; ".join(problems))


def _time_per_vector(fn, reps: int, n: int) -> float:
    import torch

    fn()  # warm-up (first-launch setup, module load)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e6 / reps / n  # ns per vector


def run_bench(config: BenchConfig) -> BenchReport:
    """Run the protocol on the current CUDA device; rows, T3 and T4 ratios."""
    import torch

    _validate(config)
    backend = config.backend or _backend.backend_name()
    _backend.get_module(backend)
    n = config.rows
    per: dict[tuple[str, str, str], list[float]] = {}
    sums: dict[tuple[str, str, str], float] = {}
    rows: list[BenchRow] = []
    for prec in config.precisions:
        ka = kernel_args_array(preset(prec))
        dt = torch.float64 if prec == "double" else torch.float32
        for dim in config.dimensions:
            task = f"normalize{dim}d"
            algos = [a for a in config.algorithms if dim in _backend.algorithm_dims(a)]
            if not algos:
                continue
            x = torch.empty((n, dim), dtype=dt, device="cuda")
            kernels = {a: _backend.batch_kernel(_backend.scalar_base(a, dim), prec, backend) for a in algos}
            outs = {a: None for a in algos}
            for exp in range(config.experiments):
                workloads.generate_regime_device(config.regime, x,
                                                 seed=_seed_int((config.seed, _PREC_ID[prec], dim, exp)))
                for a in algos:
                    k = kernels[a]
                    args = ka if _backend.takes_params(a) else None

                    def launch(k=k, args=args, a=a):
                        outs[a] = k(x, args, out=outs[a] and (outs[a].head, outs[a].body))

                    per.setdefault((task, prec, a), []).append(_time_per_vector(launch, config.reps, n))
                    res = outs[a]
                    sums[(task, prec, a)] = sums.get((task, prec, a), 0.0) + float(
                        torch.nan_to_num(res.head.double(), nan=0.0, posinf=0.0).sum().item())
            del x, outs
            for a in algos:
                v = per[(task, prec, a)]
                mean = statistics.fmean(v)
                rows.append(BenchRow(task, prec, a, backend, mean,
                                     statistics.stdev(v) if len(v) > 1 else 0.0, 1e9 / mean,
                                     sums[(task, prec, a)]))
    if not rows:
        raise BenchConfigError("no runnable (algorithm, dimension) combination in the configuration")

    ratios: list[RatioRow] = []

    def ratio(label, task, prec, num, den):
        a, b = per.get((task, prec, num)), per.get((task, prec, den))
        if not a or not b:
            return
        vals = [p / q for p, q in zip(a, b) if q > 0]
        ratios.append(RatioRow(label, task, prec, backend, num, den, statistics.fmean(vals),
                               statistics.stdev(vals) if len(vals) > 1 else 0.0, len(vals)))

    for prec in config.precisions:
        for dim in config.dimensions:
            task = f"normalize{dim}d"
            ratio("T3", task, prec, "quotient", "scaling")
            ratio("T3", task, prec, "quotient_fast", "scaling")
            ratio("T4", task, prec, "scaling", "naive")

    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    env = {"timer": "cuda events on the launching stream", "device": props.name,
           "sm_count": props.multi_processor_count, "library": _lib.version(),
           "build_flags": _lib.build_flags(), "python": platform.python_version(),
           "torch": torch.__version__, "numpy": np.__version__}
    return BenchReport(config=config, rows=rows, ratios=ratios, environment=env)
