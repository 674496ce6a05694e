"""Command line front-end (reference: pkg/src/fastnorm/cli.py), batched and on the GPU.

    python -m paper_1606_06508_b200 normalize --dim 3 [--prec double] [--algo scaling] X1 X2 X3
    python -m paper_1606_06508_b200 rotate [--method general|unit] [--apply V1 V2 V3] Q1 Q2 Q3 Q4
    python -m paper_1606_06508_b200 validate-params [--format single|double] [--file params.json]
    python -m paper_1606_06508_b200 verify-bounds --dim N [--prec] [--samples] [--regime] [--seed]
    python -m paper_1606_06508_b200 batch --dim N --in rows.npy --out result.npz [--prec] [--algo]
    python -m paper_1606_06508_b200 bench [--config 1..5] [--algo] [--steps] [--warmup]
    python -m paper_1606_06508_b200 selftest [--pairs N]

The subcommands and their options follow the reference's click CLI (normalize :55-75,
validate-params :78-114, verify-bounds :117-177, bench :180-237, rotate :240-259).
`verify-bounds` runs the double-double bound sweep on the GPU over `--samples` rows
(default 2^20 instead of the reference's 10^4 scalar oracle calls); `bench` times the
batched kernels on a BASELINE config in HBM (the reference's ns/call loop protocol has
no GPU meaning); `batch` normalizes an .npy file of rows through the host path.
Numbers can be given as decimals, hex floats (0x1.8p-3), inf/nan or 2^k.
"""

from __future__ import annotations

import argparse
import json
import math
import sys

ALGOS = ("scaling", "quotient", "quotient_fast", "naive")


def parse_number(text: str) -> float:
    """Decimal, hex float (0x1.8p+3), inf/nan, or a power of two written 2^k."""
    t = text.strip().lower()
    if t.startswith(("2^", "+2^")):
        return math.ldexp(1.0, int(t.split("^", 1)[1]))
    if t.startswith("-2^"):
        return -math.ldexp(1.0, int(t.split("^", 1)[1]))
    if "0x" in t:
        return float.fromhex(t)
    return float(t)


def _fmt(v: float, hex_out: bool, single: bool = False) -> float | str:
    if not hex_out:
        return v
    return float(v).hex()


def _normalize_call(algo: str, dim: int, prec: str, comps):
    import paper_1606_06508_b200 as fn

    p = fn.preset(prec)
    if algo == "scaling":
        return getattr(fn, f"normalize{dim}")(p, *comps)
    if algo == "naive":
        return getattr(fn, f"naive_normalize{dim}")(*comps, precision=prec)
    if algo == "quotient_fast":
        if dim != 3:
            raise SystemExit("quotient_fast is defined for --dim 3 only")
        return fn.quotient3_fast(*comps, precision=prec)
    return {2: fn.quotient2, 3: fn.quotient3_robust, 4: fn.quotient4}[dim](*comps, precision=prec)


def cmd_normalize(a) -> int:
    comps = [parse_number(c) for c in a.components]
    if len(comps) != a.dim:
        raise SystemExit(f"--dim {a.dim} needs {a.dim} components, got {len(comps)}")
    out = _normalize_call(a.algo, a.dim, a.prec, comps)
    print(json.dumps({"algo": a.algo, "precision": a.prec, "input": comps,
                      "length": _fmt(out.length, a.hex),
                      "unit": [_fmt(v, a.hex) for v in out.unit]}))
    return 0


def cmd_rotate(a) -> int:
    import paper_1606_06508_b200 as fn

    q = [parse_number(c) for c in a.components]
    try:
        m = fn.rotation_general(q) if a.method == "general" else fn.rotation_unit(q)
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    res = {"method": a.method, "quaternion": q,
           "rows": [[_fmt(v, a.hex) for v in row] for row in m.rows]}
    if a.apply:
        res["applied"] = [_fmt(v, a.hex) for v in m.apply(tuple(parse_number(v) for v in a.apply))]
    print(json.dumps(res))
    return 0


def cmd_validate_params(a) -> int:
    from paper_1606_06508_b200.params import FpParams, preset, validate_conditions

    if a.path:
        with open(a.path) as f:
            raw = json.load(f)
        p = FpParams(**{k: float(parse_number(str(v))) for k, v in raw.items()})
        label = a.path
    else:
        p = preset(a.fmt or "double")
        label = a.fmt or "double"
    violations = validate_conditions(p)
    out = {"params": label, "valid": not violations,
           "violations": [{"check": v.check, "detail": v.detail} for v in violations]}
    if a.show_derived and not a.path:
        from paper_1606_06508_b200.params import derive_tau

        lo, hi = derive_tau(a.fmt or "double")
        out["derived_tau"] = {"tau_min": lo, "tau_max": hi}
    print(json.dumps(out))
    return 0 if not violations else 1


def cmd_verify_bounds(a) -> int:
    import torch

    import paper_1606_06508_b200 as fn
    from paper_1606_06508_b200 import workloads
    from paper_1606_06508_b200.bounds import sweep_bounds

    regimes = workloads.REGIMES if a.regime == "all" else (a.regime,)
    dt = torch.float64 if a.prec == "double" else torch.float32
    results = []
    rc = 0
    for reg in regimes:
        x = torch.empty((a.samples, a.dim), dtype=dt, device="cuda")
        workloads.generate_regime_device(reg, x, seed=a.seed)
        s = sweep_bounds(fn.preset(a.prec), x)
        results.append({"regime": reg, "samples": s.samples, "violations": s.violation_count,
                        "violation_ids": s.violation_ids, "max_metrics_u": s.max_metrics,
                        "bounds_u": s.bounds_u, "first_violation_row": s.first_violation_row})
        rc |= int(s.violation_count > 0)
    print(json.dumps({"dim": a.dim, "precision": a.prec, "algo": "scaling", "results": results}))
    return rc


def cmd_batch(a) -> int:
    import numpy as np

    x = np.load(a.inp)
    want = np.float64 if a.prec == "double" else np.float32
    if x.dtype != want:
        x = x.astype(want)
    if x.ndim != 2 or x.shape[1] != a.dim:
        raise SystemExit(f"expected an [N, {a.dim}] array, got {x.shape}")
    out = _normalize_call(a.algo, a.dim, a.prec, [x])
    np.savez(a.out, length=out.length, unit=out.unit)
    print(json.dumps({"rows": int(x.shape[0]), "out": a.out, "algo": a.algo, "precision": a.prec}))
    return 0


def cmd_bench(a) -> int:
    import torch

    import paper_1606_06508_b200 as fn
    from paper_1606_06508_b200 import workloads

    c = workloads.CONFIGS[a.config]
    n = a.rows or c.rows
    dt = torch.float64 if c.dtype == "float64" else torch.float32
    prec = "double" if dt == torch.float64 else "single"
    if a.devices:
        return _bench_sharded(a, c, n, prec)
    x = torch.empty((n, c.dim), dtype=dt, device="cuda")
    workloads.generate_device(a.config, x)
    w = x.element_size()
    bytes_row = {"scaling": (2 * c.dim + 1) * w, "quotient": (2 * c.dim + 1) * w,
                 "quotient_fast": (2 * c.dim + 1) * w, "naive": (2 * c.dim + 1) * w}[a.algo]
    run = (lambda: _normalize_call(a.algo, c.dim, prec, [x]))
    for _ in range(a.warmup):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        run()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / a.steps
    print(json.dumps({"config": a.config, "algo": a.algo, "rows": n, "dim": c.dim, "dtype": c.dtype,
                      "ms_per_pass": t * 1e3, "vectors_per_s": n / t,
                      "GB_per_s": n * bytes_row / t / 1e9}))
    return 0


def _bench_sharded(a, c, n: int, prec: str) -> int:
    """`bench --devices 0,1,...`: the config's rows as device-resident shards on several GPUs
    of this one process (multigpu.DeviceShards, fn_run_sharded: one stream per shard, no
    collective).  A pass takes as long as its slowest shard (CUDA events per shard)."""
    import statistics

    import paper_1606_06508_b200 as fn
    from paper_1606_06508_b200 import multigpu

    if a.algo != "scaling":
        print("error: --devices runs the scaling algorithm", file=sys.stderr)
        return 2
    devs = [int(d) for d in a.devices.split(",")]
    p = fn.preset(prec)
    x = multigpu.DeviceShards.generate(a.config, n, devs)
    out = None
    for _ in range(max(a.warmup, 1)):
        res = multigpu.normalize_sharded(p, x, out=out)
        out = (res.head, res.body)
    ms = [max(multigpu.normalize_sharded(p, x, out=out).elapsed_ms) for _ in range(a.steps)]
    t = statistics.median(ms) / 1e3
    w = x[0].element_size()
    print(json.dumps({"config": a.config, "algo": a.algo, "rows": n, "dim": c.dim, "dtype": c.dtype,
                      "devices": devs, "rows_per_shard": [int(s.shape[0]) for s in x.tensors],
                      "ms_per_pass": t * 1e3, "vectors_per_s": n / t,
                      "GB_per_s": n * (2 * c.dim + 1) * w / t / 1e9}))
    return 0


def cmd_ratios(a) -> int:
    from paper_1606_06508_b200 import bench

    cfg = bench.BenchConfig(experiments=a.experiments, rows=a.rows, reps=a.reps,
                            dimensions=tuple(a.dims or (2, 3, 4)), precisions=tuple(a.precs or ("double",)),
                            algorithms=tuple(a.algos or ALGOS), seed=a.seed, regime=a.regime)
    try:
        rep = bench.run_bench(cfg)
    except bench.BenchConfigError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    env = rep.environment
    print(f"# {env['device']} ({env['sm_count']} SMs), {env['library']}; timer: {env['timer']}")
    print(f"# regime {cfg.regime}, {cfg.rows} vectors x {cfg.experiments} experiments x {cfg.reps} launches")
    print(f"{'task':<14}{'prec':<8}{'algorithm':<16}{'ns/vector':>12}{'std':>10}{'Gvec/s':>10}")
    for r in rep.rows:
        print(f"{r.task:<14}{r.precision:<8}{r.algorithm:<16}{r.mean_ns_per_vector:>12.5f}"
              f"{r.std_ns_per_vector:>10.5f}{r.vectors_per_s / 1e9:>10.2f}")
    print(f"{'label':<7}{'task':<14}{'prec':<8}{'ratio':<28}{'mean':>8}{'std':>8}")
    for r in rep.ratios:
        print(f"{r.label:<7}{r.task:<14}{r.precision:<8}{r.numerator + '/' + r.denominator:<28}"
              f"{r.mean:>8.2f}{r.std:>8.2f}")
    if a.csv_path:
        with open(a.csv_path, "w", encoding="utf-8") as fh:
            fh.write(rep.to_csv())
    if a.json_path:
        with open(a.json_path, "w", encoding="utf-8") as fh:
            fh.write(rep.to_json())
    return 0


def cmd_selftest(a) -> int:
    import torch

    from paper_1606_06508_b200 import _lib

    out = torch.zeros(3, dtype=torch.int64, device="cuda")
    res = {}
    for name, dt in (("f64", _lib.F64), ("f32", _lib.F32)):
        out.zero_()
        _lib.check(_lib.lib().fn_selftest_div(dt, 1, a.pairs, out.data_ptr(),
                                              torch.cuda.current_stream().cuda_stream), "selftest")
        res[name] = int(out[0].item())
    print(json.dumps({"division_pairs": a.pairs, "mismatches": res, "version": _lib.version()}))
    return 0 if not any(res.values()) else 1


def _same_bits(a, b):
    """The reference's comparison rule (tests/test_backends.py:33-38): NaN matches NaN,
    everything else must be bit-equal, zero signs included."""
    import numpy as np

    a, b = np.asarray(a), np.asarray(b)
    both_nan = np.isnan(a) & np.isnan(b)
    return both_nan | (a.view(np.uint8).reshape(a.shape + (-1,)) ==
                       b.view(np.uint8).reshape(b.shape + (-1,))).all(axis=-1)


def cmd_compare(a) -> int:
    """Compare two result files (.npz of named arrays, e.g. this build's `batch` output
    against one produced by the reference) array by array and row by row; print the
    mismatch count per array and the first mismatching rows in hex floats."""
    import numpy as np

    fa, fb = np.load(a.a), np.load(a.b)
    names = [k for k in fa.files if k in fb.files] if not a.arrays else a.arrays
    if not names:
        raise SystemExit("no array names in common")
    report, worst = {}, 0
    single = None
    for k in names:
        x, y = fa[k], fb[k]
        if x.shape != y.shape or x.dtype != y.dtype:
            raise SystemExit(f"{k}: {x.shape} {x.dtype} vs {y.shape} {y.dtype}")
        single = x.dtype == np.float32
        ok = _same_bits(x, y)
        rows_ok = ok.reshape(ok.shape[0], -1).all(axis=1) if ok.ndim > 1 else ok
        bad = np.flatnonzero(~rows_ok)
        worst = max(worst, len(bad))
        report[k] = {"rows": int(rows_ok.shape[0]), "mismatching_rows": int(len(bad)),
                     "first": [{"row": int(i),
                                "a": [_fmt(float(v), True, single) for v in np.ravel(x[i])],
                                "b": [_fmt(float(v), True, single) for v in np.ravel(y[i])]}
                               for i in bad[: a.show]]}
    print(json.dumps(report))
    return 0 if worst == 0 else 1


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_1606_06508_b200", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="cmd", required=True)

    s = sub.add_parser("normalize", help="normalize one vector (GPU)")
    s.add_argument("--dim", type=int, choices=(2, 3, 4), required=True)
    s.add_argument("--prec", choices=("single", "double"), default="double")
    s.add_argument("--algo", choices=ALGOS, default="scaling")
    s.add_argument("--hex", action="store_true", help="print results as hex floats")
    s.add_argument("components", nargs="+")
    s.set_defaults(fn=cmd_normalize)

    s = sub.add_parser("rotate", help="rotation matrix of one quaternion (GPU)")
    s.add_argument("--method", choices=("general", "unit"), default="general")
    s.add_argument("--apply", nargs=3, default=None, metavar=("V1", "V2", "V3"))
    s.add_argument("--hex", action="store_true")
    s.add_argument("components", nargs=4)
    s.set_defaults(fn=cmd_rotate)

    s = sub.add_parser("validate-params", help="check a parameter set's conditions")
    s.add_argument("--format", dest="fmt", choices=("single", "double"), default=None)
    s.add_argument("--file", dest="path", default=None, help="JSON object of the 8 FpParams fields")
    s.add_argument("--show-derived", action="store_true")
    s.set_defaults(fn=cmd_validate_params)

    s = sub.add_parser("verify-bounds", help="GPU error-bound sweep of the scaling algorithm")
    s.add_argument("--dim", type=int, choices=(2, 3, 4), required=True)
    s.add_argument("--prec", choices=("single", "double"), default="double")
    s.add_argument("--samples", type=int, default=1 << 20)
    s.add_argument("--regime", choices=("all", "normal", "subnormal", "huge", "mixed", "unit-ish"),
                   default="mixed")
    s.add_argument("--seed", type=int, default=0)
    s.set_defaults(fn=cmd_verify_bounds)

    s = sub.add_parser("batch", help="normalize an .npy file of [N, dim] rows")
    s.add_argument("--dim", type=int, choices=(2, 3, 4), required=True)
    s.add_argument("--prec", choices=("single", "double"), default="double")
    s.add_argument("--algo", choices=ALGOS, default="scaling")
    s.add_argument("--in", dest="inp", required=True)
    s.add_argument("--out", required=True)
    s.set_defaults(fn=cmd_batch)

    s = sub.add_parser("compare", help="bit-compare two result .npz files (NaN == NaN); "
                                       "report mismatching rows in hex floats")
    s.add_argument("a")
    s.add_argument("b")
    s.add_argument("--array", dest="arrays", action="append", help="array name (default: all shared)")
    s.add_argument("--show", type=int, default=5, help="mismatching rows to print per array")
    s.set_defaults(fn=cmd_compare)

    s = sub.add_parser("bench", help="time a kernel family on a BASELINE config in HBM")
    s.add_argument("--config", type=int, choices=(1, 2, 3, 4, 5), default=1)
    s.add_argument("--algo", choices=ALGOS, default="scaling")
    s.add_argument("--rows", type=int, default=0, help="override the config's row count")
    s.add_argument("--steps", type=int, default=20)
    s.add_argument("--warmup", type=int, default=3)
    s.add_argument("--devices", default="", help="comma-separated GPU ordinals: shard the rows over these "
                                                 "devices from this one process (a device may repeat)")
    s.set_defaults(fn=cmd_bench)

    s = sub.add_parser("ratios", help="per-vector times and the T3/T4 ratio tables on the GPU "
                                      "(the reference's `bench` protocol, batched)")
    s.add_argument("--experiments", type=int, default=10)
    s.add_argument("--rows", type=int, default=1 << 24, help="vectors per experiment (in HBM)")
    s.add_argument("--reps", type=int, default=5, help="timed launches per algorithm and experiment")
    s.add_argument("--dim", dest="dims", type=int, choices=(2, 3, 4), action="append")
    s.add_argument("--prec", dest="precs", choices=("single", "double"), action="append")
    s.add_argument("--algo", dest="algos", choices=ALGOS, action="append")
    s.add_argument("--regime", choices=("normal", "subnormal", "huge", "mixed", "unit-ish"), default="normal")
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--csv", dest="csv_path", default=None)
    s.add_argument("--json", dest="json_path", default=None)
    s.set_defaults(fn=cmd_ratios)

    s = sub.add_parser("selftest", help="device self-test of the exact division paths")
    s.add_argument("--pairs", type=int, default=1 << 24)
    s.set_defaults(fn=cmd_selftest)
    return ap


def main(argv=None) -> int:
    a = build_parser().parse_args(argv)
    return a.fn(a)


if __name__ == "__main__":
    sys.exit(main())
