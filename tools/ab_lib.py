"""A/B timing of two builds of libfastnorm_b200.so on a config workload (dev tool).

python tools/ab_lib.py OLD.so NEW.so [--op 1] [--dim 3] [--cfg 5] [--log2-rows 30]
Both libraries run fn_run(op, dim, FN_F64) over the same config rows, alternating
process by process (each .so carries its own static cudart, so one library per
process), timed with CUDA events on one stream.  Defaults: the bench workload
(normalize3 over 2^30 config-5 rows)."""
import argparse
import ctypes
import statistics
import subprocess
import sys

sys.path.insert(0, ".")


def parse(argv):
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--op", type=int, default=1)
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--cfg", type=int, default=5)
    ap.add_argument("--regime", default=None, help="reference regime instead of a config")
    ap.add_argument("--f32", action="store_true")
    ap.add_argument("--log2-rows", type=int, default=30)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=3)
    return ap.parse_args(argv)


def run_one(a):
    import numpy as np
    import torch

    from paper_1606_06508_b200 import batch, workloads

    L = ctypes.CDLL(a.libs[0].split("@")[0])
    L.fn_run.restype = ctypes.c_int
    L.fn_run.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 5
    n = 1 << a.log2_rows
    dt = torch.float32 if a.f32 else torch.float64
    x = torch.empty((n, a.dim), dtype=dt, device="cuda")
    if a.regime:
        workloads.generate_regime_device(a.regime, x)
    else:
        workloads.generate_device(a.cfg, x)
    w0, w1, w2 = batch.widths(a.op, a.dim)
    outs = [torch.empty((n, w), dtype=dt, device="cuda") if w else None for w in (w0, w1, w2)]
    ptr = [o.data_ptr() if o is not None else None for o in outs]
    ka = (np.array([2.0 ** -49, 2.0 ** 62, 2.0 ** 100, 2.0 ** -66, 2.0 ** -100, 2.0 ** 66]) if a.f32 else
          np.array([2.0 ** -482, 2.0 ** 510, 2.0 ** 592, 2.0 ** -514, 2.0 ** -592, 2.0 ** 514]))
    s = torch.cuda.current_stream().cuda_stream
    bytes_per_row = x.element_size() * (a.dim + w0 + w1 + w2)

    def launch():
        rc = L.fn_run(a.op, a.dim, 0 if a.f32 else 1, x.data_ptr(), n, ptr[0], ptr[1], ptr[2], ka.ctypes.data, s)
        assert rc == 0, rc

    times = []
    for _ in range(a.rounds):
        for _ in range(3):
            launch()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            launch()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / a.reps)
    ms = statistics.median(times)
    src = f"regime={a.regime}" if a.regime else f"cfg={a.cfg}"
    print(f"{a.libs[0]}: op={a.op} dim={a.dim} {src} {'f32' if a.f32 else 'f64'} {ms:.4f} ms/launch, "
          f"{n * bytes_per_row / ms / 1e6:.1f} GB/s, all={['%.3f' % v for v in times]}", flush=True)


def main():
    a = parse(sys.argv[1:])
    if len(a.libs) > 1:
        rest = [f"--op={a.op}", f"--dim={a.dim}", f"--cfg={a.cfg}", f"--log2-rows={a.log2_rows}",
                f"--reps={a.reps}", f"--rounds={a.rounds}"] + (["--f32"] if a.f32 else []) + \
            ([f"--regime={a.regime}"] if a.regime else [])
        import os

        for _ in range(3):
            for spec in a.libs:
                # "lib.so@VAR=VAL,VAR2=VAL2": the same library under other settings
                path, _, envs = spec.partition("@")
                env = dict(os.environ)
                env.update(dict(kv.split("=", 1) for kv in envs.split(",") if kv))
                subprocess.run([sys.executable, __file__, spec] + rest, check=True, env=env)
        return
    run_one(a)


if __name__ == "__main__":
    main()
