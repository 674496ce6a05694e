"""Developer probe (GPU): why back-to-back 2^30-row launches of the headline kernel run
slower than an isolated launch (bench 9.35 ms vs ncu 8.91 ms on the same box).

For normalize3 f64 over config-5 rows it times, with per-launch CUDA events on the
launching stream and NVML sampling (SM / memory clock, power, throttle reasons):
  b2b    -- 20 launches back to back (the bench's timed loop);
  gap    -- 20 launches with a 20 ms GPU sleep between them;
  sub    -- 2^30 rows as 4 launches of 2^28 rows back to back (address ranges);
  small  -- 2^28-row buffers, 20 launches back to back.
One process per FASTNORM_B200_PDL setting.  Usage: python tools/probe/steady_state.py"""

import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


class Nvml:
    def __init__(self):
        import pynvml

        pynvml.nvmlInit()
        self.p = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(0)
        self.samples = []
        self._stop = threading.Event()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        p, h = self.p, self.h
        while not self._stop.is_set():
            try:
                self.samples.append((p.nvmlDeviceGetClockInfo(h, p.NVML_CLOCK_SM),
                                     p.nvmlDeviceGetClockInfo(h, p.NVML_CLOCK_MEM),
                                     p.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                     p.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass
            self._stop.wait(0.005)

    def __exit__(self, *a):
        self._stop.set()
        self._t.join()

    def summary(self):
        if not self.samples:
            return {}
        sm = [s[0] for s in self.samples]
        mem = [s[1] for s in self.samples]
        pw = [s[2] for s in self.samples]
        capped = sum(1 for s in self.samples if s[3] & 0x4)
        return {"sm_med": statistics.median(sm), "sm_min": min(sm), "mem_med": statistics.median(mem),
                "power_med": statistics.median(pw), "power_max": max(pw), "n": len(sm),
                "power_cap_frac": capped / len(sm)}


def child():
    sys.path.insert(0, REPO)
    import torch

    import paper_1606_06508_b200 as fn
    from paper_1606_06508_b200 import workloads

    p = fn.preset("double")
    dev = torch.device("cuda:0")
    s = torch.cuda.current_stream()
    out = {"pdl": os.environ.get("FASTNORM_B200_PDL", "default"), "dyn": os.environ.get("FASTNORM_B200_DYN", "default")}

    def timed(launches, gap_ms=0.0):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(launches) + 1)]
        with Nvml() as nv:
            torch.cuda.synchronize()
            for i, f in enumerate(launches):
                if gap_ms:
                    torch.cuda._sleep(int(gap_ms * 1.9e6))
                ev[i].record(s)
                f()
                if gap_ms or i == len(launches) - 1:
                    ev[i + 1].record(s)
            torch.cuda.synchronize()
        if gap_ms:
            ts = [ev[i].elapsed_time(ev[i + 1]) for i in range(len(launches))]
        else:
            ts = [ev[i].elapsed_time(ev[i + 1]) for i in range(len(launches) - 1)]
            ts.append(ev[0].elapsed_time(ev[-1]) - sum(ts))
        return ts, nv.summary()

    n = 1 << 30
    x = torch.empty((n, 3), dtype=torch.float64, device=dev)
    workloads.generate_device(5, x)
    r = torch.empty(n, dtype=torch.float64, device=dev)
    u = torch.empty_like(x)
    for _ in range(3):
        fn.normalize3(p, x, out=(r, u))
    torch.cuda.synchronize()
    f = lambda: fn.normalize3(p, x, out=(r, u))  # noqa: E731
    for mode, launches, gap in (("b2b", [f] * 20, 0.0), ("gap", [f] * 20, 20.0), ("b2b_again", [f] * 20, 0.0)):
        ts, nv = timed(launches, gap)
        out[mode] = {"ms_each": [round(t, 3) for t in ts], "ms_mean": statistics.fmean(ts),
                     "GBs_mean": n * 56 / (statistics.fmean(ts) * 1e-3) / 1e9, "nvml": nv}
    q = n // 4
    subs = [(lambda a=a: fn.normalize3(p, x[a:a + q], out=(r[a:a + q], u[a:a + q]))) for a in range(0, n, q)]
    ts, nv = timed(subs * 5, 0.0)
    out["sub4"] = {"ms_each": [round(t, 3) for t in ts], "GBs_mean": q * 56 / (statistics.fmean(ts) * 1e-3) / 1e9,
                   "nvml": nv}
    del x, r, u
    torch.cuda.empty_cache()
    x = torch.empty((q, 3), dtype=torch.float64, device=dev)
    workloads.generate_device(5, x)
    r = torch.empty(q, dtype=torch.float64, device=dev)
    u = torch.empty_like(x)
    g = lambda: fn.normalize3(p, x, out=(r, u))  # noqa: E731
    for _ in range(3):
        g()
    ts, nv = timed([g] * 40, 0.0)
    out["small_b2b"] = {"ms_each": [round(t, 3) for t in ts], "GBs_mean": q * 56 / (statistics.fmean(ts) * 1e-3) / 1e9,
                        "nvml": nv}
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child()
        sys.exit(0)
    for env in ({}, {"FASTNORM_B200_PDL": "0"}, {"FASTNORM_B200_DYN": "0"}):
        e = dict(os.environ, **env)
        p = subprocess.run([sys.executable, os.path.abspath(__file__), "child"], env=e, capture_output=True, text=True)
        print(p.stdout.strip() or p.stderr[-2000:], flush=True)
