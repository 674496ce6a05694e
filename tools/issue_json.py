"""Turn tools/ncu_issue.sh CSVs into profiles/ncu_issue.json (developer tool).

Per kernel: warp instructions, issue-active cycles and FP64-pipe instructions per row,
the SM clock ncu saw, and DRAM bytes per row.  bench.py reads the per-row instruction
counts to put an instruction-issue roofline beside the HBM one for the division-bound
comparison kernels.
python tools/issue_json.py TAG [--merge]"""
import csv
import glob
import json
import os
import sys

ROWS = {"quotient2_f64_cfg2": 1 << 26, "normalize2_f64_cfg2": 1 << 26, "quotient3_f64_cfg5": 1 << 28,
        "quotient3_fast_f64_cfg5": 1 << 28, "quotient3_f32_cfg4": 1 << 28, "quotient3_f64_cfg1": 1 << 20,
        "normalize3_f64_cfg5": 1 << 30, "norm3_f32_cfg4": 1 << 28, "norm3_f64_cfg5": 1 << 28,
        "normalize3_f32_cfg4": 1 << 28, "scale3_f32_cfg4": 1 << 28, "normalize3_sq_f32_cfg4": 1 << 28}


_SCALE = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12, "inst": 1, "cycle": 1,
          "kinst": 1e3, "minst": 1e6, "ginst": 1e9, "kcycle": 1e3, "mcycle": 1e6, "gcycle": 1e9}


def _num(v):
    val, unit = v
    return val * _SCALE.get(unit.lower(), 1)


def parse(path):
    vals = {}
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for row in csv.DictReader(lines):
        name, unit, v = row["Metric Name"], row["Metric Unit"], row["Metric Value"].replace(",", "")
        try:
            vals[name] = (float(v), unit)
        except ValueError:
            pass
    return vals


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    out = {}
    for path in sorted(glob.glob(f"gpurun_out/{tag}_issue_*.csv")):
        name = os.path.basename(path)[len(f"{tag}_issue_"):-4]
        v = parse(path)
        if "smsp__inst_executed.sum" not in v:
            continue
        n = ROWS[name]
        t_unit = v["gpu__time_duration.sum"][1]
        t = v["gpu__time_duration.sum"][0] * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1, "s": 1}[t_unit]
        clk = v["smsp__cycles_elapsed.avg.per_second"][0] * {"hz": 1, "khz": 1e3, "mhz": 1e6, "ghz": 1e9}[
            v["smsp__cycles_elapsed.avg.per_second"][1].lower()]
        inst = _num(v["smsp__inst_executed.sum"])
        fp64 = _num(v["smsp__inst_executed_pipe_fp64.sum"])
        out[name] = {
            "rows": n, "source": f"{os.path.basename(path)} (ncu --metrics, first launch, --clock-control none)",
            "warp_inst_per_row": inst / n, "fp64_warp_inst_per_row": fp64 / n,
            "thread_inst_per_row": _num(v["smsp__thread_inst_executed.sum"]) / n,
            "issue_active_per_row": _num(v["smsp__issue_active.sum"]) / n,
            "dram_bytes_per_row": (_num(v["dram__bytes_read.sum"]) + _num(v["dram__bytes_write.sum"])) / n,
            "ncu_time_s": t, "ncu_sm_clock_hz": clk,
            # one warp instruction per SMSP per cycle, 4 SMSPs x 148 SMs
            "issue_bound_s_at_ncu_clock": inst / (148 * 4 * clk),
            "issue_frac_under_ncu": inst / (148 * 4 * clk) / t,
        }
    dst = os.path.join("profiles", "ncu_issue.json")
    if "--merge" in sys.argv and os.path.exists(dst):  # keep the kernels of earlier passes
        with open(dst) as f:
            out = {**json.load(f), **out}
    with open(dst, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
