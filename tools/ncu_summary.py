"""Summarise an ncu --set full report (developer tool; run in the build container).

python tools/ncu_summary.py gpurun_out/r01_normalize3_f64.ncu-rep ROWS [--key normalize3_f64]
Prints the metrics the roofline uses and, with --write-traffic, records DRAM bytes per
row in profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_shared_mem", "lts__t_bytes.sum", "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("rows", type=int)
    ap.add_argument("--key", default="normalize3_f64")
    ap.add_argument("--algo-bytes-per-row", type=float, default=56.0)
    ap.add_argument("--write-traffic", action="store_true")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    got = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            got[k] = (vals[i], units[i])
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    print(f"kernel: {name}")
    print(f"rows per launch: {a.rows}")
    for k, (v, u) in got.items():
        print(f"{k}: {v} {u}")

    def as_bytes(v, u):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
        return float(v.replace(",", "")) * scale

    rd = as_bytes(*got["dram__bytes_read.sum"])
    wr = as_bytes(*got["dram__bytes_write.sum"])
    t_us = float(got["gpu__time_duration.sum"][0].replace(",", "")) * {
        "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}[got["gpu__time_duration.sum"][1]]
    per_row = (rd + wr) / a.rows
    print(f"dram bytes per row: {per_row:.3f} (algorithmic {a.algo_bytes_per_row})")
    print(f"ncu duration: {t_us:.1f} us -> algorithmic {a.rows * a.algo_bytes_per_row / t_us / 1e3:.1f} GB/s "
          f"(cold-cache, serialised, clocks uncontrolled)")
    if a.write_traffic:
        path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                            "ncu_traffic.json")
        d = json.load(open(path)) if os.path.exists(path) else {}
        d[a.key] = {"dram_bytes_per_row": per_row, "dram_read_bytes": rd, "dram_write_bytes": wr,
                    "rows": a.rows, "source": os.path.basename(a.report) + " (ncu --set full)"}
        json.dump(d, open(path, "w"), indent=1)
        print("wrote", path)


if __name__ == "__main__":
    main()
