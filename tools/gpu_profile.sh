#!/bin/bash
# Developer tool, run under gpurun: tile sweep + ncu launch list of bench.py + one
# `ncu --set full` capture of the top kernel (each after its plain run exited 0).
set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=${1:-r01}
make -s -C tools tune >/dev/null 2>&1
timeout 300 tools/tune_stream 28 20 > $OUT/${TAG}_tune.csv 2>&1; echo "tune rc=$?"
BENCH="python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
timeout 600 $BENCH > $OUT/${TAG}_bench_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
     --log-file $OUT/${TAG}_launches.csv $BENCH > $OUT/${TAG}_ncu_launch.log 2>&1; echo "launch list rc=$?"
PROF="python tools/prof_target.py --cfg 5 --log2-rows 26 --iters 2"
timeout 300 $PROF > $OUT/${TAG}_prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tma_stream_kernel -c 1 \
     -o $OUT/${TAG}_normalize3_f64 $PROF > $OUT/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
