#!/bin/bash
# Instruction-issue roofline inputs for the division-bound comparison kernels and the
# headline kernel: one ncu metrics pass per kernel (first launch, cold), CSV into
# gpurun_out/$TAG_issue_*.csv; tools/issue_json.py turns them into profiles/ncu_issue.json.
TAG=${1:-r02}
OUT=gpurun_out; mkdir -p $OUT
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.sum,sm__cycles_elapsed.avg,smsp__cycles_elapsed.avg.per_second,smsp__inst_executed_pipe_fp64.sum,smsp__pipe_fp64_cycles_active.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed.sum
run() {  # name, prof_target args
  local name=$1; shift
  timeout 300 python tools/prof_target.py "$@" --iters 1 > /dev/null 2>&1 || { echo "$name: plain run failed"; return; }
  timeout 900 ncu --metrics $M --clock-control none -k regex:tma_stream_kernel -c 1 --csv \
    python tools/prof_target.py "$@" --iters 1 > $OUT/${TAG}_issue_$name.csv 2> $OUT/${TAG}_issue_$name.err
  echo "$name rc=$?"
}
run quotient2_f64_cfg2 --cfg 2 --log2-rows 26 --op quotient
run normalize2_f64_cfg2 --cfg 2 --log2-rows 26 --op normalize
run quotient3_f64_cfg5 --cfg 5 --log2-rows 28 --op quotient
run quotient3_fast_f64_cfg5 --cfg 5 --log2-rows 28 --op quotient3_fast
run quotient3_f32_cfg4 --cfg 4 --log2-rows 28 --op quotient
run quotient3_f64_cfg1 --cfg 1 --log2-rows 20 --op quotient
run normalize3_f64_cfg5 --cfg 5 --log2-rows 30 --op normalize
