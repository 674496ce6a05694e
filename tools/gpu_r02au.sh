# Issue-roofline inputs (warp instructions per row) for the binary32 3-D scaling kernels and
# norm3: one ncu metrics pass per kernel, as tools/ncu_issue.sh.
TAG=r02au
OUT=gpurun_out; mkdir -p $OUT
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.sum,sm__cycles_elapsed.avg,smsp__cycles_elapsed.avg.per_second,smsp__inst_executed_pipe_fp64.sum,smsp__pipe_fp64_cycles_active.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__thread_inst_executed.sum
run() {  # name, prof_target args
  local name=$1; shift
  timeout 300 python tools/prof_target.py "$@" --iters 1 > /dev/null 2>&1 || { echo "$name: plain run failed"; return; }
  timeout 900 ncu --metrics $M --clock-control none -k regex:tma_stream_kernel -c 1 --csv \
    python tools/prof_target.py "$@" --iters 1 > $OUT/${TAG}_issue_$name.csv 2> $OUT/${TAG}_issue_$name.err
  echo "$name rc=$?"
}
run norm3_f32_cfg4 --cfg 4 --log2-rows 28 --op norm
run norm3_f64_cfg5 --cfg 5 --log2-rows 28 --op norm
run normalize3_f32_cfg4 --cfg 4 --log2-rows 28 --op normalize
run scale3_f32_cfg4 --cfg 4 --log2-rows 28 --op scale
run normalize3_sq_f32_cfg4 --cfg 4 --log2-rows 28 --op normalize_sq
