#!/bin/bash
# Developer tool, run under gpurun: one `ncu --set full` capture per BASELINE config's
# main kernel (each after its plain run exited 0).  Usage: bash tools/gpu_ncu_configs.sh TAG
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-rX}
run() {  # name cfg log2rows op
  P="python tools/prof_target.py --cfg $2 --log2-rows $3 --iters 2 --op $4"
  timeout 300 $P > $OUT/${TAG}_$1_plain.log 2>&1 && \
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:tma_stream_kernel -s 1 -c 1 \
      -o $OUT/${TAG}_$1 $P > $OUT/${TAG}_$1_ncu.log 2>&1
  echo "$1 rc=$?"
}
run cfg2_normalize2_f64 2 26 normalize
run cfg3_normalize4_sq_f64 3 25 normalize_sq
run cfg3_normalize4_rotation_f64 3 24 normalize4_rotation
run cfg4_normalize3_f32 4 26 normalize
run cfg5_norm3_f64 5 26 norm
