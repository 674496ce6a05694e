#!/bin/bash
# Developer tool, run under gpurun: one `ncu --set full` capture per BASELINE config's
# main kernel (each after its plain run exited 0), ONE capture per gpurun call:
#   bash tools/gpu_ncu_configs.sh TAG cfg2_normalize2_f64
# (names below; without a name it lists them)
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-rX}
run() {  # name cfg log2rows op
  P="python tools/prof_target.py --cfg $2 --log2-rows $3 --iters 2 --op $4"
  timeout 300 $P > $OUT/${TAG}_$1_plain.log 2>&1 && \
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:tma_stream_kernel -s 1 -c 1 \
      -o $OUT/${TAG}_$1 $P > $OUT/${TAG}_$1_ncu.log 2>&1
  echo "$1 rc=$?"
}
case "${2:-}" in
  cfg2_normalize2_f64) run cfg2_normalize2_f64 2 26 normalize ;;
  cfg3_normalize4_sq_f64) run cfg3_normalize4_sq_f64 3 25 normalize_sq ;;
  cfg3_normalize4_rotation_f64) run cfg3_normalize4_rotation_f64 3 24 normalize4_rotation ;;
  cfg4_normalize3_f32) run cfg4_normalize3_f32 4 26 normalize ;;
  cfg5_norm3_f64) run cfg5_norm3_f64 5 26 norm ;;
  cfg2_quotient2_f64) run cfg2_quotient2_f64 2 24 quotient ;;
  *) echo "configs: cfg2_normalize2_f64 cfg3_normalize4_sq_f64 cfg3_normalize4_rotation_f64 cfg4_normalize3_f32 cfg5_norm3_f64 cfg2_quotient2_f64" ;;
esac
