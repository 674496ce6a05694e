# quotient2 two-stage confirmation A/B over regimes, then the GPU suite and the bench.
set -u
mkdir -p gpurun_out/r02q
A="tools/ab/lib_g0.so tools/ab/lib_q2s2.so"
( python tools/ab_lib.py $A --op 4 --dim 2 --cfg 2 --log2-rows 26 --reps 10
  for r in normal unit-ish mixed subnormal; do python tools/ab_lib.py $A --op 4 --dim 2 --regime $r --log2-rows 26 --reps 10; done
  python tools/ab_lib.py $A --op 4 --dim 3 --cfg 5 --log2-rows 28 --reps 5 ) > gpurun_out/r02q/ab.txt 2>&1; echo "ab rc=$?"
bash tools/gpu_round.sh r02q tests,bench
