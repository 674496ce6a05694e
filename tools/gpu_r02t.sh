# Tiles per claim of the dynamic schedule (FASTNORM_B200_SCHED_BATCH) vs the static schedule.
set -u
mkdir -p gpurun_out/r02t
L=tools/ab/lib_cur.so
A="$L@FASTNORM_B200_DYN=0 $L@FASTNORM_B200_SCHED_BATCH=1 $L@FASTNORM_B200_SCHED_BATCH=2 $L@FASTNORM_B200_SCHED_BATCH=4 $L@FASTNORM_B200_SCHED_BATCH=8 $L@FASTNORM_B200_SCHED_BATCH=16"
( python tools/ab_lib.py $A --op 3 --dim 3 --regime normal --log2-rows 24 --reps 20 --rounds 2
  python tools/ab_lib.py $A --op 5 --dim 3 --regime normal --log2-rows 24 --reps 20 --rounds 2
  python tools/ab_lib.py $A --op 4 --dim 3 --regime normal --log2-rows 24 --reps 20 --rounds 2
  python tools/ab_lib.py $A --op 1 --dim 3 --cfg 5 --log2-rows 28 --reps 5 --rounds 2
  python tools/ab_lib.py $A --op 1 --dim 2 --cfg 2 --log2-rows 26 --reps 10 --rounds 2
  python tools/ab_lib.py $A --op 4 --dim 3 --cfg 1 --log2-rows 28 --reps 5 --rounds 2
  python tools/ab_lib.py $A --op 2 --dim 3 --cfg 5 --log2-rows 28 --reps 5 --rounds 2
  python tools/ab_lib.py $A --op 3 --dim 3 --cfg 5 --log2-rows 28 --reps 5 --rounds 2
  python tools/ab_lib.py $A --op 1 --dim 3 --cfg 4 --log2-rows 28 --reps 5 --rounds 2 --f32 ) > gpurun_out/r02t/ab.txt 2>&1; echo "ab rc=$?"
