# CTAs per SM of the streaming kernel under the dynamic schedule, per kernel family.
set -u
mkdir -p gpurun_out/r02w
C=paper_1606_06508_b200/libfastnorm_b200.so
A="$C@FASTNORM_B200_CTAS_PER_SM=2 $C@FASTNORM_B200_CTAS_PER_SM=3 $C@FASTNORM_B200_CTAS_PER_SM=4"
( python tools/ab_lib.py $A --op 1 --dim 3 --cfg 5 --log2-rows 30 --reps 10
  python tools/ab_lib.py $A --op 1 --dim 3 --cfg 5 --log2-rows 28 --reps 10
  python tools/ab_lib.py $A --op 1 --dim 2 --cfg 2 --log2-rows 26 --reps 10
  python tools/ab_lib.py $A --op 1 --dim 4 --cfg 3 --log2-rows 27 --reps 10
  python tools/ab_lib.py $A --op 6 --dim 4 --cfg 3 --log2-rows 27 --reps 10
  python tools/ab_lib.py $A --op 9 --dim 4 --cfg 3 --log2-rows 27 --reps 10
  python tools/ab_lib.py $A --op 0 --dim 3 --cfg 5 --log2-rows 28 --reps 10
  python tools/ab_lib.py $A --op 1 --dim 3 --cfg 4 --log2-rows 28 --reps 10 --f32
  python tools/ab_lib.py $A --op 1 --dim 2 --regime normal --log2-rows 27 --reps 10 --f32
  python tools/ab_lib.py $A --op 1 --dim 4 --regime normal --log2-rows 26 --reps 10 --f32
  python tools/ab_lib.py $C@FASTNORM_B200_CTAS_PER_SM=4 $C@FASTNORM_B200_CTAS_PER_SM=3 $C@FASTNORM_B200_CTAS_PER_SM=6 --op 2 --dim 3 --cfg 5 --log2-rows 28 --reps 10
) > gpurun_out/r02w/ab.txt 2>&1; echo "ab rc=$?"
