# Round-1 build vs current build (static and dynamic schedule) on the naive and
# quotient3_fast kernels, which the ratio tables showed slower than in round 1.
set -u
mkdir -p gpurun_out/r02s
A="tools/ab/lib_r1.so tools/ab/lib_cur.so@FASTNORM_B200_DYN=0 tools/ab/lib_cur.so@FASTNORM_B200_DYN=1"
( python tools/ab_lib.py $A --op 3 --dim 3 --regime normal --log2-rows 24 --reps 20
  python tools/ab_lib.py $A --op 3 --dim 4 --regime normal --log2-rows 24 --reps 20
  python tools/ab_lib.py $A --op 5 --dim 3 --regime normal --log2-rows 24 --reps 20
  python tools/ab_lib.py $A --op 5 --dim 3 --cfg 5 --log2-rows 28 --reps 5
  python tools/ab_lib.py $A --op 3 --dim 3 --cfg 5 --log2-rows 28 --reps 5
  python tools/ab_lib.py $A --op 4 --dim 3 --regime normal --log2-rows 24 --reps 20 ) > gpurun_out/r02s/ab.txt 2>&1; echo "ab rc=$?"
