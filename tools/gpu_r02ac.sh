# Exponent insertion (FNB_EXPONENT_INSERTION=1, libfastnorm_b200_insert.so) against the
# default exact power-of-two multiply on the current geometry, process-alternated.
set -u
mkdir -p gpurun_out/r02ac
A="paper_1606_06508_b200/libfastnorm_b200.so paper_1606_06508_b200/libfastnorm_b200_insert.so"
( python tools/ab_lib.py $A --op 1 --dim 3 --cfg 5 --log2-rows 30 --reps 10
  python tools/ab_lib.py $A --op 1 --dim 3 --cfg 4 --log2-rows 28 --f32 --reps 10
  python tools/ab_lib.py $A --op 1 --dim 2 --cfg 2 --log2-rows 26 --reps 20
  python tools/ab_lib.py $A --op 6 --dim 4 --cfg 3 --log2-rows 27 --reps 10
  python tools/ab_lib.py $A --op 1 --dim 3 --cfg 1 --log2-rows 20 --reps 50
) > gpurun_out/r02ac/ab_insert.txt 2>&1; echo "ab rc=$?"
