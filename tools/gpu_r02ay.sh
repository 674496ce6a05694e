# binary32 division-bound kernels with smaller tiles (more CTAs per SM): A/B.
set -u
O=gpurun_out/r02ay; mkdir -p $O
L=paper_1606_06508_b200/libfastnorm_b200.so
V="$L tools/ab/lib_d32s1.so tools/ab/lib_d32s2.so"
run() { python tools/ab_lib.py $V "$@" --f32 --reps 10 --rounds 2 >> $O/div32.txt 2>&1; }
run --op 4 --dim 2 --regime normal --log2-rows 27
run --op 4 --dim 2 --regime mixed --log2-rows 27
run --op 4 --dim 3 --cfg 4 --log2-rows 28
run --op 4 --dim 3 --regime normal --log2-rows 27
run --op 4 --dim 4 --regime mixed --log2-rows 27
run --op 3 --dim 2 --regime mixed --log2-rows 27
run --op 3 --dim 3 --regime normal --log2-rows 27
run --op 5 --dim 3 --cfg 4 --log2-rows 28
run --op 4 --dim 3 --regime normal --log2-rows 20
echo done
