# Build with half tiles for the 2-D binary32 division-bound kernels: GPU suite + smoke + bench
# + reference arm, and the A/B against the previous default.
set -u
O=gpurun_out/r02az; mkdir -p $O
bash tools/gpu_round.sh r02az tests,bench
L=paper_1606_06508_b200/libfastnorm_b200.so
python tools/ab_lib.py $L tools/ab/lib_d32s1.so --op 4 --dim 2 --regime mixed --f32 --log2-rows 27 --reps 10 --rounds 2 >> $O/check.txt 2>&1
python tools/ab_lib.py $L tools/ab/lib_d32s1.so --op 4 --dim 3 --cfg 4 --f32 --log2-rows 28 --reps 10 --rounds 2 >> $O/check.txt 2>&1
python tools/ab_lib.py $L tools/ab/lib_d32s1.so --op 3 --dim 3 --regime normal --f32 --log2-rows 27 --reps 10 --rounds 2 >> $O/check.txt 2>&1
