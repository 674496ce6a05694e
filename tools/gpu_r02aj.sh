# norm3 eager: previous build (67b8ba0) against the current one, and the rows sweep.
set -u
O=gpurun_out/r02aj; mkdir -p $O
L=paper_1606_06508_b200/libfastnorm_b200.so
for lg in 26 28; do
python tools/ab_lib.py tools/ab/lib_prev.so $L $L@FASTNORM_B200_DYN_VARIANT=4 tools/ab/lib_prev.so@FASTNORM_B200_DYN=0 --op 2 --dim 3 --cfg 5 --log2-rows $lg --reps 10 --rounds 2 >> $O/eager_norm3.txt 2>&1
done
python tools/ab_lib.py tools/ab/lib_prev.so $L $L@FASTNORM_B200_DYN_VARIANT=4 --op 1 --dim 3 --cfg 5 --log2-rows 28 --reps 10 --rounds 2 >> $O/eager_normalize3.txt 2>&1
python tools/ab_lib.py tools/ab/lib_prev.so $L $L@FASTNORM_B200_DYN_VARIANT=4 --op 1 --dim 2 --cfg 2 --log2-rows 26 --reps 10 --rounds 2 >> $O/eager_normalize2.txt 2>&1
echo done
