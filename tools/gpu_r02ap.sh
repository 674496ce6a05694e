# normalize3 f32 on the dynamic schedule at 3 CTAs per SM; normalize2_sq with a 3-deep ring.
set -u
O=gpurun_out/r02ap; mkdir -p $O
L=paper_1606_06508_b200/libfastnorm_b200.so
D=tools/ab/lib_f32dyn.so
S=tools/ab/lib_sq2s3.so
python tools/ab_lib.py $L $D@FASTNORM_B200_CTAS_PER_SM=3 $D@FASTNORM_B200_CTAS_PER_SM=4 $D@FASTNORM_B200_CTAS_PER_SM=3,FASTNORM_B200_SCHED_BATCH=4 $L@FASTNORM_B200_CTAS_PER_SM=3 --op 1 --dim 3 --cfg 4 --f32 --log2-rows 28 --reps 10 --rounds 2 >> $O/f32_normalize3.txt 2>&1
python tools/ab_lib.py $L $D@FASTNORM_B200_CTAS_PER_SM=3 $D@FASTNORM_B200_CTAS_PER_SM=4 --op 1 --dim 3 --regime normal --f32 --log2-rows 26 --reps 10 --rounds 2 >> $O/f32_normalize3.txt 2>&1
for a in "--regime normal --f32" "--regime mixed --f32" "--regime normal" "--regime mixed"; do
python tools/ab_lib.py $L $S $S@FASTNORM_B200_CTAS_PER_SM=4 $S@FASTNORM_B200_DYN=0 --op 6 --dim 2 $a --log2-rows 27 --reps 10 --rounds 2 >> $O/sq2.txt 2>&1
done
echo done
