# All kernels on the final build; binary32 kernels at 2 / 4 / 8 tiles per claim; normalize3 f32
# on the dynamic schedule (FNB_DYN_F32_NORMALIZE3=1 build) at the same batches.
set -u
O=gpurun_out/r02an; mkdir -p $O
timeout 900 python tools/probe/all_kernels_rate.py > $O/all_kernels.jsonl 2>&1; echo "all rc=$?"
L=paper_1606_06508_b200/libfastnorm_b200.so
D=tools/ab/lib_f32dyn.so
python tools/ab_lib.py $L $D@FASTNORM_B200_SCHED_BATCH=2 $D@FASTNORM_B200_SCHED_BATCH=4 $D@FASTNORM_B200_SCHED_BATCH=8 --op 1 --dim 3 --cfg 4 --f32 --log2-rows 28 --reps 10 --rounds 2 >> $O/f32_normalize3.txt 2>&1
V="$L@FASTNORM_B200_SCHED_BATCH=2 $L@FASTNORM_B200_SCHED_BATCH=4 $L@FASTNORM_B200_SCHED_BATCH=8 $L@FASTNORM_B200_DYN=0"
for dim in 2 4; do
python tools/ab_lib.py $V --op 1 --dim $dim --regime mixed --f32 --log2-rows 28 --reps 10 --rounds 2 >> $O/f32_batch.txt 2>&1
done
python tools/ab_lib.py $V --op 0 --dim 3 --regime mixed --f32 --log2-rows 28 --reps 10 --rounds 2 >> $O/f32_batch.txt 2>&1
python tools/ab_lib.py $V --op 1 --dim 2 --cfg 2 --log2-rows 26 --reps 10 --rounds 2 >> $O/f64_batch.txt 2>&1
python tools/ab_lib.py $V --op 0 --dim 3 --cfg 5 --log2-rows 28 --reps 10 --rounds 2 >> $O/f64_batch.txt 2>&1
python tools/ab_lib.py $V --op 6 --dim 4 --cfg 3 --log2-rows 27 --reps 10 --rounds 2 >> $O/f64_batch.txt 2>&1
echo done
