# The kernels the all-kernels table shows below the copy peak: schedule / CTAs / batch sweeps.
set -u
O=gpurun_out/r02ao; mkdir -p $O
L=paper_1606_06508_b200/libfastnorm_b200.so
V="$L $L@FASTNORM_B200_DYN=0 $L@FASTNORM_B200_CTAS_PER_SM=2 $L@FASTNORM_B200_CTAS_PER_SM=3 $L@FASTNORM_B200_CTAS_PER_SM=4 $L@FASTNORM_B200_SCHED_BATCH=4 $L@FASTNORM_B200_SCHED_BATCH=1"
run() { python tools/ab_lib.py $V "$@" --log2-rows 27 --reps 10 --rounds 2 >> $O/sweep.txt 2>&1; }
run --op 0 --dim 3 --regime normal --f32
run --op 2 --dim 3 --regime normal --f32
run --op 6 --dim 2 --regime normal --f32
run --op 6 --dim 3 --regime normal --f32
run --op 6 --dim 2 --regime mixed
run --op 6 --dim 2 --regime normal
echo done
