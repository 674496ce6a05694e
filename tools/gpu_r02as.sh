# 3-D binary32 scaling kernels inside one process (the all-kernels probe): schedule variants.
set -u
O=gpurun_out/r02as; mkdir -p $O
for v in "X=0" "FASTNORM_B200_SCHED_BATCH=4" "FASTNORM_B200_SCHED_BATCH=8" "FASTNORM_B200_CTAS_PER_SM=4" "FASTNORM_B200_CTAS_PER_SM=2" "FASTNORM_B200_DYN=0"; do
 for lg in 26 28; do
  echo "== $v 2^$lg" >> $O/f32_dim3.txt
  env $v timeout 300 python tools/probe/all_kernels_rate.py --precs single --dims 3 --kernels scale,normalize,norm,normalize_sq --log2-rows $lg --reps 10 >> $O/f32_dim3.txt 2>&1
 done
done
echo done
