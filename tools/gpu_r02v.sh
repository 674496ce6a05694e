# normalize3 f32 static vs dynamic (2-tile claims), and CTAs per SM of the headline kernel.
set -u
mkdir -p gpurun_out/r02v
L=tools/ab/lib_f32dyn.so
( python tools/ab_lib.py $L@FASTNORM_B200_DYN=0 $L@FASTNORM_B200_DYN=1 --op 1 --dim 3 --cfg 4 --log2-rows 28 --reps 10 --f32
  python tools/ab_lib.py $L@FASTNORM_B200_DYN=0 $L@FASTNORM_B200_DYN=1 --op 1 --dim 3 --regime normal --log2-rows 26 --reps 10 --f32
  C=paper_1606_06508_b200/libfastnorm_b200.so
  python tools/ab_lib.py $C@FASTNORM_B200_CTAS_PER_SM=2 $C@FASTNORM_B200_CTAS_PER_SM=3 $C@FASTNORM_B200_CTAS_PER_SM=4 $C@FASTNORM_B200_CTAS_PER_SM=1 --op 1 --dim 3 --cfg 5 --log2-rows 30 --reps 10
  python tools/ab_lib.py $C@FASTNORM_B200_CTAS_PER_SM=2 $C@FASTNORM_B200_CTAS_PER_SM=3 $C@FASTNORM_B200_CTAS_PER_SM=4 --op 1 --dim 2 --cfg 2 --log2-rows 26 --reps 10
  python tools/ab_lib.py $C@FASTNORM_B200_CTAS_PER_SM=2 $C@FASTNORM_B200_CTAS_PER_SM=3 $C@FASTNORM_B200_CTAS_PER_SM=4 --op 6 --dim 4 --cfg 3 --log2-rows 27 --reps 10
) > gpurun_out/r02v/ab.txt 2>&1; echo "ab rc=$?"
