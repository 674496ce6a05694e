# ncu --set full of quotient2 f64 on config 2 with and without the in-tile row sort.
set -u
mkdir -p gpurun_out/r02o
for v in sort0 sort1; do
  P="python tools/prof_target.py --cfg 2 --log2-rows 26 --iters 1 --op quotient"
  FASTNORM_B200_LIB=tools/ab/lib_$v.so timeout 300 $P > gpurun_out/r02o/plain_$v.log 2>&1 && \
  FASTNORM_B200_LIB=tools/ab/lib_$v.so timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:tma_stream_kernel -c 1 -o gpurun_out/r02o_quotient2_cfg2_$v $P > gpurun_out/r02o/ncu_$v.log 2>&1
  echo "$v rc=$?"
done
