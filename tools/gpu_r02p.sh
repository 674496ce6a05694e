# Geometry of the binary64 division-bound kernels (tile rows, stages, CTAs, register cap).
set -u
mkdir -p gpurun_out/r02p
timeout 2400 bash tools/ab_quotient.sh tools/ab/lib_g0.so tools/ab/lib_g_r1s3.so tools/ab/lib_g_s2.so tools/ab/lib_g_r1s4.so tools/ab/lib_g_s2mb6.so tools/ab/lib_g_r1s2.so > gpurun_out/r02p/ab.txt 2>&1; echo "ab rc=$?"
