# 3-D f64 / f32 tile geometry confirmation (2^30 and 2^28 rows, three rounds).
set -u
mkdir -p gpurun_out/r02z
A="tools/ab/lib_base.so tools/ab/lib_tb16k.so tools/ab/lib_st3.so tools/ab/lib_v512s3.so tools/ab/lib_v512s2c2.so"
( python tools/ab_lib.py $A --op 1 --dim 3 --cfg 5 --log2-rows 30 --reps 10 --rounds 3
  python tools/ab_lib.py $A --op 1 --dim 3 --cfg 5 --log2-rows 28 --reps 10 --rounds 3
  python tools/ab_lib.py $A --op 1 --dim 3 --cfg 1 --log2-rows 28 --reps 10 --rounds 2
  python tools/ab_lib.py $A --op 0 --dim 3 --cfg 5 --log2-rows 28 --reps 10 --rounds 2
  python tools/ab_lib.py tools/ab/lib_base.so tools/ab/lib_st5.so tools/ab/lib_st6.so --op 1 --dim 3 --cfg 4 --log2-rows 28 --reps 10 --f32 --rounds 3 ) > gpurun_out/r02z/ab.txt 2>&1; echo "ab rc=$?"
