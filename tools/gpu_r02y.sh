# Ring depth / stage size of the streaming kernel under 3 CTAs per SM + dynamic schedule.
set -u
mkdir -p gpurun_out/r02y
A="tools/ab/lib_base.so tools/ab/lib_st3.so tools/ab/lib_st5.so tools/ab/lib_tb16k.so tools/ab/lib_tb4k.so"
( python tools/ab_lib.py $A --op 1 --dim 3 --cfg 5 --log2-rows 30 --reps 10
  python tools/ab_lib.py $A --op 1 --dim 2 --cfg 2 --log2-rows 26 --reps 10
  python tools/ab_lib.py $A --op 6 --dim 4 --cfg 3 --log2-rows 27 --reps 10
  python tools/ab_lib.py $A --op 1 --dim 3 --cfg 4 --log2-rows 28 --reps 10 --f32
  python tools/ab_lib.py $A --op 0 --dim 3 --cfg 5 --log2-rows 28 --reps 10
  python tools/ab_lib.py $A --op 9 --dim 4 --cfg 3 --log2-rows 26 --reps 10 ) > gpurun_out/r02y/ab.txt 2>&1; echo "ab rc=$?"
