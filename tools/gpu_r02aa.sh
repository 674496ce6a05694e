# Big-tile build: GPU suite, smoke, bench, and the other row layouts' rate probes.
set -u
mkdir -p gpurun_out/r02aa
bash tools/gpu_round.sh r02aa tests,bench
timeout 600 python tools/probe/padded_rate.py 27 > gpurun_out/r02aa/padded.txt 2>&1; echo "padded rc=$?"
timeout 600 python tools/probe/unaligned_rate.py > gpurun_out/r02aa/unaligned.txt 2>&1; echo "unaligned rc=$?"
timeout 600 python tools/probe/many_rate.py > gpurun_out/r02aa/many.txt 2>&1; echo "many rc=$?"
A="tools/ab/lib_base.so paper_1606_06508_b200/libfastnorm_b200.so"
( python tools/ab_lib.py $A --op 2 --dim 3 --cfg 5 --log2-rows 28 --reps 10
  python tools/ab_lib.py $A --op 10 --dim 3 --cfg 5 --log2-rows 28 --reps 10
  python tools/ab_lib.py $A --op 1 --dim 3 --cfg 5 --log2-rows 30 --reps 10
  python tools/ab_lib.py $A --op 6 --dim 3 --cfg 5 --log2-rows 28 --reps 10 ) > gpurun_out/r02aa/ab.txt 2>&1; echo "ab rc=$?"
