#!/bin/bash
# Static vs dynamic tile schedule (FASTNORM_B200_DYN) of one library on every config
# kernel, back-to-back launches as in the bench.  usage: bash tools/ab_dyn.sh LIB.so
L=${1:-paper_1606_06508_b200/libfastnorm_b200.so}
A="$L@FASTNORM_B200_DYN=0 $L@FASTNORM_B200_DYN=1"
python tools/ab_lib.py $A --op 1 --dim 3 --cfg 5 --log2-rows 30 --reps 10
python tools/ab_lib.py $A --op 1 --dim 3 --cfg 4 --log2-rows 28 --reps 10 --f32
python tools/ab_lib.py $A --op 6 --dim 4 --cfg 3 --log2-rows 27 --reps 10
python tools/ab_lib.py $A --op 1 --dim 2 --cfg 2 --log2-rows 26 --reps 20
python tools/ab_lib.py $A --op 4 --dim 2 --cfg 2 --log2-rows 26 --reps 10
python tools/ab_lib.py $A --op 4 --dim 3 --cfg 5 --log2-rows 28 --reps 5
python tools/ab_lib.py $A --op 4 --dim 3 --cfg 1 --log2-rows 28 --reps 5
python tools/ab_lib.py $A --op 4 --dim 4 --cfg 3 --log2-rows 27 --reps 5
python tools/ab_lib.py $A --op 4 --dim 3 --cfg 4 --log2-rows 28 --reps 5 --f32
python tools/ab_lib.py $A --op 2 --dim 3 --cfg 5 --log2-rows 28 --reps 10
