#!/bin/bash
# A/B of quotient-family builds (tools/build_ab.sh) on every config that runs them.
# usage: bash tools/ab_quotient.sh tools/ab/lib_A.so tools/ab/lib_B.so ...
python tools/ab_lib.py "$@" --op 4 --dim 2 --cfg 2 --log2-rows 26 --reps 10
python tools/ab_lib.py "$@" --op 4 --dim 3 --cfg 5 --log2-rows 28 --reps 5
python tools/ab_lib.py "$@" --op 4 --dim 3 --cfg 1 --log2-rows 28 --reps 5
python tools/ab_lib.py "$@" --op 4 --dim 4 --cfg 3 --log2-rows 27 --reps 5
python tools/ab_lib.py "$@" --op 4 --dim 3 --cfg 4 --log2-rows 28 --reps 5 --f32
python tools/ab_lib.py "$@" --op 5 --dim 3 --cfg 5 --log2-rows 28 --reps 5
