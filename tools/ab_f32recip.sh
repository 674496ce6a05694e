# binary32 division: Markstein in binary64 (old) vs one product with the shared binary64 reciprocal
A=tools/ab/lib_f32_markstein.so; B=tools/ab/lib_f32_recip.so
for op in 4 3 5; do
  timeout 300 python tools/ab_lib.py $A $B --op $op --dim 3 --cfg 4 --f32 --log2-rows 28 --reps 10
done
timeout 300 python tools/ab_lib.py $A $B --op 4 --dim 3 --regime normal --f32 --log2-rows 28 --reps 10
