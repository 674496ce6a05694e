# A/B of the binary32 division paths: quotient3 / naive3 / quotient3_fast f32 on config 4
# (full range) and on the in-band regime, plus the device self-test of Divider<float>.
A=tools/ab/libfastnorm_base.so; B=tools/ab/libfastnorm_f32native.so
for op in 4 3 5; do
  timeout 300 python tools/ab_lib.py $A $B --op $op --dim 3 --cfg 4 --f32 --log2-rows 28 --reps 10
  timeout 300 python tools/ab_lib.py $A $B --op $op --dim 3 --regime normal --f32 --log2-rows 28 --reps 10
done
