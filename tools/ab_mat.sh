# per-row matrix apply (FN_OP_MAT_APPLY) tile geometry variants, through the library
for i in 1 2; do
for v in 64_4 128_4 128_3 256_2 256_3; do
  FASTNORM_B200_LIB=tools/ab/lib_mat_$v.so timeout 120 python tools/probe/rotate_rows_rate.py 26 | grep apply_rotations | sed "s/^/$v /"
done; done
