# A/B of the binary64 division variants on the division-bound kernels (tools/ab/tune_*)
for i in 1 2; do for v in "$@"; do echo "== $v $i"; timeout 300 tools/ab/tune_$v 28 10 div | grep f64; done; done
