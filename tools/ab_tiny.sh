# A/B of the binary64 division (tiny-result path) on the division-bound variants
for i in 1 2; do for v in base tiny; do echo "== $v $i"; timeout 300 tools/ab/tune_$v 28 10 div | grep f64; done; done
