# normalize2 f64 at 2^24 and 2^26 rows per CTAs-per-SM setting (stream kernel launch shape)
for cps in 0 2 3 4 6 8; do
  for lg in 24 26; do
    if [ $cps = 0 ]; then unset FASTNORM_B200_CTAS_PER_SM; else export FASTNORM_B200_CTAS_PER_SM=$cps; fi
    echo "cps=$cps rows=2^$lg"
    timeout 120 python -m paper_1606_06508_b200 ratios --dim 2 --algo scaling --algo quotient --experiments 3 --rows $((1<<lg)) | grep -E "^normalize2d"
  done
done
