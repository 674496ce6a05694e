# The paper's T3/T4 ratio tables on the GPU for every reference regime (both precisions)
for regime in normal mixed huge subnormal unit-ish; do
  timeout 300 python -m paper_1606_06508_b200 ratios --regime $regime --prec double --prec single \
    --experiments 5 --rows 16777216 --json gpurun_out/r01bj_ratios_$regime.json
done
