# Fuzz tests of every family and the paper's ratio tables (normal and mixed regimes).
set -u
mkdir -p gpurun_out/r02r
timeout 900 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider > gpurun_out/r02r/pytest_fuzz.log 2>&1; echo "fuzz rc=$?"; tail -3 gpurun_out/r02r/pytest_fuzz.log
for regime in normal mixed; do
  timeout 300 python -m paper_1606_06508_b200 ratios --regime $regime --prec double --prec single \
    --experiments 5 --rows 16777216 --json gpurun_out/r02r/ratios_$regime.json > gpurun_out/r02r/ratios_$regime.txt 2>&1
  echo "ratios $regime rc=$?"
done
