# Sharded driver tests; SoA parity tests on the dynamic schedule; SoA CTAs-per-SM sweep.
set -u
O=gpurun_out/r02af; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py tests/test_gpu_dynamic_schedule.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for rep in 1 2; do
for v in "FASTNORM_B200_CTAS_PER_SM=2" "FASTNORM_B200_CTAS_PER_SM=3" "FASTNORM_B200_CTAS_PER_SM=4"; do
  echo "== $v" >> $O/soa_ctas.txt
  env $v timeout 200 python tools/probe/soa_rate.py >> $O/soa_ctas.txt 2>&1
done
done
echo "soa ctas rc=$?"
for f in soa_columns_rate soa_misaligned_rate; do timeout 200 python tools/probe/$f.py > $O/$f.jsonl 2>&1; echo "$f rc=$?"; done
