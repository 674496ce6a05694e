# Sharded driver tests + rate, SoA kernel with the dynamic schedule: parity tests and A/B.
set -u
O=gpurun_out/r02ae; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py tests/test_gpu_dynamic_schedule.py -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 600 python tools/probe/sharded_rate.py --log2-rows 28 > $O/sharded_rate.jsonl 2>&1; echo "sharded rc=$?"
timeout 300 python tools/probe/sharded_rate.py --log2-rows 30 --reps 5 >> $O/sharded_rate.jsonl 2>&1; echo "sharded30 rc=$?"
for rep in 1 2; do
for v in "FASTNORM_B200_SOA_DYN=0" "FASTNORM_B200_SOA_DYN=1" "FASTNORM_B200_SOA_DYN=1 FASTNORM_B200_SCHED_BATCH=1" "FASTNORM_B200_SOA_DYN=1 FASTNORM_B200_SCHED_BATCH=4"; do
  echo "== $v" >> $O/soa_ab.txt
  env $v timeout 200 python tools/probe/soa_rate.py >> $O/soa_ab.txt 2>&1
done
done
echo "soa ab rc=$?"
