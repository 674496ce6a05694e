# Capture-safe dynamic schedule + many-batch kernel on the dynamic schedule: tests, A/B.
set -u
O=gpurun_out/r02ah; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_dynamic_schedule.py tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for rep in 1 2; do
  for m in 0 1; do FASTNORM_B200_DYN_CAPTURE=$m timeout 300 python tools/probe/graph_dyn.py >> $O/graph_dyn.jsonl 2>&1; done
  for v in "FASTNORM_B200_MANY_DYN=0 FASTNORM_B200_DYN_CAPTURE=0" "FASTNORM_B200_MANY_DYN=1 FASTNORM_B200_DYN_CAPTURE=0" "FASTNORM_B200_MANY_DYN=1 FASTNORM_B200_DYN_CAPTURE=1"; do
    echo "== $v" >> $O/many_ab.txt
    env $v timeout 200 python tools/probe/many_rate.py >> $O/many_ab.txt 2>&1
  done
done
echo "ab rc=$?"
