# norm kernels: tiles per claim (2 / 4 / 8) across dims and precisions; captured launches
# (dynamic for >= 32 tiles per CTA); many-batch kernel; tests on this build.
set -u
O=gpurun_out/r02al; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_dynamic_schedule.py tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_fuzz.py -m gpu -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
L=paper_1606_06508_b200/libfastnorm_b200.so
V="$L@FASTNORM_B200_SCHED_BATCH=2 $L $L@FASTNORM_B200_SCHED_BATCH=8 $L@FASTNORM_B200_DYN=0"
python tools/ab_lib.py $V --op 2 --dim 3 --cfg 5 --log2-rows 28 --reps 10 --rounds 2 >> $O/norm_batch.txt 2>&1
python tools/ab_lib.py $V --op 2 --dim 3 --cfg 5 --log2-rows 30 --reps 5 --rounds 2 >> $O/norm_batch.txt 2>&1
python tools/ab_lib.py $V --op 2 --dim 2 --cfg 2 --log2-rows 26 --reps 10 --rounds 2 >> $O/norm_batch.txt 2>&1
python tools/ab_lib.py $V --op 2 --dim 4 --cfg 3 --log2-rows 27 --reps 10 --rounds 2 >> $O/norm_batch.txt 2>&1
python tools/ab_lib.py $V --op 2 --dim 3 --cfg 4 --f32 --log2-rows 28 --reps 10 --rounds 2 >> $O/norm_batch.txt 2>&1
python tools/ab_lib.py $V --op 2 --dim 3 --cfg 1 --log2-rows 20 --reps 50 --rounds 2 >> $O/norm_batch.txt 2>&1
for rep in 1 2; do
  for m in 0 1; do FASTNORM_B200_DYN_CAPTURE=$m timeout 300 python tools/probe/graph_dyn.py >> $O/graph_dyn.jsonl 2>&1; done
  for v in "FASTNORM_B200_MANY_DYN=0 FASTNORM_B200_DYN_CAPTURE=0" "FASTNORM_B200_MANY_DYN=1 FASTNORM_B200_DYN_CAPTURE=1"; do
    echo "== $v" >> $O/many_ab.txt
    env $v timeout 200 python tools/probe/many_rate.py >> $O/many_ab.txt 2>&1
  done
done
echo done
