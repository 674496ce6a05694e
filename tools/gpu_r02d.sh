mkdir -p gpurun_out/r02d
timeout 600 python tools/probe/cfg1_dyn.py > gpurun_out/r02d/cfg1_dyn.txt 2>&1; echo "dyn rc=$?"; cat gpurun_out/r02d/cfg1_dyn.txt
timeout 900 python -m pytest tests/test_gpu_dynamic_schedule.py tests/test_gpu_host_pool.py tests/test_gpu_multirank.py -m gpu -q -p no:cacheprovider > gpurun_out/r02d/pytest_new.log 2>&1; echo "new rc=$?"; tail -3 gpurun_out/r02d/pytest_new.log
timeout 900 python tools/probe/host_default.py 28 > gpurun_out/r02d/host_default.txt 2>&1; echo "host rc=$?"; cat gpurun_out/r02d/host_default.txt
