mkdir -p gpurun_out/r02h
timeout 2400 bash tools/ab_dyn.sh > gpurun_out/r02h/ab_dyn.txt 2>&1; echo "ab rc=$?"
timeout 600 python tools/probe/host_sweep.py 28 > gpurun_out/r02h/host_sweep.txt 2>&1; echo "host rc=$?"; cat gpurun_out/r02h/host_sweep.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_host_pool.py -m gpu -q -p no:cacheprovider -k "host" > gpurun_out/r02h/pytest_host.log 2>&1; echo "host tests rc=$?"; tail -2 gpurun_out/r02h/pytest_host.log
