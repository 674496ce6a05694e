mkdir -p gpurun_out/r02c
free -g > gpurun_out/r02c/host.txt; nproc >> gpurun_out/r02c/host.txt; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/r02c/host.txt
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_host_pool.py tests/test_gpu_signatures.py -m gpu -q -p no:cacheprovider > gpurun_out/r02c/pytest_new.log 2>&1; echo "new rc=$?"; tail -3 gpurun_out/r02c/pytest_new.log
timeout 900 python bench.py > gpurun_out/r02c/bench.json 2> gpurun_out/r02c/bench.err; echo "bench rc=$?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02c/pytest_gpu.log 2>&1; echo "all rc=$?"; tail -3 gpurun_out/r02c/pytest_gpu.log
