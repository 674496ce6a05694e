mkdir -p gpurun_out/r02f
timeout 1500 python -m pytest tests/test_gpu_dynamic_schedule.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_host_pool.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r02f/pytest_default.log 2>&1; echo "default rc=$?"; tail -3 gpurun_out/r02f/pytest_default.log
FASTNORM_B200_LIB=$PWD/tools/ab/lib_qtiny.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -q -p no:cacheprovider -k "golden or random_full_range or reference_regimes or tail or cfg2 or cfg5 or division" > gpurun_out/r02f/pytest_qtiny.log 2>&1; echo "qtiny rc=$?"; tail -3 gpurun_out/r02f/pytest_qtiny.log
timeout 1200 bash tools/ab_quotient.sh tools/ab/lib_qpiv0.so tools/ab/lib_qpiv1.so tools/ab/lib_qtiny.so > gpurun_out/r02f/ab_quotient.txt 2>&1; echo "ab rc=$?"
timeout 600 python tools/probe/cfg1_dyn.py > gpurun_out/r02f/cfg1_dyn.txt 2>&1; echo "dyn rc=$?"; cat gpurun_out/r02f/cfg1_dyn.txt
timeout 600 python tools/probe/host_sweep.py 28 > gpurun_out/r02f/host_sweep.txt 2>&1; echo "host rc=$?"; cat gpurun_out/r02f/host_sweep.txt
timeout 900 python bench.py > gpurun_out/r02f/bench.json 2> gpurun_out/r02f/bench.err; echo "bench rc=$?"
