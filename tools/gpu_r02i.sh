mkdir -p gpurun_out/r02i
timeout 2400 bash tools/ab_dyn.sh > gpurun_out/r02i/ab_dyn.txt 2>&1; echo "ab rc=$?"
timeout 900 python -m pytest tests/test_gpu_dynamic_schedule.py -m gpu -q -p no:cacheprovider > gpurun_out/r02i/pytest_dyn.log 2>&1; echo "dyn tests rc=$?"; tail -2 gpurun_out/r02i/pytest_dyn.log
timeout 600 python tools/probe/cfg1_dyn.py > gpurun_out/r02i/cfg1_dyn.txt 2>&1; echo "cfg1 rc=$?"
