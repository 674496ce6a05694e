mkdir -p gpurun_out/r02e
timeout 600 python tools/probe/cfg1_dyn.py > gpurun_out/r02e/cfg1_dyn.txt 2>&1; echo "dyn rc=$?"; cat gpurun_out/r02e/cfg1_dyn.txt
timeout 900 python tools/probe/host_sweep.py 28 > gpurun_out/r02e/host_sweep.txt 2>&1; echo "host rc=$?"; cat gpurun_out/r02e/host_sweep.txt
timeout 1200 bash tools/ab_quotient.sh tools/ab/lib_qpiv0.so tools/ab/lib_qpiv1.so tools/ab/lib_qpiv1m.so > gpurun_out/r02e/ab_quotient.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/r02e/ab_quotient.txt
