# In-tile row sort for the binary64 quotient kernels: parity, fuzz, A/B.
set -u
mkdir -p gpurun_out/r02n
timeout 600 python tools/probe/quotient_fuzz.py 1048576 2 > gpurun_out/r02n/fuzz.txt 2>&1; echo "fuzz rc=$?"; tail -1 gpurun_out/r02n/fuzz.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "quotient or baseline or selftest or division or golden or config or hypothesis or dynamic" > gpurun_out/r02n/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02n/pytest.log
timeout 1500 bash tools/ab_quotient.sh tools/ab/lib_sort0.so tools/ab/lib_sort1.so > gpurun_out/r02n/ab.txt 2>&1; echo "ab rc=$?"
