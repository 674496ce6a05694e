# WideDivider (warp-uniform exact binary64 division): self-test, quotient parity, A/B.
set -u
mkdir -p gpurun_out/r02l
timeout 900 python tools/selftest_big.py 2 > gpurun_out/r02l/selftest.txt 2>&1; echo "selftest rc=$?"; cat gpurun_out/r02l/selftest.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "quotient or baseline or selftest or division or golden or config or hypothesis or insertion or dynamic" > gpurun_out/r02l/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02l/pytest.log
timeout 1500 bash tools/ab_quotient.sh tools/ab/lib_wide0.so tools/ab/lib_wide1.so > gpurun_out/r02l/ab.txt 2>&1; echo "ab rc=$?"
