# Full GPU suite + smoke + bench + reference arm on the build with fn_run_sharded, the SoA
# dynamic schedule and 3 SoA CTAs per SM; SoA rates on the final build.
set -u
O=gpurun_out/r02ag; mkdir -p $O
bash tools/gpu_round.sh r02ag tests,bench
timeout 200 python tools/probe/soa_rate.py > $O/soa_rate.jsonl 2>&1; echo "soa rc=$?"
timeout 200 python tools/probe/soa_columns_rate.py > $O/soa_columns_rate.jsonl 2>&1
timeout 200 python tools/probe/soa_misaligned_rate.py > $O/soa_misaligned_rate.jsonl 2>&1
