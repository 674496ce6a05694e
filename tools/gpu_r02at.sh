# Final build of the round: GPU suite + smoke + bench + reference arm, all-kernels table.
set -u
O=gpurun_out/r02at; mkdir -p $O
bash tools/gpu_round.sh r02at tests,bench
timeout 900 python tools/probe/all_kernels_rate.py --log2-rows 28 --reps 5 > $O/all_kernels_2p28.jsonl 2>&1; echo "all28 rc=$?"
timeout 900 python tools/probe/all_kernels_rate.py > $O/all_kernels_2p26.jsonl 2>&1; echo "all26 rc=$?"
