# Build with normalize3 f32 dynamic at 3 CTAs, normalize2_sq 3-deep: GPU suite + smoke + bench
# + reference arm, all-kernels table (2^26 and 2^28 rows), graph probe.
set -u
O=gpurun_out/r02aq; mkdir -p $O
bash tools/gpu_round.sh r02aq tests,bench
timeout 900 python tools/probe/all_kernels_rate.py > $O/all_kernels_2p26.jsonl 2>&1; echo "all26 rc=$?"
timeout 900 python tools/probe/all_kernels_rate.py --log2-rows 28 --reps 5 > $O/all_kernels_2p28.jsonl 2>&1; echo "all28 rc=$?"
timeout 300 python tools/probe/graph_dyn.py > $O/graph_dyn.jsonl 2>&1
