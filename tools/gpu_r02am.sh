# Full GPU suite + smoke + bench + reference arm on the build with the capture-safe
# dynamic schedule, the many-batch dynamic schedule and norm at 4 tiles per claim; then
# the ratio tables and the other-layout probes on the same build.
set -u
O=gpurun_out/r02am; mkdir -p $O
bash tools/gpu_round.sh r02am tests,bench
for f in soa_rate unaligned_rate padded_rate many_rate; do timeout 300 python tools/probe/$f.py > $O/$f.jsonl 2>&1; echo "$f rc=$?"; done
