# Other row layouts and call shapes on the last build of the round.
set -u
O=gpurun_out/r02ax; mkdir -p $O
for f in padded_rate unaligned_rate soa_rate soa_columns_rate soa_misaligned_rate many_rate; do timeout 300 python tools/probe/$f.py > $O/$f.jsonl 2>&1; echo "$f rc=$?"; done
timeout 300 python tools/probe/sharded_rate.py --log2-rows 30 --reps 5 > $O/sharded_rate.jsonl 2>&1
timeout 300 python tools/probe/graph_dyn.py > $O/graph_dyn.jsonl 2>&1
