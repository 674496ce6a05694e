# Round-2 re-entry run: GPU suite + smoke + bench (gpu_round.sh), the dynamic-schedule
# A/B on the batched-claim build, the issue-roofline ncu passes, and one --set full
# capture of the headline kernel at the bench size (2^30 rows).
set -u
mkdir -p gpurun_out/r02j
bash tools/gpu_round.sh r02j tests,bench
timeout 1500 bash tools/ab_dyn.sh > gpurun_out/r02j/ab_dyn.txt 2>&1; echo "ab rc=$?"
timeout 600 python tools/probe/cfg1_dyn.py > gpurun_out/r02j/cfg1_dyn.txt 2>&1; echo "cfg1 rc=$?"
timeout 2400 bash tools/ncu_issue.sh r02j 2>&1 | tail -10
P="python tools/prof_target.py --cfg 5 --log2-rows 30 --iters 1 --op normalize"
timeout 300 $P > gpurun_out/r02j/prof_plain.log 2>&1 && \
  timeout 1800 ncu --set full --clock-control none --import-source on --replay-mode application \
    -k regex:tma_stream_kernel -c 1 -o gpurun_out/r02j_normalize3_f64_2p30 $P > gpurun_out/r02j/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/r02j/ncu_full.log
B="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-configs --no-default-api"
timeout 600 $B > gpurun_out/r02j/bench_plain.json 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/r02j_launches.csv $B > gpurun_out/r02j/ncu_launch.log 2>&1
echo "launch list rc=$?"
