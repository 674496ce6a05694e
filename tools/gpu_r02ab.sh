# Re-entry run on the final big-tile build: GPU suite + smoke + bench + reference arm,
# the launch list of the bench command, and one --set full capture of the headline
# kernel at the bench size (2^30 rows) so roofline.traffic comes from this build.
set -u
mkdir -p gpurun_out/r02ab
bash tools/gpu_round.sh r02ab tests,bench
P="python tools/prof_target.py --cfg 5 --log2-rows 30 --iters 1 --op normalize"
timeout 300 $P > gpurun_out/r02ab/prof_plain.log 2>&1 && \
  timeout 1800 ncu --set full --clock-control none --import-source on --replay-mode application \
    -k regex:tma_stream_kernel -c 1 -o gpurun_out/r02ab_normalize3_f64_2p30 $P > gpurun_out/r02ab/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/r02ab/ncu_full.log
B="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-configs --no-default-api"
timeout 600 $B > gpurun_out/r02ab/bench_plain.json 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/r02ab_launches.csv $B > gpurun_out/r02ab/ncu_launch.log 2>&1
echo "launch list rc=$?"
