# After the claim-batch change: GPU suite, smoke, bench (+ reference arm), ratio tables,
# the config-1 probe and a launch list of the bench command.
set -u
mkdir -p gpurun_out/r02u
bash tools/gpu_round.sh r02u tests,bench
timeout 300 python -m paper_1606_06508_b200 ratios --regime normal --prec double --prec single \
    --experiments 5 --rows 16777216 --json gpurun_out/r02u/ratios_normal.json > gpurun_out/r02u/ratios_normal.txt 2>&1; echo "ratios rc=$?"
timeout 600 python tools/probe/cfg1_dyn.py > gpurun_out/r02u/cfg1_dyn.txt 2>&1; echo "cfg1 rc=$?"
B="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-configs --no-default-api"
timeout 600 $B > gpurun_out/r02u/bench_plain.json 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/r02u_launches.csv $B > gpurun_out/r02u/ncu_launch.log 2>&1
echo "launch list rc=$?"
