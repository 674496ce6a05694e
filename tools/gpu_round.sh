#!/bin/bash
# Developer tool, run under gpurun: GPU tests, bench, tile sweep, ncu (launch list of the
# bench + one full capture of the top kernel).  Usage: bash tools/gpu_round.sh TAG [parts]
set -u
OUT=gpurun_out; mkdir -p $OUT
TAG=${1:-rX}; PARTS=${2:-tests,bench,tune}
# ncu parts (one ncu run per gpurun call): ncu_launch (launch list of the bench command)
# and ncu_full (one --set full capture of the headline kernel), e.g. PARTS=ncu_launch
has() { [[ ",$PARTS," == *",$1,"* ]]; }
if has tests; then
  timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/${TAG}_pytest_gpu.log 2>&1
  echo "pytest rc=$?"; tail -3 $OUT/${TAG}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
fi
if has bench; then
  timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err; echo "bench rc=$?"
  timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/${TAG}_bench_ref.json 2>&1; echo "bench ref rc=$?"
fi
if has tune; then
  make -s -C tools tune >/dev/null 2>&1
  timeout 900 tools/tune_stream 28 10 all > $OUT/${TAG}_tune.csv 2>&1; echo "tune rc=$?"
fi
if has ncu_launch; then
  BENCH="python bench.py --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
  timeout 600 $BENCH > $OUT/${TAG}_bench_plain.log 2>&1 && \
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv \
      --log-file $OUT/${TAG}_launches.csv $BENCH > $OUT/${TAG}_ncu_launch.log 2>&1; echo "launch list rc=$?"
fi
if has ncu_full; then
  PROF="python tools/prof_target.py --cfg 5 --log2-rows 26 --iters 2"
  timeout 300 $PROF > $OUT/${TAG}_prof_plain.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:tma_stream_kernel -c 1 \
      -o $OUT/${TAG}_normalize3_f64 $PROF > $OUT/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
