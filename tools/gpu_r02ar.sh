# Final-build ncu evidence: one --set full capture of the headline kernel at the bench size
# (2^30 rows), one of normalize3 f32 on config 4 (new geometry), one of norm3 f64 (4 tiles
# per claim), and the launch list of the bench command.  Each capture follows a plain run
# of the same command that exited 0.  Reports are summarised on the box (tools/ncu_summary.py);
# only the headline report travels back (gpurun_out is capped at 64 MiB).
set -u
O=gpurun_out/r02ar; mkdir -p $O /tmp/r02ar_reps
cap() {  # name, rows, algorithmic bytes per row, prof_target args
  local name=$1 rows=$2 bpr=$3; shift 3
  local P="python tools/prof_target.py --iters 1 $*"
  timeout 300 $P > $O/${name}_plain.log 2>&1 && \
    timeout 1800 ncu --set full --clock-control none --import-source on --replay-mode application \
      -k regex:tma_stream_kernel -c 1 -o /tmp/r02ar_reps/r02ar_$name $P > $O/${name}_ncu.log 2>&1
  echo "$name rc=$?"
  python tools/ncu_summary.py /tmp/r02ar_reps/r02ar_$name.ncu-rep $rows --key $name --algo-bytes-per-row $bpr > $O/${name}_summary.txt 2>&1
  ls -la /tmp/r02ar_reps/r02ar_$name.ncu-rep >> $O/sizes.txt
}
cap normalize3_f64_2p30 1073741824 56 --cfg 5 --log2-rows 30 --op normalize
cap normalize3_f32_cfg4 268435456 28 --cfg 4 --log2-rows 28 --op normalize
cap norm3_f64_cfg5 268435456 32 --cfg 5 --log2-rows 28 --op norm
sz=$(stat -c %s /tmp/r02ar_reps/r02ar_normalize3_f64_2p30.ncu-rep 2>/dev/null || echo 0)
if [ "$sz" -gt 0 ] && [ "$sz" -lt 40000000 ]; then cp /tmp/r02ar_reps/r02ar_normalize3_f64_2p30.ncu-rep gpurun_out/; fi
B="python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-configs --no-default-api"
timeout 600 $B > $O/bench_plain.json 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/r02ar_launches.csv $B > $O/ncu_launch.log 2>&1
echo "launch list rc=$?"
du -sh gpurun_out
