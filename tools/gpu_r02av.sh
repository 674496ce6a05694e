# Why the default host call runs 1.0-1.1 G rows/s at 2^30 rows but 1.4-1.5 at 2^28: size
# sweep, the host's memory setup, and the two staging knobs at 2^30.
set -u
O=gpurun_out/r02av; mkdir -p $O
( echo "THP: $(cat /sys/kernel/mm/transparent_hugepage/enabled 2>/dev/null)"; echo "THP defrag: $(cat /sys/kernel/mm/transparent_hugepage/defrag 2>/dev/null)";
  echo "nodes: $(ls -d /sys/devices/system/node/node* 2>/dev/null | wc -l)"; nproc; grep -E "MemTotal|MemFree|MemAvailable|AnonHugePages|HugePages_Total" /proc/meminfo ) > $O/host.txt 2>&1
for lg in 27 28 29 30; do python tools/probe/host_default.py child $lg >> $O/sizes.jsonl 2>&1; done
for v in "FASTNORM_B200_COPY_THREADS=16" "FASTNORM_B200_HOST_CHUNK_MB=32" "FASTNORM_B200_HOST_CHUNK_MB=64" "FASTNORM_B200_HOST_PIPES=4" "FASTNORM_B200_HOST_PIPES=4 FASTNORM_B200_HOST_CHUNK_MB=32"; do
  env $v python tools/probe/host_default.py child 30 >> $O/knobs_2p30.jsonl 2>&1
done
grep -E "AnonHugePages" /proc/meminfo >> $O/host.txt
echo done
