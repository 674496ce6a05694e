# norm3 eager on the current build: tiles per claim sweep (is the slow mode bound by the
# counter's same-address atomic rate?)
set -u
O=gpurun_out/r02ak; mkdir -p $O
L=paper_1606_06508_b200/libfastnorm_b200.so
for lg in 26 28; do
python tools/ab_lib.py $L@FASTNORM_B200_SCHED_BATCH=1 $L@FASTNORM_B200_SCHED_BATCH=2 $L@FASTNORM_B200_SCHED_BATCH=4 $L@FASTNORM_B200_SCHED_BATCH=8 $L@FASTNORM_B200_SCHED_BATCH=16 $L@FASTNORM_B200_SCHED_BATCH=32 $L@FASTNORM_B200_DYN=0 --op 2 --dim 3 --cfg 5 --log2-rows $lg --reps 10 --rounds 2 >> $O/norm3_batch.txt 2>&1
done
export GRAPH_DYN_ONLY=norm3
for b in 2 8 16; do
  echo "== batch $b" >> $O/graph_norm3.txt
  FASTNORM_B200_SCHED_BATCH=$b timeout 200 python tools/probe/graph_dyn.py >> $O/graph_norm3.txt 2>&1
done
echo done
