# Why captured-dynamic loses on norm3 and config-1-sized launches: variants of the
# self-reset protocol (1: report after the store drain, 2: no fence, 4: eager self-reset).
set -u
O=gpurun_out/r02ai; mkdir -p $O
export GRAPH_DYN_ONLY=norm3,normalize3
for v in "FASTNORM_B200_DYN_CAPTURE=0" "FASTNORM_B200_DYN_CAPTURE=1" "FASTNORM_B200_DYN_CAPTURE=1 FASTNORM_B200_DYN_VARIANT=1" "FASTNORM_B200_DYN_CAPTURE=1 FASTNORM_B200_DYN_VARIANT=2" "FASTNORM_B200_DYN_CAPTURE=1 FASTNORM_B200_DYN_VARIANT=3" "FASTNORM_B200_DYN_CAPTURE=1 FASTNORM_B200_PDL=0" "FASTNORM_B200_DYN_CAPTURE=0 FASTNORM_B200_PDL=0"; do
  echo "== $v" >> $O/graph_variants.txt
  env $v timeout 300 python tools/probe/graph_dyn.py >> $O/graph_variants.txt 2>&1
done
L=paper_1606_06508_b200/libfastnorm_b200.so
python tools/ab_lib.py $L@FASTNORM_B200_DYN_VARIANT=0 $L@FASTNORM_B200_DYN_VARIANT=4 $L@FASTNORM_B200_DYN_VARIANT=5 $L@FASTNORM_B200_DYN_VARIANT=6 $L@FASTNORM_B200_DYN=0 --op 2 --dim 3 --cfg 5 --log2-rows 28 --reps 10 --rounds 2 > $O/eager_norm3.txt 2>&1
python tools/ab_lib.py $L@FASTNORM_B200_DYN_VARIANT=0 $L@FASTNORM_B200_DYN_VARIANT=4 $L@FASTNORM_B200_DYN_VARIANT=5 $L@FASTNORM_B200_DYN=0 --op 1 --dim 3 --cfg 1 --log2-rows 20 --reps 50 --rounds 2 > $O/eager_cfg1.txt 2>&1
echo done
