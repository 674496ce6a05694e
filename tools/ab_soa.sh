# SoA bulk-copy kernel geometry variants (run bytes per array, stages, CTAs per SM)
for v in 2048_3_2 4096_3_2 4096_4_2 8192_3_2 4096_3_3 2048_4_4; do
  FASTNORM_B200_LIB=tools/ab/lib_soa_$v.so timeout 200 python tools/probe/soa_rate.py | python3 -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('$v', d['kernel'], round(d['GB_per_s']), round(d['frac'], 3))"
done
