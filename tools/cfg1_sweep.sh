for c in 1 2 3 4 8; do FASTNORM_B200_CTAS_PER_SM=$c timeout 120 python tools/bench_configs.py --configs 1 --reps 20 | sed "s/^/cps=$c /"; done
timeout 120 python tools/bench_configs.py --configs 1 --reps 20 | sed "s/^/auto /"
