# Config-1 launch-shape sweep (lone launch after an L2 flush, and stream of batches)
timeout 120 python tools/cfg1_probe.py
for c in 1 2 3 4 8; do FASTNORM_B200_CTAS_PER_SM=$c timeout 120 python tools/cfg1_probe.py; done
FASTNORM_B200_PATH=direct timeout 120 python tools/cfg1_probe.py
