for i in 1 2; do
timeout 120 python tools/cfg1_probe.py
FASTNORM_B200_PDL=0 timeout 120 python tools/cfg1_probe.py
done
