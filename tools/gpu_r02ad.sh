# Re-entry run on the rebuilt tree (same sources as r02ab): GPU suite + smoke + bench +
# reference arm, then the exponent-insertion A/B of tools/gpu_r02ac.sh on the current geometry.
set -u
mkdir -p gpurun_out/r02ad
bash tools/gpu_round.sh r02ad tests,bench
bash tools/gpu_r02ac.sh
