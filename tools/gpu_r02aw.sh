# Last build of the round: GPU suite + smoke + bench + reference arm.
set -u
bash tools/gpu_round.sh r02aw tests,bench
