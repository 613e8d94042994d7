#!/bin/bash
# ncu evidence for the round (run on the GPU box, one GPU, after bench.py exited 0 without ncu):
#   1. launch list (per-kernel gpu__time_duration, cold & serialised) of a short bench run
#   2. one full capture of the persistent run kernel (the timed region's only launch;
#      source-level, raw metrics for DRAM bytes), and of the three-kernel path's copy kernel
set -e
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
R=${1:-r03}
STEPS=${STEPS:-200}
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/ncu_launches_$R.csv python bench.py --steps $STEPS --warmup 5 --no-cpu --e2e-steps 10 \
    > gpurun_out/ncu_launches_$R.log 2>&1
# bench.py launches drb_run_kernel for the prefill (7 runs), the warm-up (1), then the timed run
ncu --set full --import-source on --clock-control none -k regex:drb_run_kernel --launch-skip 8 -c 1 \
    -o gpurun_out/ncu_run_$R -f python bench.py --steps $STEPS --warmup 5 --no-cpu --e2e-steps 10 \
    > gpurun_out/ncu_run_$R.log 2>&1
DRB_PERSIST=0 ncu --set full --import-source on --clock-control none -k regex:drb_copy_tma_kernel --launch-skip 300 -c 1 \
    -o gpurun_out/ncu_copy_$R -f python bench.py --steps 60 --warmup 5 --no-cpu --e2e-steps 10 \
    > gpurun_out/ncu_copy_$R.log 2>&1
echo profile done
