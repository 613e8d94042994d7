#!/bin/bash
# ncu evidence for the round (run on the GPU box, one GPU, after bench.py exited 0 without ncu):
#   1. launch list (per-kernel gpu__time_duration, cold & serialised) of a short bench run,
#      past the prefill so the steady state is captured
#   2. one full capture of the copy kernel (source-level, raw metrics for DRAM bytes)
set -e
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
R=${1:-r02}
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 1500 -c 300 --csv \
    --log-file gpurun_out/ncu_launches_$R.csv python bench.py --steps 60 --warmup 5 --no-cpu --e2e-steps 10 \
    > gpurun_out/ncu_launches_$R.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:drb_copy_tma_kernel --launch-skip 300 -c 1 \
    -o gpurun_out/ncu_copy_$R -f python bench.py --steps 60 --warmup 5 --no-cpu --e2e-steps 10 \
    > gpurun_out/ncu_copy_$R.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:drb_sel_kernel --launch-skip 500 -c 1 \
    -o gpurun_out/ncu_sel_$R -f python bench.py --steps 60 --warmup 5 --no-cpu --e2e-steps 10 \
    > gpurun_out/ncu_sel_$R.log 2>&1
echo profile done
