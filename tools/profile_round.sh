#!/bin/bash
# ncu evidence for the round (run on the GPU box, one GPU, after bench.py exited 0 without ncu):
#   1. launch list (per-kernel gpu__time_duration, cold & serialised) of the driver's bench command
#   2. one full capture of the resident engine instance that runs a 200-step c2 run
#      (tools/ncu_run.py: instance 2), source-level, raw metrics for DRAM bytes
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
R=${1:-r2}
BENCH_NO_CPP=1 ncu --target-processes application-only --metrics gpu__time_duration.sum --clock-control none \
    -c 4000 --csv --log-file gpurun_out/ncu_launches_$R.csv python bench.py --steps 20 --warmup 5 --no-cpu --e2e-steps 10 \
    > gpurun_out/ncu_launches_$R.log 2>&1
echo "launch list rc $?"
ncu --set full --import-source on --clock-control none -k regex:drb_run_kernel --launch-skip 1 -c 1 \
    -o gpurun_out/ncu_run_$R -f python tools/ncu_run.py 200 > gpurun_out/ncu_run_$R.log 2>&1
echo "full capture rc $?"
ncu -i gpurun_out/ncu_run_$R.ncu-rep --page raw --csv > gpurun_out/ncu_run_${R}_raw.csv 2>/dev/null
ncu -i gpurun_out/ncu_run_$R.ncu-rep --page details --csv > gpurun_out/ncu_run_${R}_details.csv 2>/dev/null
echo profile done
