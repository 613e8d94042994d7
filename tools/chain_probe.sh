#!/bin/bash
# Which latency chain binds the resident engine's steady state (tools/, GPU box, one GPU):
# builds the product library with ~1 us of delay added per iteration to one chain
# (-DDRB_DELAY=1 sel, 2 plan, 3 B engines, 4 arrivals) and times a 2000-step c2 run with each;
# the chain whose delay moves the step time is the bound.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p tools/ablib gpurun_out
SRC="paper_2406_03285_b200/csrc/drb_kernels.cu paper_2406_03285_b200/csrc/drb_capi.cu paper_2406_03285_b200/csrc/drb_dataset.cu"
for d in 0 1 2 3 4; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared \
    -DDRB_DELAY=$d -o tools/ablib/libdrb_delay$d.so $SRC || exit 1
done
for rep in 1 2; do
  for d in 0 1 2 3 4; do
    echo -n "delay chain $d: "
    DRB_LIB=tools/ablib/libdrb_delay$d.so DRB_IDLE_US=100 python tools/ncu_run.py ${STEPS:-2000} 2>&1 | tail -1
  done
done
