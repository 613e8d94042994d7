#!/bin/bash
# Persistent-run grid sweep (DRB_GRID) at N=1 and N=2: us/step per grid size.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
show() { tail -1 "$1" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['ms_per_step']*1e3,3), 'us frac', round(d['roofline']['frac'],3))"; }
for g in ${GRIDS:-148 112 76}; do
  DRB_GRID=$g timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 2981$((g % 10)) bench.py --gpus 2 --no-cpu > gpurun_out/sweep_n2_$g.json 2>/dev/null
  show gpurun_out/sweep_n2_$g.json "N=2 grid $g"
  DRB_GRID=$g timeout 200 python bench.py --no-cpu > gpurun_out/sweep_n1_$g.json 2>/dev/null
  show gpurun_out/sweep_n1_$g.json "N=1 grid $g"
done
