#!/bin/bash
# Device-gather knob sweep (DRB_GATHER="unroll,ctas_per_sm") at the c2 batch; parity of each variant.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for k in 4,4 2,4 8,4 4,2 4,8 8,2 2,8 8,8; do
  echo "$k $(DRB_GATHER=$k timeout 120 python tools/input_bench.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['gather']; print(d['us_per_gather'], 'us', d['GB_per_s'], 'GB/s')")"
done
for k in 2,4 8,8; do DRB_GATHER=$k timeout 300 python -m pytest tests/test_gpu_input.py -q 2>&1 | tail -1; done
