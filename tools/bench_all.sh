#!/bin/bash
# Bench lines at N = 1 2 4 (one process per GPU), optional DRB_DBG variants: bench_all.sh "<dbg values>"
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
port=29600
for d in ${1:-0}; do
  for n in ${NS:-1 2 4}; do
    port=$((port + 1))
    out=gpurun_out/bench_d${d}_n${n}.json
    DRB_DBG=$d timeout 300 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $port \
      --nproc-per-node $n bench.py --gpus $n --steps ${STEPS:-20000} ${EXTRA:---no-cpu} > $out 2> ${out%.json}.err
    python - "$out" "$d" "$n" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"dbg {sys.argv[2]} N={sys.argv[3]}: {d['ms_per_step']*1e3:.3f} us/step  value {d['value']/1e6:.2f} M/s  "
          f"frac {d['roofline']['frac']:.3f}  e2e {d['e2e']['value']/1e3:.0f} K/s  clocks {d['clocks']}")
except Exception as e:
    print(f"dbg {sys.argv[2]} N={sys.argv[3]}: FAILED {e}")
PY
  done
done
