#!/bin/bash
# Same-box A/B of library builds: ab_bench.sh "<lib paths>" (NS, DBGS env)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
port=29800
for rep in 1 2; do
for n in ${NS:-1}; do
for lib in $1; do
for d in ${DBGS:-0}; do
  port=$((port + 1))
  out=gpurun_out/ab_$(basename $lib .so)_d${d}_n${n}.json
  DRB_LIB=$(realpath $lib) DRB_DBG=$d timeout 300 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 \
    --master-port $port --nproc-per-node $n bench.py --gpus $n --steps ${STEPS:-20000} --no-cpu --e2e-steps 20 > $out 2> ${out%.json}.err
  python - "$out" "$lib" "$n" "$d" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"{sys.argv[2]:40s} dbg {sys.argv[4]:6s} N={sys.argv[3]}: {d['ms_per_step']*1e3:.3f} us/step frac {d['roofline']['frac']:.3f}")
except Exception as e:
    print(f"{sys.argv[2]} N={sys.argv[3]}: FAILED {e}")
PY
done; done; done; done
