#!/bin/bash
# Round evidence on a 4-GPU box: GPU tests, bench lines N=1/2/4 (+ reference arm), ncu profiles.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
R=${1:-r04}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_$R.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_$R.log
timeout 300 python bench.py > gpurun_out/bench_${R}_n1.json 2> gpurun_out/bench_${R}_n1.err; echo "bench n1 rc=$?"
timeout 300 python bench.py --impl reference > gpurun_out/bench_${R}_ref_n1.json 2>&1; echo "ref n1 rc=$?"
for n in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 2990$n --nproc-per-node $n \
    bench.py --gpus $n > gpurun_out/bench_${R}_n$n.json 2> gpurun_out/bench_${R}_n$n.err; echo "bench n$n rc=$?"
done
for f in gpurun_out/bench_${R}_n1.json gpurun_out/bench_${R}_n2.json gpurun_out/bench_${R}_n4.json gpurun_out/bench_${R}_ref_n1.json; do
  python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
if d.get("impl") == "reference":
    print(f"{sys.argv[1]}: reference {d['value']:.0f} aug/s cores {d['cpu_baseline']['cores']}")
else:
    print(f"{sys.argv[1]}: {d['ms_per_step']*1e3:.3f} us/step value {d['value']/1e6:.2f} M/s frac {d['roofline']['frac']:.3f} "
          f"e2e {d['e2e']['value']/1e3:.0f} K/s cpu {d['cpu_baseline'] and d['cpu_baseline']['value']}")
PY
done
timeout 1500 bash tools/profile_round.sh $R; echo "profile rc=$?"
