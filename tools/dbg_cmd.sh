for t in 1 2; do timeout 300 python bench.py --steps 2000 --no-cpu > gpurun_out/e2e_$t.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/e2e_$t.json').read().strip().splitlines()[-1]);print('persist', d['e2e']['value'], d['e2e']['pcie_ceiling']['value'])"; done
for t in 1 2; do DRB_PERSIST=0 timeout 300 python bench.py --steps 2000 --no-cpu > gpurun_out/e2e_p0_$t.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/e2e_p0_$t.json').read().strip().splitlines()[-1]);print('3-kernel', d['e2e']['value'], d['e2e']['pcie_ceiling']['value'])"; done
for t in 1 2; do timeout 300 python bench.py --steps 2000 --no-cpu --e2e-steps 1000 > gpurun_out/e2e_l_$t.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/e2e_l_$t.json').read().strip().splitlines()[-1]);print('persist 1000 e2e steps', d['e2e']['value'], d['e2e']['pcie_ceiling']['value'])"; done
