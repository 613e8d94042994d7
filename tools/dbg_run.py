"""Debug helper: graph-captured three-kernel run parity, report mismatching rows."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_03285_b200 as drb
from oracle.py_oracle import Backend
from paper_2406_03285_b200.workload import stream_spec
K, cap, S, b, c, r, seed, ring = 10, 6, 64, 24, 14, 7, 8, 6
graph = sys.argv[1] == "graph"
buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=seed)
eng = drb.engine(buf); eng.start()
rep = Backend("port").replay(1, K, cap, S, c, r, seed)
spec = stream_spec(K, 2, b, S, steps_per_task=7, seed=seed)
def dev(d, l): return torch.from_numpy(np.ascontiguousarray(d)).cuda(), torch.from_numpy(np.ascontiguousarray(l).astype(np.int32)).cuda()
def step(i, tag):
    d_, l_ = spec.payload(0, i), spec.labels(0, i)
    o, ol, oc = rep.step(d_[None], l_[None])
    aug = eng.update(dev(d_, l_)); d, l = aug.tensors(); cnt = aug.count()
    d = d.cpu().numpy()
    bad = [j for j in range(cnt) if not np.array_equal(d[j], o[0, j])]
    print(tag, i, "count", cnt, int(oc[0]), "bad rows", bad)
i = 0
for _ in range(2): step(i, "pre"); i += 1
for run_no, (steps, first) in enumerate([(25, 1), (7, 0)]):
    rd = np.stack([spec.payload(0, 1000 * (run_no + 1) + x) for x in range(ring)])
    rl = np.stack([spec.labels(0, 1000 * (run_no + 1) + x) for x in range(ring)])
    dr, lr = dev(rd, rl)
    if graph:
        g = eng.prepare_run(dr, lr, steps, first=first); g.launch()
    else:
        eng.run(dr, lr, steps, first=first)
    for k in range(steps): rep.step(rd[(first + k) % ring][None], rl[(first + k) % ring][None])
    torch.cuda.synchronize()
    for _ in range(3): step(i, f"post{run_no}"); i += 1
