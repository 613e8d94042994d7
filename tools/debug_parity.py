import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2406_03285_b200 as drb
from oracle.py_oracle import Backend
from paper_2406_03285_b200.workload import stream_spec
K, cap, S, b, c, r = [int(x) for x in sys.argv[1:7]]
seed = K + cap
buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=seed)
eng = drb.engine(buf); eng.start()
rep = Backend("port").replay(1, K, cap, S, c, r, seed)
spec = stream_spec(K, 1, b, S, steps_per_task=10**9, seed=seed)
prev_slab = None; prev_plan = None
def find(slab, occ, row):
    return [(kk, s) for kk in range(K) for s in range(occ[kk]) if np.array_equal(slab[kk, s], row)]
for i in range(4):
    lab = spec.labels(0, i); data = spec.payload(0, i)
    o, ol, oc = rep.step(data[None], lab[None])
    aug = eng.update((torch.from_numpy(data).cuda(), torch.from_numpy(lab.astype(np.int32)).cuda()))
    d, l = aug.tensors(); d = d.cpu().numpy()
    occ, ver, slab, sl = rep.dump(0)
    bad_rows = [j for j in range(aug.count()) if not np.array_equal(d[j], o[0, j])]
    print(f"step {i}: bad rows {bad_rows}")
    for j in bad_rows[:6]:
        if j >= b and prev_slab is not None:
            pe = prev_plan[j - b]
            print(f"   row {j}: oracle plan entry {pe.tolist()}; oracle row at prev slot {find(prev_slab, prev_occ, o[0, j])}; gpu row at prev slot {find(prev_slab, prev_occ, d[j])}; gpu row == batch row {[x for x in range(b) if np.array_equal(data[x], d[j])]}")
            nz = np.nonzero(d[j] != o[0, j])[0]
            print(f"      differing bytes {nz[:8]}...{nz[-4:]} count {len(nz)}")
    prev_slab, prev_occ, prev_plan = slab.copy(), occ.copy(), rep.last_plan(0)
