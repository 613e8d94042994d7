"""Debug: find the first run length whose slab diverges from the oracle (slab pre-filled with
0xA5 so a lost write is visible). Usage: python tools/dbg_slab.py K cap S b c r T maxsteps"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2406_03285_b200 as drb
from oracle.py_oracle import Backend
from paper_2406_03285_b200.workload import stream_spec
K, cap, S, b, c, r, T, maxsteps = [int(x) for x in sys.argv[1:9]]
ring = 6
spec = stream_spec(K, T, b, S, steps_per_task=max(1, maxsteps // T), seed=1)
rd = np.stack([spec.payload(0, x) for x in range(ring)])
labs = np.stack([spec.labels(0, k) for k in range(maxsteps)])
dring = torch.from_numpy(rd).cuda()
idx = torch.arange(maxsteps, device="cuda") % ring
data = dring[idx]
lab = torch.from_numpy(labs.astype(np.int32)).cuda()
for steps in range(1, maxsteps + 1):
    buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=1)
    d, l = buf.slab()
    d.fill_(0xA5)
    torch.cuda.synchronize()
    eng = drb.engine(buf)
    eng.start()
    eng.run(data[:steps], lab[:steps], steps, first=0)
    torch.cuda.synchronize()
    err = eng.device_error()
    rep = Backend("port").replay(1, K, cap, S, c, r, 1)
    for k in range(steps):
        rep.step(rd[k % ring][None], labs[k][None])
    occ, ver, slab, sl = rep.dump(0)
    g = d.cpu().numpy()
    bad = []
    for k in range(K):
        for s_ in range(occ[k]):
            if not np.array_equal(g[k, s_], slab[k, s_]):
                src = [j for j in range(b) if np.array_equal(rd[(steps - 1) % ring][j], slab[k, s_])]
                gsrc = [(kk, j) for kk in range(max(0, steps - 3), steps) for j in range(b)
                        if np.array_equal(rd[kk % ring][j], g[k, s_])]
                frac = float((g[k, s_] != slab[k, s_]).mean())
                bad.append((k, s_, "pattern" if (g[k, s_] == 0xA5).all() else "data", f"diff {frac:.3f}",
                            "oracle=batch row", src, "gpu=(step,row)", gsrc[:3]))
    print(f"steps {steps}: err {err} mismatches {len(bad)}", bad[:6], flush=True)
    eng.shutdown()
    buf.close()
    if bad:
        break
