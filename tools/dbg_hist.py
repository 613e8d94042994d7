"""Debug: repeat a single-rank persistent run (gc.collect between trials) and, on a slab
mismatch, print the write history of the bad slots (oracle) and where the GPU bytes came from.
Usage: python tools/dbg_hist.py K cap S b c r steps trials"""
import gc, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2406_03285_b200 as drb
from oracle.py_oracle import Backend
from paper_2406_03285_b200.workload import stream_spec
K, cap, S, b, c, r, steps, trials = [int(x) for x in sys.argv[1:9]]
ring = 6
spec = stream_spec(K, 1, b, S, steps_per_task=steps, seed=1)
rd = np.stack([spec.payload(0, x) for x in range(ring)])
labs = np.stack([spec.labels(0, k) for k in range(steps)])
# fingerprint of each ring row (first 16 bytes) -> (ring slot, row)
fp = {rd[x, j, :16].tobytes(): (x, j) for x in range(ring) for j in range(b)}
for trial in range(trials):
    gc.collect()
    buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=1)
    d, l = buf.slab()
    d.fill_(0xA5)
    torch.cuda.synchronize()
    eng = drb.engine(buf)
    eng.start()
    dr = torch.from_numpy(rd).cuda()[torch.arange(steps, device="cuda") % ring]
    lr = torch.from_numpy(labs.astype(np.int32)).cuda()
    eng.run(dr, lr, steps, first=0)
    torch.cuda.synchronize()
    err = eng.device_error()
    rep = Backend("port").replay(1, K, cap, S, c, r, 1)
    for k in range(steps):
        rep.step(rd[k % ring][None], labs[k][None])
    occ, ver, slab, sl = rep.dump(0)
    g = d.cpu().numpy()
    bad = [(k, s_) for k in range(K) for s_ in range(occ[k]) if not np.array_equal(g[k, s_], slab[k, s_])]
    print(f"trial {trial}: err {err} bad {len(bad)}", flush=True)
    if bad:
        for (k, s_) in bad[:3]:
            gsrc = fp.get(g[k, s_, :16].tobytes(), "pattern" if (g[k, s_] == 0xA5).all() else "?")
            osrc = fp.get(slab[k, s_, :16].tobytes())
            ncol = int((g[k, s_].reshape(-1, 16) != slab[k, s_].reshape(-1, 16)).any(1).sum())
            print(f"  slot ({k},{s_}): gpu bytes from ring {gsrc}, oracle from ring {osrc}, "
                  f"{ncol} of {S // 16} 16B units differ", flush=True)
            # history: replay again, record content after each step
            rp2 = Backend("port").replay(1, K, cap, S, c, r, 1)
            hist, last = [], None
            for kk in range(steps):
                rp2.step(rd[kk % ring][None], labs[kk][None])
                o2, _, s2, _ = rp2.dump(0)
                cur = fp.get(s2[k, s_, :16].tobytes()) if s_ < o2[k] else None
                if cur != last:
                    hist.append((kk, cur))
                    last = cur
            print(f"    oracle history (step, ring src): {hist}", flush=True)
        break
    eng.shutdown()
    buf.close()
    del d, l, dr, lr
