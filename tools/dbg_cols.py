"""Debug: single-rank persistent run; on a slab mismatch decompose each bad slot by copy-CTA
byte column and name which historical write (oracle) each column holds.
Usage: python tools/dbg_cols.py K cap S b c r steps trials"""
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
parts = torch.cuda.get_device_properties(0).multi_processor_count - 2
c16 = S // 16
cols = [((c16 * p // parts) * 16, (c16 * (p + 1) // parts) * 16) for p in range(parts)]
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
    hist = {}
    prev = None
    # write history per slot from the oracle's per-step reports: track by content fingerprint
    fp = {rd[x, j, :16].tobytes(): (x, j) for x in range(ring) for j in range(b)}
    snap_prev = None
    for k in range(steps):
        rep.step(rd[k % ring][None], labs[k][None])
    occ, ver, slab, sl = rep.dump(0)
    g = d.cpu().numpy()
    bad = [(kk, s_) for kk in range(K) for s_ in range(occ[kk]) if not np.array_equal(g[kk, s_], slab[kk, s_])]
    print(f"trial {trial}: err {err} bad {len(bad)}", flush=True)
    if bad:
        # oracle history for the bad slots: replay again, dumping after each step (slow but exact)
        want = set(bad)
        rp2 = Backend("port").replay(1, K, cap, S, c, r, 1)
        hist = {s: [] for s in want}
        for k in range(steps):
            rp2.step(rd[k % ring][None], labs[k][None])
            o2, _, s2, _ = rp2.dump(0)
            for (kk, s_) in want:
                if s_ < o2[kk]:
                    cur = fp.get(s2[kk, s_, :16].tobytes())
                    if not hist[(kk, s_)] or hist[(kk, s_)][-1][1] != cur:
                        hist[(kk, s_)].append((k, cur))
        for (kk, s_) in bad[:4]:
            h = hist[(kk, s_)]
            desc = []
            for p, (a, e) in enumerate(cols):
                if e <= a:
                    continue
                gb = g[kk, s_, a:e]
                if np.array_equal(gb, slab[kk, s_, a:e]):
                    continue
                who = "pattern" if (gb == 0xA5).all() else None
                for (k, src) in h:
                    if src is not None and np.array_equal(gb, rd[src[0], src[1], a:e]):
                        who = f"write@{k}"
                desc.append((p, who))
            print(f"  slot ({kk},{s_}) history {h[-4:]} final {h[-1]}; bad columns {len(desc)}: {desc[:12]}", flush=True)
        break
    eng.shutdown()
    buf.close()
    del d, l, dr, lr
