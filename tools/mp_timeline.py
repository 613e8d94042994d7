#!/usr/bin/env python3
"""torchrun: per-rank kernel timeline of a graph-captured run (DRB_TIMELINE); rank 0 prints
per-step sel/plan/copy windows of every rank (globaltimer, per-GPU clock; relative to each
rank's own first copy start) and summary statistics."""
import os
import sys

os.environ["DRB_TIMELINE"] = "4096"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2406_03285_b200 as drb  # noqa: E402
from paper_2406_03285_b200._lib import check, lib  # noqa: E402
from paper_2406_03285_b200.workload import device_ring, stream_spec  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("gloo", init_method="env://")
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
STEPS = int(sys.argv[2]) if len(sys.argv) > 2 else 64
K, cap, S, b, r, c = cfg["K"], cfg["cap"], cfg["S"], cfg["b"], cfg["r"], cfg["c"]
spec = stream_spec(K, cfg["T"], b, S, steps_per_task=100, seed=1)
buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=1, rank=rank, world=world,
                           device=local)
blobs = [None] * world
dist.all_gather_object(blobs, buf.export_handle())
buf.connect(blobs)
eng = drb.engine(buf)
eng.start()
data, lab = device_ring(spec, rank, 16, f"cuda:{local}")
eng.run(data, lab, 450)
torch.cuda.synchronize()
first = eng.iteration
g = eng.prepare_run(data, lab, STEPS)
dist.barrier()
g.launch()
torch.cuda.synchronize()
n = C.c_uint32(0)
check(lib.drb_rb_timeline_read(buf.h, None, C.byref(n)))
W = 32 + 16 * 160  # kTlStride words per step (drb_internal.cuh)
t = np.zeros(n.value * W, np.uint64)
check(lib.drb_rb_timeline_read(buf.h, t.ctypes.data, C.byref(n)))
full = t.reshape(n.value, W).astype(np.int64)
t = full[:, :6].reshape(n.value, 3, 2)
rows = [(first + i) % n.value for i in range(STEPS)]
mine = np.stack([t[row] for row in rows])  # [STEPS, 3, 2]
allt = [None] * world
dist.all_gather_object(allt, mine)
if rank == 0:
    for w in range(world):
        m = allt[w]
        cs, ce = m[:, 2, 0], m[:, 2, 1]
        ss, se = m[:, 0, 0], m[:, 0, 1]
        ps, pe = m[:, 1, 0], m[:, 1, 1]
        print(f"rank {w}: copy period {np.median(np.diff(cs))/1e3:.2f} us, copy dur {np.median(ce-cs)/1e3:.2f}, "
              f"gap {np.median(cs[1:]-ce[:-1])/1e3:.2f}; sel dur {np.median(se-ss)/1e3:.2f} ends "
              f"{np.median(cs-se)/1e3:.2f} before copy; plan dur {np.median(pe-ps)/1e3:.2f} ends "
              f"{np.median(cs[1:]-pe[:-1])/1e3:.2f} before next copy; plan start after copy(i-1) end "
              f"{np.median(ps[1:]-ce[:-1])/1e3:.2f}")
    t0 = [allt[w][0, 2, 0] for w in range(world)]
    print("step | " + " | ".join(f"r{w} sel / plan / copy" for w in range(world)))
    for i in list(range(8)) + list(range(STEPS - 3, STEPS)):
        cells = []
        for w in range(world):
            m = allt[w][i] - t0[w]
            cells.append(" ".join(f"{m[k,0]/1e3:6.1f}-{m[k,1]/1e3:6.1f}" for k in range(3)))
        print(f"{first+i:4d} | " + " | ".join(cells))
# per-CTA copy stamps of this rank (slots as in tools/timeline.py), medians over steps
CN = {0: "start", 2: "A issued", 11: "A 1st land", 5: "A m' stored", 1: "lists", 10: "B wait", 3: "A wait+ready",
      4: "B issued", 9: "B done", 6: "A done", 7: "end"}
cta = full[:, 32:].reshape(n.value, 160, 16)
grid = int((cta[rows[8], :, 0] > 0).sum())
rel = np.array([(cta[row, :grid].astype(np.float64) - cta[row, :grid, 0].min()) / 1e3 for row in rows[8:]])
lines = [f"rank {rank} copy CTA stamps (us from first CTA start, median step, p50 / p90 over CTAs):"]
for k, nm in CN.items():
    v = np.median(rel[:, :, k], axis=0)
    lines.append(f"  {nm:12s} {np.percentile(v, 50):6.2f} {np.percentile(v, 90):6.2f}")
allc = [None] * world
dist.all_gather_object(allc, "\n".join(lines))
if rank == 0:
    print("\n".join(allc))
dist.destroy_process_group()
