#!/usr/bin/env python3
"""torchrun: in-kernel phase stamps (DRB_TRACE) of per-iteration launches on every rank."""
import ctypes as C
import os
import sys

os.environ["DRB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2406_03285_b200 as drb  # noqa: E402
from paper_2406_03285_b200._lib import check, lib  # noqa: E402
from paper_2406_03285_b200.workload import device_ring, stream_spec  # noqa: E402

NAMES = {14: "copy grid first start", 16: "copy start (cta0)", 20: "lists staged + peers ready",
         21: "first B chunk", 22: "first warp done", 18: "last warp done (cta0)", 19: "C done (cta0)",
         23: "last CTA of rank (done ticket)", 15: "copy grid last end"}
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("gloo", init_method="env://")
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
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
rows = []
for i in range(20):
    dist.barrier()
    eng.update((data[i % 16], lab[i % 16]))
    t = np.zeros(32, np.uint64)
    check(lib.drb_rb_trace_read(buf.h, t.ctypes.data))
    rows.append(t.astype(np.int64))
rows = np.stack(rows)
allr = [None] * world
dist.all_gather_object(allr, rows)
if rank == 0:
    for w in range(world):
        rr = allr[w]
        t0 = rr[:, 14]
        print(f"rank {w}:")
        for slot in (14, 16, 20, 21, 22, 18, 19, 23, 15):
            v = rr[:, slot] - t0
            ok = rr[:, slot] > 0
            print(f"   {NAMES[slot]:30s} median {np.median(v[ok]) / 1000 if ok.any() else float('nan'):7.2f} us")
dist.destroy_process_group()
