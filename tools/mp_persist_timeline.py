#!/usr/bin/env python3
"""torchrun: per-rank loop periods of the persistent run kernel's roles (DRB_TIMELINE) —
sel CTA, plan CTA, and the copy CTAs' B starts — to find the chain that bounds a
multi-rank step. Usage: torchrun --nproc-per-node N tools/mp_persist_timeline.py [config] [steps]"""
import os
import sys

os.environ["DRB_TIMELINE"] = "1024"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2406_03285_b200 as drb  # noqa: E402
from paper_2406_03285_b200._lib import check, lib  # noqa: E402
from paper_2406_03285_b200.dist import connect_world  # noqa: E402
from paper_2406_03285_b200.workload import device_ring, stream_spec  # noqa: E402

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("gloo", init_method="env://")
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
STEPS = int(sys.argv[2]) if len(sys.argv) > 2 else 200
K, cap, S, b, r, c = cfg["K"], cfg["cap"], cfg["S"], cfg["b"], cfg["r"], cfg["c"]
spec = stream_spec(K, cfg["T"], b, S, steps_per_task=100, seed=1)
buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=1, rank=rank, world=world,
                           device=local)
if world > 1:
    connect_world(buf)
eng = drb.engine(buf)
eng.start()
data, lab = device_ring(spec, rank, 16, f"cuda:{local}")
eng.run(data, lab, 450)
torch.cuda.synchronize()
dist.barrier()
first = eng.iteration
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
eng.run(data, lab, STEPS)
ev1.record()
torch.cuda.synchronize()
us = ev0.elapsed_time(ev1) * 1e3 / STEPS
n = C.c_uint32(0)
check(lib.drb_rb_timeline_read(buf.h, None, C.byref(n)))
W = 32 + 16 * 160
t = np.zeros(n.value * W, np.uint64)
check(lib.drb_rb_timeline_read(buf.h, t.ctypes.data, C.byref(n)))
t = t.reshape(n.value, W).astype(np.int64)
rows = [(first + i) % n.value for i in range(STEPS)][8:-2]
cta = t[:, 32:].reshape(n.value, 160, 16)
ncta = torch.cuda.get_device_properties(local).multi_processor_count


def per(vals):
    return np.median(np.diff(vals)) / 1e3


out = [f"rank {rank}: {us:.2f} us/step"]
for cidx, nm, slots in ((0, "sel", (1, 2, 3, 4)), (1, "plan", (1, 3))):
    rel = {s_: np.median([(cta[row, cidx, s_] - cta[row, cidx, 0]) / 1e3 for row in rows]) for s_ in slots}
    out.append(f"  {nm} CTA loop period {per([cta[row, cidx, 0] for row in rows]):.2f} us; "
               + ", ".join(f"stamp{s_} +{v:.2f}" for s_, v in rel.items()))
bs = [np.median(cta[row, 2:ncta, 0]) for row in rows]
out.append(f"  B start period {per(bs):.2f} us; B iter (start->end) "
           f"{np.median([np.median(cta[row, 2:ncta, 9] - cta[row, 2:ncta, 0]) for row in rows]) / 1e3:.2f} us")
NAMES = {1: "lists parsed", 10: "W published", 11: "W(k-1) seen", 12: "addresses", 3: "B loads issued",
         6: "B loads landed", 4: "B stores issued", 9: "B iter end"}
out.append("  B stamps after B start: " + ", ".join(
    f"{nm} {np.nanmedian([np.median(cta[row, 2:ncta, s_] - cta[row, 2:ncta, 0]) for row in rows]) / 1e3:.2f}"
    for s_, nm in NAMES.items()))
sel_start = [cta[row, 0, 0] for row in rows]
plan_start = [cta[row, 1, 0] for row in rows]
out.append(f"  lead: sel start - B start {np.median(np.array(sel_start) - np.array(bs)) / 1e3:.2f} us, "
           f"plan start - B start {np.median(np.array(plan_start) - np.array(bs)) / 1e3:.2f} us")
ph = t[:, 8:32]


def phase(a, e):
    return np.median([(ph[row, e] - ph[row, a]) / 1e3 for row in rows])


out.append(f"  sel_core phases: select {phase(1, 2):.2f}, assign {phase(2, 3):.2f}, W/state/publish {phase(3, 4):.2f} us")
out.append(f"  plan phases: rendezvous {phase(5, 6):.2f}, draws+locate {phase(6, 7):.2f}, push list {phase(7, 8):.2f} us")
allout = [None] * world
dist.all_gather_object(allout, "\n".join(out))
if rank == 0:
    print("\n".join(allout), flush=True)
eng.shutdown()
dist.destroy_process_group()
