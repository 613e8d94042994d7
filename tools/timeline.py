#!/usr/bin/env python3
"""Kernel timeline of a graph-captured multi-step run (DRB_TIMELINE): per step, start/end of
sel / plan / copy relative to the first copy start. Usage: python tools/timeline.py [config] [steps]"""
import ctypes as C
import os
import sys

STEPS = int(sys.argv[2]) if len(sys.argv) > 2 else 64
os.environ["DRB_TIMELINE"] = str(1024)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2406_03285_b200 as drb  # noqa: E402
from paper_2406_03285_b200._lib import check, lib  # noqa: E402
from paper_2406_03285_b200.workload import device_ring, stream_spec  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
K, cap, S, b, r, c = cfg["K"], cfg["cap"], cfg["S"], cfg["b"], cfg["r"], cfg["c"]
spec = stream_spec(K, cfg["T"], b, S, steps_per_task=100, seed=1)
buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=1)
eng = drb.engine(buf)
eng.start()
data, lab = device_ring(spec, 0, 16, "cuda:0")
eng.run(data, lab, 450)
torch.cuda.synchronize()
first = eng.iteration
g = eng.prepare_run(data, lab, STEPS)
g.launch()
torch.cuda.synchronize()
n = C.c_uint32(0)
check(lib.drb_rb_timeline_read(buf.h, None, C.byref(n)))
W = 32 + 16 * 160
t = np.zeros(n.value * W, np.uint64)
check(lib.drb_rb_timeline_read(buf.h, t.ctypes.data, C.byref(n)))
t = t.reshape(n.value, W).astype(np.int64)
ph = t[:, 8:32]
cta = t[:, 32:].reshape(n.value, 160, 16)
t = t[:, :6].reshape(n.value, 3, 2)
rows = [(first + i) % n.value for i in range(STEPS)]
t0 = t[rows[0], 2, 0]
print(f"{'step':>5} {'sel':>17} {'plan':>17} {'copy':>17}  (us from first copy start)")
for i, row in enumerate(rows[:24] + rows[-4:]):
    cells = []
    for k in range(3):
        a, e = t[row, k]
        cells.append(f"{(a - t0) / 1e3:7.2f}-{(e - t0) / 1e3:7.2f}" if e > 0 else f"{'-':>15}")
    print(f"{first + rows.index(row) if row in rows else row:5d} " + " ".join(f"{x:>17}" for x in cells))
cs = np.array([t[row, 2, 0] for row in rows])
ce = np.array([t[row, 2, 1] for row in rows])
print(f"copy period median {np.median(np.diff(cs)) / 1e3:.2f} us, copy duration median {np.median(ce - cs) / 1e3:.2f} us, "
      f"gap copy(i) end -> copy(i+1) start median {np.median(cs[1:] - ce[:-1]) / 1e3:.2f} us")
for k, name in ((0, "sel"), (1, "plan")):
    s_ = np.array([t[row, k, 0] for row in rows]); e_ = np.array([t[row, k, 1] for row in rows])
    print(f"{name}: duration median {np.median(e_ - s_) / 1e3:.2f} us; start after copy(i-1) end median "
          f"{np.median(s_[1:] - ce[:-1]) / 1e3:.2f} us; end before copy(i) start median {np.median(cs - e_) / 1e3:.2f} us")

# phase stamps (CTA 0; trace slot s -> timeline word 8+s), medians relative to kernel start
PH = {"sel": [0, 1, 2, 3, 4], "plan": [5, 6, 7, 8], "copy(cta0)": [16, 20, 19]}
NM = {0: "start", 1: "loads", 2: "S1", 3: "S2", 4: "end", 5: "start", 6: "view", 7: "draw+locate", 8: "end",
      16: "start", 20: "lists", 19: "end"}
for name, slots in PH.items():
    base = np.array([ph[row, slots[0]] for row in rows])
    parts = []
    for s_ in slots[1:]:
        v = np.array([ph[row, s_] for row in rows])
        ok = (v > 0) & (base > 0)
        parts.append(f"{NM[s_]} +{np.median(v[ok] - base[ok]) / 1e3:.2f}" if ok.any() else f"{NM[s_]} -")
    print(f"{name} phases (us after start): " + ", ".join(parts))

# per-CTA copy stamps relative to the copy's first CTA start, medians over steps
CN = ["start", "lists", "A issued", "A wait+ready", "B issued", "A m' stored", "A done", "end", "prologue", "B done",
      "B wait", "A 1st land"]
grid = int(((cta[rows[0], :, 0]) > 0).sum())
rel = []
for row in rows[8:]:
    c = cta[row, :grid].astype(np.float64)
    rel.append((c - c[:, 0].min()) / 1e3)
rel = np.array(rel)  # steps x ctas x 8
print(f"copy CTAs: {grid}; per-slot over CTAs (median step): p10 / p50 / p90 / max  [us from first CTA start]")
for k, nm in enumerate(CN):
    v = np.median(rel[:, :, k], axis=0)
    print(f"  {nm:10s} {np.percentile(v, 10):6.2f} {np.percentile(v, 50):6.2f} {np.percentile(v, 90):6.2f} {v.max():6.2f}")
