#!/usr/bin/env python3
"""Per-CTA timeline of the persistent run kernel (DRB_TIMELINE): for the copy CTAs, median
over CTAs of each stamp relative to that CTA's B start of the same iteration, and the B-start
period. Usage: python tools/persist_timeline.py [config] [steps]"""
import os
import sys

STEPS = int(sys.argv[2]) if len(sys.argv) > 2 else 64
os.environ["DRB_TIMELINE"] = "1024"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

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
eng.run(data, lab, STEPS)
torch.cuda.synchronize()
n = C.c_uint32(0)
check(lib.drb_rb_timeline_read(buf.h, None, C.byref(n)))
W = 32 + 16 * 160
t = np.zeros(n.value * W, np.uint64)
check(lib.drb_rb_timeline_read(buf.h, t.ctypes.data, C.byref(n)))
t = t.reshape(n.value, W).astype(np.int64)
rows = [(first + i) % n.value for i in range(STEPS)]
cta = t[:, 32:].reshape(n.value, 160, 16)
ncta = torch.cuda.get_device_properties(0).multi_processor_count
NAMES = {0: "B start", 1: "lists parsed", 10: "W published", 11: "W(k-1) seen", 12: "addresses", 3: "B loads issued",
         7: "prev drained", 8: "arrived", 6: "B loads landed", 4: "B stores issued", 9: "B iter end", 2: "A start",
         5: "A end"}
sel = rows[8:-2]
print(f"{'stamp':16s} median over copy CTAs / iterations, us after the CTA's B start")
for s_, nm in NAMES.items():
    v = []
    for row in sel:
        x = cta[row, 2:ncta, s_]
        bs = cta[row, 2:ncta, 0]
        ok = (x > 0) & (bs > 0)
        v.append(np.median((x[ok] - bs[ok]) / 1e3) if ok.any() else np.nan)
    print(f"{nm:16s} {np.nanmedian(v):8.2f}")
bs = np.array([np.median(cta[row, 2:ncta, 0]) for row in rows])
print(f"B start period (median CTA) {np.median(np.diff(bs)) / 1e3:.2f} us; "
      f"A start period {np.median(np.diff([np.median(cta[row, 2:ncta, 2]) for row in rows])) / 1e3:.2f} us")
ph = t[:, 8:32]
for name, a, e in (("sel", 0, 4), ("plan", 5, 8)):
    d = [(ph[row, e] - ph[row, a]) / 1e3 for row in sel]
    st = [ph[row, a] for row in rows]
    print(f"{name}: duration {np.median(d):.2f} us, period {np.median(np.diff(st)) / 1e3:.2f} us; "
          f"start vs B start (median CTA) {np.median([(ph[row, a] - np.median(cta[row, 2:ncta, 0])) / 1e3 for row in sel]):.2f} us")

# control CTAs: CTA 0 (sel) stamps 0 loop top, 1 flags ok, 2 sel_core start, 3 sel_core end, 4 loop end;
# CTA 1 (plan) 0 loop top, 1 flags ok, 3 released. Medians relative to the loop top.
for c, nm, slots in ((0, "sel", (1, 2, 3, 4)), (1, "plan", (1, 3))):
    rel = {s_: np.median([(cta[row, c, s_] - cta[row, c, 0]) / 1e3 for row in sel]) for s_ in slots}
    per = np.median(np.diff([cta[row, c, 0] for row in rows])) / 1e3
    print(f"{nm} CTA: loop period {per:.2f} us; " + ", ".join(f"stamp{s_} +{v:.2f}" for s_, v in rel.items()))
