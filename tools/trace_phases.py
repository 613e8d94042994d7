#!/usr/bin/env python3
"""Per-phase timeline of the step kernel (DRB_TRACE=1): globaltimer stamps written by CTA 0
plus the grid-wide first start / last end. Usage: python tools/trace_phases.py [config]"""
import ctypes as C
import os
import sys

os.environ["DRB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2406_03285_b200 as drb  # noqa: E402
from paper_2406_03285_b200._lib import check, lib  # noqa: E402
from paper_2406_03285_b200.workload import device_ring, stream_spec  # noqa: E402

NAMES = {0: "sel start", 1: "sel loads", 2: "sel S1 done", 3: "sel S2 done", 4: "sel end",
         5: "plan start", 6: "plan view loaded", 7: "plan draws+locate", 8: "plan end",
         16: "copy start (cta0)", 20: "copy lists staged", 21: "copy first B chunk",
         22: "copy first warp done", 18: "copy last warp done", 19: "copy end (cta0)", 14: "copy grid first start",
         15: "copy grid last end"}


def main():
    cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    K, cap, S, b, r, c = cfg["K"], cfg["cap"], cfg["S"], cfg["b"], cfg["r"], cfg["c"]
    spec = stream_spec(K, cfg["T"], b, S, steps_per_task=100, seed=1)
    buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=1)
    eng = drb.engine(buf)
    eng.start()
    data, lab = device_ring(spec, 0, 16, "cuda:0")
    for i in range(450):
        eng.update((data[i % 16], lab[i % 16]))
    torch.cuda.synchronize()
    rows = []
    for i in range(20):
        eng.update((data[i % 16], lab[i % 16]))
        t = np.zeros(32, np.uint64)
        check(lib.drb_rb_trace_read(buf.h, t.ctypes.data))
        rows.append(t.astype(np.int64))
    rows = np.stack(rows)
    t0 = rows[:, 14]
    print(f"config {sys.argv[1] if len(sys.argv) > 1 else 'c2'}; grid={buf.launch_info()}")
    for slot in (0, 1, 2, 3, 4, 5, 6, 7, 8, 14, 16, 20, 21, 22, 18, 19, 15):
        v = rows[:, slot] - t0
        print(f"  {NAMES[slot]:34s} median {np.median(v) / 1000:7.2f} us")
    print(f"  {'grid last end':34s} median {np.median(rows[:, 15] - t0) / 1000:7.2f} us")
    # host submission rate of the native multi-step loop (no sync inside)
    import time
    lab_ring = lab
    torch.cuda.synchronize()
    t0h = time.perf_counter()
    eng.run(data, lab_ring, 2000)
    t1h = time.perf_counter()
    torch.cuda.synchronize()
    t2h = time.perf_counter()
    print(f"  host submit {1e6 * (t1h - t0h) / 2000:.2f} us/step, wall incl. drain {1e6 * (t2h - t0h) / 2000:.2f} us/step (trace on)")


if __name__ == "__main__":
    main()
