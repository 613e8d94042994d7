"""Probe (tools/, not product): costs of the resident engine's update() path at the c2 shape.
Prints host microseconds per update() (Python) and per raw drb_rb_step call, device time per
serial update, the single-step latency with the instance resident and after it left, and
the run() time for several lengths. Env knobs (DRB_RUN_GRID, DRB_IDLE_US, DRB_FEEDER_LAST) pass
through to the library."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_03285_b200 as drb  # noqa: E402
from paper_2406_03285_b200 import _lib  # noqa: E402
from paper_2406_03285_b200.workload import device_ring, stream_spec  # noqa: E402

K, cap, S, b, r, c = 100, 48, 150528, 56, 7, 14
spec = stream_spec(K, 4, b, S, steps_per_task=100, seed=1)
buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=1)
eng = drb.engine(buf)
eng.start()
ring = 64
data, lab = device_ring(spec, 0, ring, "cuda:0")
s = torch.cuda.Stream()
eng.run(data, lab, 400, stream=s)
torch.cuda.synchronize()
out = {"engine": eng.engine_info()}


def ev():
    return torch.cuda.Event(enable_timing=True)


# host cost of update() in Python and of the raw C call (the first 100 calls: nothing waits for
# descriptor ring space yet)
t0 = time.perf_counter()
for k in range(100):
    eng.update((data[k % ring], lab[k % ring]), stream=s)
out["host_us_per_update_first100"] = (time.perf_counter() - t0) / 100 * 1e6
torch.cuda.synchronize()
n = 2000
t0 = time.perf_counter()
for k in range(n):
    eng.update((data[k % ring], lab[k % ring]), stream=s)
t_py = (time.perf_counter() - t0) / n * 1e6
torch.cuda.synchronize()
aug = _lib.drb_aug()
ptrs = [(data[k].data_ptr(), lab[k].data_ptr()) for k in range(ring)]
sh = C.c_void_p(s.cuda_stream)
t0 = time.perf_counter()
for k in range(n):
    dp, lp = ptrs[k % ring]
    _lib.lib.drb_rb_step(buf.h, dp, lp, b, sh, C.byref(aug))
t_c = (time.perf_counter() - t0) / n * 1e6
torch.cuda.synchronize()
out["host_us_per_update_python"] = t_py
out["host_us_per_update_ctypes"] = t_c

# device time of serial updates (raw calls), instance resident
for nn in (20, 200):
    e0, e1 = ev(), ev()
    e0.record(s)
    for k in range(nn):
        dp, lp = ptrs[k % ring]
        _lib.lib.drb_rb_step(buf.h, dp, lp, b, sh, C.byref(aug))
    e1.record(s)
    torch.cuda.synchronize()
    out[f"device_us_per_serial_update_{nn}"] = 1000 * e0.elapsed_time(e1) / nn

# single-step latency: resident (right after a step) and cold (after the instance left)
lat_res, lat_cold = [], []
for rep in range(20):
    dp, lp = ptrs[rep % ring]
    _lib.lib.drb_rb_step(buf.h, dp, lp, b, sh, C.byref(aug))
    e0, e1 = ev(), ev()
    e0.record(s)
    _lib.lib.drb_rb_step(buf.h, dp, lp, b, sh, C.byref(aug))
    e1.record(s)
    s.synchronize()
    lat_res.append(1000 * e0.elapsed_time(e1))
    torch.cuda.synchronize()  # the instance leaves
    e0, e1 = ev(), ev()
    e0.record(s)
    _lib.lib.drb_rb_step(buf.h, dp, lp, b, sh, C.byref(aug))
    e1.record(s)
    s.synchronize()
    lat_cold.append(1000 * e0.elapsed_time(e1))
out["single_step_us_resident_median"] = float(np.median(lat_res))
out["single_step_us_cold_median"] = float(np.median(lat_cold))

# run() of K steps (sync before: the instance launch is inside)
runs = {}
for ks in (1, 5, 20, 200, 2000):
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record(s)
    eng.run(data, lab, ks, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    runs[ks] = 1000 * e0.elapsed_time(e1) / ks
out["run_us_per_step"] = runs
out["engine_after"] = eng.engine_info()
assert eng.device_error() == 0
eng.shutdown()
print(json.dumps(out))
