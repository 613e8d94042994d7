"""Debug: one short persistent run at a given shape, then report the run counters."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("DRB_PERSIST", "1")
os.environ.setdefault("DRB_DBG", "1024")
os.environ.setdefault("DRB_TIMEOUT_MS", "2000")
import torch
import paper_2406_03285_b200 as drb
from paper_2406_03285_b200.workload import device_ring, stream_spec
K, cap, S, b, c, r, steps = [int(x) for x in (sys.argv[1:] or ["10", "6", "64", "24", "14", "7", "20"])]
spec = stream_spec(K, 2, b, S, steps_per_task=7, seed=3)
buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=3)
eng = drb.engine(buf)
eng.start()
data, lab = device_ring(spec, 0, 5, "cuda:0")
eng.run(data, lab, steps)
eng.synchronize()
print("device_error", eng.device_error())
