"""Per-phase cycle accounting of the persistent run's sel / plan CTAs (DRB_DBG 65536|1024; needs the
instrumented build: DRB_INSTRUMENT=1 python -c "import __graft_entry__ as g; g.build_library(force=True)"):
one c2-shape run, single rank. Usage: python tools/prof_run.py [config] [steps]"""
import os, sys
os.environ["DRB_DBG"] = str(65536 | 1024)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2406_03285_b200 as drb
from paper_2406_03285_b200.workload import device_ring, stream_spec
cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
spec = stream_spec(cfg["K"], cfg["T"], cfg["b"], cfg["S"], steps_per_task=100, seed=1)
buf = drb.rehearsal_buffer(cfg["K"], cfg["cap"], cfg["S"], max_batch=cfg["b"], candidate_count=cfg["c"],
                           rep_count=cfg["r"], seed=1)
eng = drb.engine(buf)
eng.start()
data, lab = device_ring(spec, 0, 16, "cuda:0")
s = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
eng.run(data, lab, steps, stream=s)
e1.record(s)
torch.cuda.synchronize()
print(f"{e0.elapsed_time(e1) * 1e3 / steps:.3f} us/step over {steps} steps", flush=True)
eng.synchronize()
