"""ncu target (tools/, not product): the resident engine at the c2 shape on the whole GPU —
instance 1 is a 400-step prefill, instance 2 the measured run of argv[1] steps (capture it with
`ncu -k regex:drb_run_kernel --launch-skip 1 -c 1`). DRB_IDLE_US defaults to 5 here so the
instance leaves right after its last step (the idle tail is not part of the run)."""
import os
import sys

os.environ.setdefault("DRB_IDLE_US", "5")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_03285_b200 as drb  # noqa: E402
from paper_2406_03285_b200.workload import device_ring, stream_spec  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
K, cap, S, b, r, c = 100, 48, 150528, 56, 7, 14
K, cap = int(os.environ.get("NCU_K", K)), int(os.environ.get("NCU_CAP", cap))  # c3: NCU_K=1000 NCU_CAP=128
spec = stream_spec(K, 4, b, S, steps_per_task=100, seed=1)
sms = torch.cuda.get_device_properties(0).multi_processor_count
ring = int(os.environ.get("AUG_RING", "0"))
buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=1, engine_ctas=sms,
                           aug_ring=ring)
eng = drb.engine(buf)
eng.start()
data, lab = device_ring(spec, 0, 64, "cuda:0")
s = torch.cuda.Stream()
eng.run(data, lab, 400, stream=s)
torch.cuda.synchronize()
reps = int(os.environ.get("REPS", "1"))
ts = []
for _ in range(reps):  # each rep: synchronise (the instance leaves), then one timed run
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    eng.run(data, lab, steps, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1000 / steps)
ts.sort()
print(f"run of {steps} steps (aug_ring {ring or 32}, A ahead {os.environ.get('DRB_A_AHEAD', 8)}): "
      f"{ts[len(ts) // 2]:.2f} us/step (median of {reps}, min {ts[0]:.2f}), instances {eng.engine_info()}")
assert eng.device_error() == 0
eng.shutdown()
