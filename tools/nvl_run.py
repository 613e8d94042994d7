"""ncu target (tools/, not product): the resident engine at the c2 shape, one process per GPU
(torchrun), for NVLink byte counters per rank. Instance 1 is a 400-step prefill, instance 2 the
measured run of argv[1] steps. Capture with single-pass metrics only (nvltx/nvlrx bytes and
duration: no kernel replay, so the ranks' instances still meet on the device), e.g.
  ncu --target-processes all -k regex:drb_run_kernel --metrics gpu__time_duration.sum,\
      nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum --csv \
      python -m torch.distributed.run --nproc-per-node 2 ... tools/nvl_run.py 200
Expected pushes per rank per step: r*S*(N-1)/N bytes (the reps owned here, requested by peers)."""
import os
import sys

os.environ.setdefault("DRB_IDLE_US", "5")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2406_03285_b200 as drb  # noqa: E402
from paper_2406_03285_b200.dist import connect_world  # noqa: E402
from paper_2406_03285_b200.workload import device_ring, stream_spec  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("gloo", init_method="env://")
K, cap, S, b, r, c = 100, 48, 150528, 56, 7, 14
spec = stream_spec(K, 4, b, S, steps_per_task=100, seed=1)
sms = torch.cuda.get_device_properties(local).multi_processor_count
buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=1, engine_ctas=sms,
                           rank=rank, world=world, device=local)
connect_world(buf)
eng = drb.engine(buf)
eng.start()
data, lab = device_ring(spec, rank, 64, f"cuda:{local}")
s = torch.cuda.Stream()
for n_steps in (400, steps):
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    eng.run(data, lab, n_steps, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    print(f"rank {rank}: run of {n_steps} steps {e0.elapsed_time(e1) * 1000 / n_steps:.2f} us/step "
          f"(expected pushes {r * S * (world - 1) / world / 1e6:.3f} MB/step/rank)", flush=True)
assert eng.device_error() == 0
eng.shutdown()
dist.barrier()
dist.destroy_process_group()
