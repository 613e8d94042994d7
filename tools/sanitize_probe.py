"""Small engine workload for compute-sanitizer (tools/, run under memcheck / racecheck /
synccheck / initcheck): a few single steps, a split-stream step, one multi-step run and the
buffer-level calls, at a small shape; every m' checked against the oracle so a sanitizer
that perturbs timing still has to produce the right bytes. Exit 0 = parity."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_03285_b200 as drb  # noqa: E402
from oracle.py_oracle import Backend  # noqa: E402
from paper_2406_03285_b200.workload import stream_spec  # noqa: E402

K, cap, S, b, c, r, seed = 8, 3, 256, 16, 6, 5, 4
steps_single, steps_run = 6, 10
spec = stream_spec(K, 2, b, S, steps_per_task=8, seed=seed)
buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=seed, engine_ctas=6,
                           aug_ring=steps_run + 2)
eng = drb.engine(buf)
eng.start()
rep = Backend("port").replay(1, K, cap, S, c, r, seed)
bad = 0
i = 0
for _ in range(steps_single):
    d, lab = spec.payload(0, i), spec.labels(0, i)
    o, ol, oc = rep.step(d[None], lab[None])
    aug = eng.update((torch.from_numpy(d).cuda(), torch.from_numpy(lab.astype(np.int32)).cuda()))
    x, y = aug.tensors()
    bad += int(aug.count() != oc[0] or not np.array_equal(x.cpu().numpy(), o[0, :oc[0]]))
    i += 1
rd = np.stack([spec.payload(0, i + k) for k in range(steps_run)])
rl = np.stack([spec.labels(0, i + k) for k in range(steps_run)])
eng.run(torch.from_numpy(rd).cuda(), torch.from_numpy(rl.astype(np.int32)).cuda(), steps_run)
torch.cuda.synchronize()
for k in range(steps_run):
    o, ol, oc = rep.step(rd[k][None], rl[k][None])
    aug = eng.aug_slot(i + k, b)
    x, y = aug.tensors()
    bad += int(aug.count() != oc[0] or not np.array_equal(x.cpu().numpy(), o[0, :oc[0]]))
i += steps_run
loader, trainer = torch.cuda.Stream(), torch.cuda.Stream()
d, lab = spec.payload(0, i), spec.labels(0, i)
o, ol, oc = rep.step(d[None], lab[None])
aug = eng.update((torch.from_numpy(d).cuda(), torch.from_numpy(lab.astype(np.int32)).cuda()), stream=loader,
                 consumer=trainer)
x, y = aug.tensors()
bad += int(aug.count() != oc[0] or not np.array_equal(x.cpu().numpy(), o[0, :oc[0]]))
snap = buf.snapshot()
assert eng.device_error() == 0
eng.shutdown()
print(f"sanitize probe: {steps_single + steps_run + 1} steps, mismatches {bad}, occupancy {snap.per_class}")
sys.exit(1 if bad else 0)
