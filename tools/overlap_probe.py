"""Probe (tools/, not product): the overlap bench of paper_2406_03285_b200/overlap.py for a
given engine partition (argv[1] = engine CTAs, 0 = default) — prints the overlap_result."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_03285_b200 as drb  # noqa: E402
from paper_2406_03285_b200.overlap import conv_classifier, make_train_step, run_overlap_bench  # noqa: E402
from paper_2406_03285_b200.workload import device_ring, stream_spec  # noqa: E402

ctas = int(sys.argv[1]) if len(sys.argv) > 1 else 0
K, cap, S, b, c, r = 20, 16, 224 * 224 * 3, 56, 14, 7
spec = stream_spec(K, 2, b, S, steps_per_task=50, seed=9)
buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=9, engine_ctas=ctas)
eng = drb.engine(buf)
eng.start()
data, lab = device_ring(spec, 0, 8, "cuda:0")
eng.run(data, lab, 100)
torch.cuda.synchronize()
model = conv_classifier(224, 3, K, width=64).cuda().to(memory_format=torch.channels_last)
res = run_overlap_bench(eng, data, lab, make_train_step(model), 200)
info = eng.engine_info()
eng.shutdown()
print(json.dumps({"engine_ctas": ctas, "idle_us": os.environ.get("DRB_IDLE_US"), **res.__dict__,
                  "wait_fraction": res.wait_fraction, "slowdown_fraction": res.slowdown_fraction, **info}))
