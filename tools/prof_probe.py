"""Probe (tools/): per-phase cycle counts of the sel (CTA 0) and plan (CTA 1) chains of the
resident engine in a long c2 run, from the instrumented build's clock64 accumulators
(DRB_DBG 65536; printed to stderr by synchronize() with DRB_DBG 1024)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "tools", "ablib", "libdrb_inst.so")
if not os.path.exists(LIB) or os.environ.get("REBUILD"):
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    src = [os.path.join(ROOT, "paper_2406_03285_b200", "csrc", f) for f in ("drb_kernels.cu", "drb_capi.cu", "drb_dataset.cu")]
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
                    "-Xcompiler", "-fvisibility=hidden", "-shared", "-DDRB_INSTRUMENT=1", "-o", LIB, *src], check=True)
os.environ["DRB_LIB"] = LIB
os.environ["DRB_DBG"] = str(65536 | 1024)
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2406_03285_b200 as drb  # noqa: E402
from paper_2406_03285_b200.workload import device_ring, stream_spec  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
K, cap, S, b, r, c = 100, 48, 150528, 56, 7, 14
spec = stream_spec(K, 4, b, S, steps_per_task=100, seed=1)
buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=1, engine_ctas=148)
eng = drb.engine(buf)
eng.start()
data, lab = device_ring(spec, 0, 64, "cuda:0")
s = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
eng.run(data, lab, steps, stream=s)
e1.record(s)
torch.cuda.synchronize()
print(f"{steps} steps: {e0.elapsed_time(e1) * 1000 / steps:.2f} us/step (instrumented, prof on)", flush=True)
eng.synchronize()
eng.shutdown()
