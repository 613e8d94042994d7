"""Probe (tools/, not product): where the time of one serial update() goes in the resident
engine. Builds the instrumented library (DRB_INSTRUMENT=1) into tools/ablib/, runs serial
updates at the c2 shape with DRB_TIMELINE stamps, and prints, per stamp, the median time
(us) after the posting stream reached the update (a globaltimer stamp kernel just before the
call) — and when the stream got past the wait (stamp kernel right after)."""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.environ.get("INST_LIB") or os.path.join(ROOT, "tools", "ablib", "libdrb_inst.so")
if not os.environ.get("INST_LIB") and (not os.path.exists(LIB) or os.environ.get("REBUILD")):
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    src = [os.path.join(ROOT, "paper_2406_03285_b200", "csrc", f) for f in ("drb_kernels.cu", "drb_capi.cu", "drb_dataset.cu")]
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
                    "-Xcompiler", "-fvisibility=hidden", "-shared", "-DDRB_INSTRUMENT=1", "-o", LIB, *src], check=True)
os.environ["DRB_LIB"] = LIB
os.environ.setdefault("DRB_TIMELINE", "256")
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_03285_b200 as drb  # noqa: E402
from paper_2406_03285_b200 import _lib  # noqa: E402
from paper_2406_03285_b200.workload import device_ring, stream_spec  # noqa: E402

ctas = int(sys.argv[1]) if len(sys.argv) > 1 else 148
mode = sys.argv[2] if len(sys.argv) > 2 else "serial"
world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method="env://")
K, cap, S, b, r, c = 100, 48, 150528, 56, 7, 14
spec = stream_spec(K, 4, b, S, steps_per_task=100, seed=1)
buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=1, engine_ctas=ctas,
                           rank=rank, world=world, device=local)
if world > 1:
    from paper_2406_03285_b200.dist import connect_world
    connect_world(buf)
eng = drb.engine(buf)
eng.start()
data, lab = device_ring(spec, rank, 16, f"cuda:{local}")
s = torch.cuda.Stream()
eng.run(data, lab, 400, stream=s)
torch.cuda.synchronize()
stamp = _lib.lib.drb_dbg_stamp
stamp.argtypes = [C.c_void_p, C.c_void_p]
N = 40 if mode == "serial" else 200
pre = torch.zeros(N, dtype=torch.int64, device=f"cuda:{local}")
post = torch.zeros(N, dtype=torch.int64, device=f"cuda:{local}")
first = eng.iteration
if world > 1:
    dist.barrier()
if mode == "serial":
    for k in range(N):
        stamp(pre.data_ptr() + 8 * k, C.c_void_p(s.cuda_stream))
        eng.update((data[k % 16], lab[k % 16]), stream=s)
        stamp(post.data_ptr() + 8 * k, C.c_void_p(s.cuda_stream))
elif mode == "split":  # update(m, loader, trainer) back to back (the pipelined trainer form)
    loader = torch.cuda.Stream()
    for k in range(N):
        eng.update((data[k % 16], lab[k % 16]), stream=loader, consumer=s)
elif mode == "splitraw":  # the same through raw ctypes calls (the Python wrapper is slower than a step)
    loader = torch.cuda.Stream()
    loader.wait_stream(s)
    fn = _lib.lib.drb_rb_step_split
    out = _lib.drb_aug()
    ptrs = [(C.c_void_p(data[k].data_ptr()), C.c_void_p(lab[k].data_ptr())) for k in range(16)]
    hl, hs, hb = C.c_void_p(loader.cuda_stream), C.c_void_p(s.cuda_stream), buf.h
    for k in range(N):
        fn(hb, ptrs[k % 16][0], ptrs[k % 16][1], b, hl, hs, C.byref(out))
else:  # one run of N pipelined steps: stamps relative to each step's admission
    eng.run(data, lab, N, stream=s)
torch.cuda.synchronize()
n = C.c_uint32(0)
_lib.check(_lib.lib.drb_rb_timeline_read(buf.h, None, C.byref(n)))
W = 32 + 16 * 160
t = np.zeros(n.value * W, np.uint64)
_lib.check(_lib.lib.drb_rb_timeline_read(buf.h, t.ctypes.data, C.byref(n)))
t = t.reshape(n.value, W).astype(np.int64)
cta = t[:, 32:].reshape(n.value, 160, 16)
G = eng.engine_info()["grid"]
pre, post = pre.cpu().numpy(), post.cpu().numpy()
rows = []
for k in range(8, N):
    i = first + k
    row = i % n.value
    base = pre[k] if mode == "serial" else cta[row, 0, 0]  # pipelined: the sel loop top
    rec = {"post_stream_past_wait": post[k] - base}
    def rel(v):
        return (v - base) / 1e3 if v > 0 else np.nan
    rec = {"stream past wait (stamp kernel)": (post[k] - base) / 1e3,
           "feeder admitted": rel(cta[row, G - 1, 13]),
           "sel top": rel(cta[row, 0, 0]), "sel waits done": rel(cta[row, 0, 1]), "sel start": rel(cta[row, 0, 2]),
           "sel handed over": rel(cta[row, 0, 3]), "sel end": rel(cta[row, 0, 4]),
           "plan top": rel(cta[row, 1, 0]), "plan waits done": rel(cta[row, 1, 1]), "plan handed over": rel(cta[row, 1, 3])}
    ph = t[row, 8:32]
    for slot, nm in ((12, "sel: loop top"), (0, "sel: sel_core called"), (1, "sel: sel_core entry"),
                     (2, "sel: S1 drawn"), (3, "sel: S2 assigned"), (4, "sel: W, state, row published"),
                     (13, "plan: loop top"), (5, "plan: plan_core"), (6, "plan: rendezvous done"),
                     (7, "plan: drawn + located"), (8, "plan: push list done")):
        rec[nm] = rel(ph[slot])
    for slot, nm in ((2, "A start"), (5, "A end"), (0, "B start"), (10, "B lists parsed"), (11, "B W(k-1) seen"),
                     (12, "B addresses"), (3, "B loads issued"), (6, "B loads landed"),
                     (4, "B stores issued"), (8, "arrival")):
        v = cta[row, 2:G, slot]
        v = v[v > 0]
        rec[nm + " (median CTA)"] = (np.median(v) - base) / 1e3 if len(v) else np.nan
        if nm == "arrival":
            rec["arrival (last CTA)"] = (v.max() - base) / 1e3 if len(v) else np.nan
    rec["b_done published"] = rel(cta[row, :, 9].max())
    rec["ready published"] = rel(cta[row, G - 1, 14])
    rows.append(rec)
keys = list(rows[0].keys())
print(f"== rank {rank} of {world}")
if mode != "serial":
    tops = [cta[(first + k) % n.value, 0, 0] for k in range(8, N)]
    adm = [cta[(first + k) % n.value, G - 1, 13] for k in range(8, N)]
    rdy = [cta[(first + k) % n.value, G - 1, 14] for k in range(8, N)]
    print(f"feeder admission period {np.median(np.diff(adm)) / 1e3:.2f} us; ready period {np.median(np.diff(rdy)) / 1e3:.2f} us")
    print(f"pipelined run: sel loop-top period {np.median(np.diff(tops)) / 1e3:.2f} us")
    for nm, sl, cc in (("plan top", 0, 1), ("B start", 0, None), ("arrival", 8, None)):
        if cc is not None:
            v = [cta[(first + k) % n.value, cc, sl] for k in range(8, N)]
        else:
            v = [np.median(cta[(first + k) % n.value, 2:G, sl]) for k in range(8, N)]
        print(f"  {nm} period {np.median(np.diff(v)) / 1e3:.2f} us")
print(f"grid {G}, {len(rows)} {mode} steps; us after {'the posting stream reached update()' if mode == 'serial' else 'the sel loop top'} (median):")
for kname in keys:
    print(f"  {kname:34s} {np.nanmedian([r_[kname] for r_ in rows]):8.2f}")
if world > 1:
    dist.barrier()
eng.shutdown()
if world > 1:
    dist.barrier()
