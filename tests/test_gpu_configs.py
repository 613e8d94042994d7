"""BASELINE.json configs 3-5 at their full sample shapes and class counts, vs the replay oracle.

configs[2] (c3): ImageNet-1K shape, 1000 classes, cap 128 per class per GPU (a 19.3 GB slab),
b=56, r=7; configs[3] (c4): 224x224x3 fp16 (S = 301056 B), b=128, r in {7, 14, 28};
configs[4] (c5): 128x128x1 fp32 (S = 65536 B), 50 classes, b=256, r=32. Payload bytes are
opaque to the path (fp16/fp32 payloads are copied, never computed on), so parity is bytes.

Each case runs the persistent kernel over a device ring long enough to fill classes past
capacity (replacements), checks occupancy/version against the oracle, then checks the m' of
later update() steps bit for bit — their representative rows were pushed by the run's last
iteration from the slab the run left, at version i+1 (S5). Where the slab fits a host
comparison, the occupied slab rows are compared too. The multi-rank variants run every
rank's ring at once over NVLink (N = min(GPUs, 4)).
"""
import numpy as np
import pytest
import torch

from oracle.py_oracle import Backend
from paper_2406_03285_b200.workload import stream_spec

pytestmark = pytest.mark.gpu

C3 = dict(K=1000, cap=128, S=150528, b=56, c=14, r=7, T=4)
C4 = {r: dict(K=100, cap=48, S=301056, b=128, c=14, r=r, T=4) for r in (7, 14, 28)}
C5 = dict(K=50, cap=40, S=65536, b=256, c=14, r=32, T=1)


def ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def to_dev(x, w, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(x))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda(w)


def config_parity(K, cap, S, b, c, r, T, N=1, ring=6, steps=120, post=3, seed=1, spt=None, slab_check=False,
                  small_cap=None, post_steps=True):
    """One world of N ranks (N=1: a plain single-rank buffer); a persistent ring run on every
    rank at once, then `post` update() steps compared with the N-rank replay."""
    import paper_2406_03285_b200 as drb
    cap = small_cap or cap
    spt = spt or max(1, steps // T)
    if N == 1:
        bufs = [drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=seed)]
    else:
        bufs = [drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=seed, rank=w,
                                     world=N, device=w) for w in range(N)]
        blobs = [bf.export_handle() for bf in bufs]
        for bf in bufs:
            bf.connect(blobs)
    if slab_check:  # a slab row no write reached keeps this pattern (cudaMalloc'd slabs are not cleared)
        for bf in bufs:
            bf.slab()[0].fill_(0xA5)
            torch.cuda.synchronize(bf.device)
    engs = [drb.engine(bf) for bf in bufs]
    for e in engs:
        e.start()
    spec = stream_spec(K, T, b, S, steps_per_task=spt, seed=seed)
    rep = Backend("port").replay(N, K, cap, S, c, r, seed)
    # ring slot x holds step x's batch; labels are re-drawn per step from the schedule so
    # the run walks through the tasks (ring payloads repeat, labels do not)
    rd = [np.stack([spec.payload(w, x) for x in range(ring)]) for w in range(N)]
    rings = []
    for w in range(N):
        with torch.cuda.device(w):
            lab = np.stack([spec.labels(w, k) for k in range(steps)])
            rings.append((to_dev(rd[w], w), to_dev(lab.astype(np.int32), w)))
    # data ring of `ring` batches reused cyclically; label ring of `steps` entries: the run
    # indexes both with the same (first + k) % ring, so build a steps-long data view instead
    runs = []
    for w in range(N):
        with torch.cuda.device(w):
            idx = torch.arange(steps, device=f"cuda:{w}") % ring
            runs.append((rings[w][0][idx], rings[w][1]))
    for w in range(N):  # every rank's run in flight at once (they rendezvous on the device)
        with torch.cuda.device(w):
            engs[w].run(runs[w][0], runs[w][1], steps, first=0)
    for k in range(steps):
        rep.step(np.stack([rd[w][k % ring] for w in range(N)]),
                 np.stack([spec.labels(w, k) for w in range(N)]))
    for w in range(N):
        torch.cuda.synchronize(w)
    del runs
    for w in range(N):
        engs[w].synchronize()
        assert engs[w].device_error() == 0, ("run failed on the device", w)
    for w in range(N):
        occ, ver, slab, sl = rep.dump(w) if slab_check else rep.dump(w, occupancy_only=True)
        snap = bufs[w].snapshot()
        assert np.array_equal(np.asarray(snap.per_class, np.uint32), occ), w
        assert snap.version == ver, w
        if slab_check:
            d, l = bufs[w].slab()
            d = d.cpu().numpy().reshape(K, cap, -1)
            l = l.cpu().numpy().reshape(K, cap).astype(np.uint32)
            fp = {rd[w][x, j, :16].tobytes(): (x, j) for x in range(ring) for j in range(b)}
            bad = [(k, s_, "never written" if (d[k, s_] == 0xA5).all() else "stale/wrong",
                    "gpu", fp.get(d[k, s_, :16].tobytes()), "oracle", fp.get(slab[k, s_, :16].tobytes()),
                    int((d[k, s_].reshape(-1, 16) != slab[k, s_].reshape(-1, 16)).any(1).sum()))
                   for k in range(K) for s_ in range(occ[k]) if not np.array_equal(d[k, s_], slab[k, s_])]
            if bad:  # per copy-CTA column detail of the first bad slot (diagnostics)
                k0, s0 = bad[0][0], bad[0][1]
                parts = torch.cuda.get_device_properties(w).multi_processor_count - 2
                c16 = S // 16
                cols = [((c16 * p_ // parts) * 16, (c16 * (p_ + 1) // parts) * 16) for p_ in range(parts)]
                fpc = lambda a, e, row: next((f"{x},{j}" for x in range(ring) for j in range(b)
                                              if np.array_equal(rd[w][x, j, a:e], row[a:e])), None)
                det = [(p_, "pattern" if (d[k0, s0, a:e] == 0xA5).all() else fpc(a, e, d[k0, s0]), fpc(a, e, slab[k0, s0]))
                       for p_, (a, e) in enumerate(cols) if e > a and not np.array_equal(d[k0, s0, a:e], slab[k0, s0, a:e])]
                bad.append(("columns of the first", len(det), det[:10]))
                flat_o = slab.reshape(K * cap, S)
                flat_g = d.reshape(K * cap, S)
                bad.append(("gpu row equals oracle rows", [divmod(x, cap) for x in range(K * cap)
                                                            if np.array_equal(flat_o[x], d[k0, s0])][:6],
                            "oracle row found at gpu rows", [divmod(x, cap) for x in range(K * cap)
                                                             if np.array_equal(flat_g[x], slab[k0, s0])][:6],
                            "gpu row zero", bool((d[k0, s0] == 0).all()),
                            "gpu first bytes", d[k0, s0, :8].tolist()))
                import json
                import os
                if os.environ.get("DRB_TEST_DIAG"):
                    with open(os.environ["DRB_TEST_DIAG"], "a") as f:
                        f.write(json.dumps([str(x) for x in bad]) + "\n")
            assert not bad, (w, len(bad), bad[:8] + bad[-1:])
            for k in range(K):
                assert np.array_equal(l[k, :occ[k]], sl[k, :occ[k]]), (w, k)
    streams = [torch.cuda.Stream(device=w) for w in range(N)]
    fpa = {rd[w][x, j, :16].tobytes(): ("ring", w, x, j) for w in range(N) for x in range(ring) for j in range(b)}
    for i in range(steps, steps + (post if post_steps else 0)):
        data = np.stack([spec.payload(w, i) for w in range(N)])
        labs = np.stack([spec.labels(w, i) for w in range(N)])
        fpa.update({data[w][j, :16].tobytes(): ("post", i, w, j) for w in range(N) for j in range(b)})
        plans_before = [rep.last_plan(w) for w in range(N)]
        o, ol, oc = rep.step(data, labs)
        augs = []
        for w in range(N):
            with torch.cuda.device(w):
                m = (to_dev(data[w], w), to_dev(labs[w].astype(np.int32), w))
                torch.cuda.synchronize(w)
                augs.append(engs[w].update(m, stream=streams[w]))
        for w in range(N):
            d, l = augs[w].tensors()
            cnt = augs[w].count()
            assert cnt == int(oc[w]), (i, w)
            assert np.array_equal(l.cpu().numpy().astype(np.uint32), ol[w, :cnt]), (i, w)
            dd = d.cpu().numpy()
            bad = [j for j in range(cnt) if not np.array_equal(dd[j], o[w, j])]
            info = [(j, "gpu", fpa.get(dd[j, :16].tobytes()), "oracle", fpa.get(o[w, j, :16].tobytes()),
                     "plan", plans_before[w][j - b].tolist() if 0 <= j - b < len(plans_before[w]) else None)
                    for j in bad[:4]]
            assert not bad, (i, w, "rows differ", bad[:16], info)
    for e in engs:
        assert e.device_error() == 0
        e.shutdown()
    for bf in bufs:
        bf.close()


def test_c3_imagenet1k_shape_full_slab():
    """K=1000, cap=128 (19.3 GB slab), 224x224x3 u8, b=56, r=7: 1000-class occupancy table and
    plan locate over N*K = 1000 prefix entries."""
    config_parity(**C3, steps=300)


def test_c3_class_pressure():
    """c3 class count and sample shape with cap=2 so every class replaces (evictions under K=1000)."""
    config_parity(**{**C3, "T": 1}, steps=400, small_cap=2, slab_check=True)


@pytest.mark.parametrize("r", [7, 14, 28])
def test_c4_fp16_b128(r):
    """224x224x3 fp16 (301056 B), b=128, r in {7, 14, 28}; cap 6 so classes fill and replace."""
    config_parity(**C4[r], steps=160, small_cap=6, slab_check=True)


def test_c5_sensor_b256_r32():
    """128x128x1 fp32 (65536 B), 50 classes, b=256, r=32 (a full warp of draws)."""
    config_parity(**C5, steps=120, slab_check=True)


@pytest.mark.multigpu
@pytest.mark.parametrize("name", ["c3", "c4r28", "c5"])
def test_configs_multi_rank(name):
    if ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    N = min(ngpu(), 4)
    if name == "c3":
        config_parity(**C3, N=N, steps=120, small_cap=4)
    elif name == "c4r28":
        config_parity(**C4[28], N=N, steps=100, small_cap=6)
    else:
        config_parity(**C5, N=N, steps=80)
