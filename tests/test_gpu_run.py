"""Multi-iteration runs over a device-resident input ring (drb_rb_run, the bench path).

The persistent cooperative launch (default) and the three-kernel path (DRB_PERSIST=0) must
leave the engine exactly where the synchronous-replay oracle is after the same batches:
slab bytes, stored labels, occupancy and version, and every later update() step's m'
(whose representative rows the run's last iteration pushed) bit-exact. Runs are also
captured into CUDA graphs (prepare_run) and interleaved with single steps.
"""
import numpy as np
import pytest
import torch

from oracle.py_oracle import Backend
from paper_2406_03285_b200.workload import stream_spec

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["persistent", "three-kernel"])
def drb(request, monkeypatch):
    import paper_2406_03285_b200 as drb
    monkeypatch.setenv("DRB_PERSIST", "1" if request.param == "persistent" else "0")
    return drb


def dev(data, labels):
    return (torch.from_numpy(np.ascontiguousarray(data)).cuda(),
            torch.from_numpy(np.ascontiguousarray(labels).astype(np.int32)).cuda())


def check_step(eng, rep, data, lab, where):
    o, ol, oc = rep.step(data[None], lab[None])
    aug = eng.update(dev(data, lab))
    d, l = aug.tensors()
    cnt = aug.count()
    assert cnt == int(oc[0]), where
    assert np.array_equal(l.cpu().numpy().astype(np.uint32), ol[0, :cnt]), where
    assert np.array_equal(d.cpu().numpy(), o[0, :cnt]), where


def check_state(buf, rep, K, cap, where):
    occ, ver, slab, sl = rep.dump(0)
    snap = buf.snapshot()
    assert np.array_equal(np.asarray(snap.per_class, np.uint32), occ), where
    assert snap.version == ver, where
    d, l = buf.slab()
    d = d.cpu().numpy().reshape(K, cap, -1)
    l = l.cpu().numpy().reshape(K, cap).astype(np.uint32)
    for k in range(K):  # only occupied slots are defined
        assert np.array_equal(d[k, :occ[k]], slab[k, :occ[k]]), (where, k)
        assert np.array_equal(l[k, :occ[k]], sl[k, :occ[k]]), (where, k)


def ring_parity(drb, K, cap, S, b, c, r, seed, pre, runs, post, ring, T=2, spt=7, graph=False):
    buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=seed)
    eng = drb.engine(buf)
    eng.start()
    rep = Backend("port").replay(1, K, cap, S, c, r, seed)
    spec = stream_spec(K, T, b, S, steps_per_task=spt, seed=seed)
    i = 0
    for _ in range(pre):
        check_step(eng, rep, spec.payload(0, i), spec.labels(0, i), ("pre", i))
        i += 1
    for run_no, (steps, first) in enumerate(runs):
        rd = np.stack([spec.payload(0, 1000 * (run_no + 1) + x) for x in range(ring)])
        rl = np.stack([spec.labels(0, 1000 * (run_no + 1) + x) for x in range(ring)])
        data_ring, lab_ring = dev(rd, rl)
        if graph:
            g = eng.prepare_run(data_ring, lab_ring, steps, first=first)
            g.launch()
        else:
            eng.run(data_ring, lab_ring, steps, first=first)
        for k in range(steps):
            rep.step(rd[(first + k) % ring][None], rl[(first + k) % ring][None])
        torch.cuda.synchronize()
        if graph:
            g.close()
        check_state(buf, rep, K, cap, ("run", run_no))
        for _ in range(post):
            check_step(eng, rep, spec.payload(0, i), spec.labels(0, i), ("post", run_no, i))
            i += 1
    assert eng.device_error() == 0
    eng.shutdown()


def test_run_small(drb):
    ring_parity(drb, K=10, cap=6, S=64, b=24, c=14, r=7, seed=3, pre=3, runs=[(20, 0), (9, 5)], post=4, ring=5)


def test_run_from_start_and_replacement_heavy(drb):
    # run as the very first iterations (reps(-1) empty), tiny capacity -> replacements and
    # reps pushed from slots written in the same round (winner batch rows)
    ring_parity(drb, K=4, cap=2, S=32, b=16, c=12, r=5, seed=9, pre=0, runs=[(30, 2)], post=5, ring=3, T=1)


def test_run_exhaustion_r_ge_total(drb):
    ring_parity(drb, K=3, cap=2, S=48, b=8, c=3, r=40, seed=4, pre=1, runs=[(12, 0)], post=3, ring=4, T=1)


def test_run_c2_sample_shape(drb):
    # 224x224x3 u8 samples, b=56, r=7, c=14 (c2), fewer classes to keep the slab dump small
    ring_parity(drb, K=12, cap=8, S=150528, b=56, c=14, r=7, seed=1, pre=2, runs=[(40, 0)], post=3, ring=6,
                T=3, spt=10)


def test_run_graph_captured(drb):
    ring_parity(drb, K=10, cap=6, S=64, b=24, c=14, r=7, seed=8, pre=2, runs=[(25, 1), (7, 0)], post=3, ring=6,
                graph=True)


def test_run_and_step_ordered_after_default_stream_producer(drb):
    """The batch ring is produced on torch's default stream right before run()/update() with no
    host synchronisation (a long sleep kernel delays the producer): the engine must order its
    reads behind it (the default stream's handle is 0, which the C ABI would otherwise read as
    the engine's own, unordered stream)."""
    K, cap, S, b, c, r, seed, ring = 10, 3, 4096, 24, 14, 7, 21, 4
    buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=seed)
    eng = drb.engine(buf)
    eng.start()
    rep = Backend("port").replay(1, K, cap, S, c, r, seed)
    spec = stream_spec(K, 1, b, S, steps_per_task=10**9, seed=seed)
    rd = np.stack([spec.payload(0, x) for x in range(ring)])
    rl = np.stack([spec.labels(0, x) for x in range(ring)])
    src_d, src_l = dev(rd, rl)
    data = torch.zeros_like(src_d)
    lab = torch.zeros_like(src_l)
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000_000)  # ~0.1 s on the default stream before the producer copies
    data.copy_(src_d)
    lab.copy_(src_l)
    eng.run(data, lab, 12, first=0)
    for k in range(12):
        rep.step(rd[k % ring][None], rl[k % ring][None])
    torch.cuda.synchronize()
    check_state(buf, rep, K, cap, "run after a delayed producer")
    m_d = torch.zeros((b, S), dtype=torch.uint8, device="cuda")
    m_l = torch.zeros((b,), dtype=torch.int32, device="cuda")
    pd, pl = dev(spec.payload(0, 99), spec.labels(0, 99))
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000_000)
    m_d.copy_(pd)
    m_l.copy_(pl)
    aug = eng.update((m_d, m_l))
    o, ol, oc = rep.step(spec.payload(0, 99)[None], spec.labels(0, 99)[None])
    d, l = aug.tensors()
    assert aug.count() == int(oc[0])
    assert np.array_equal(d.cpu().numpy(), o[0, :aug.count()])
    assert np.array_equal(l.cpu().numpy().astype(np.uint32), ol[0, :aug.count()])
    assert eng.device_error() == 0
    eng.shutdown()


def test_runs_on_different_streams_and_graph_then_run(drb):
    """a run() on one stream, another run() on a second stream and a prepared run
    launched on a third, back to back with no host synchronisation, still apply in call order
    (the resident engine admits posts in order; the three-kernel path orders every run behind
    the handle's latest work)."""
    K, cap, S, b, c, r, seed, ring = 10, 4, 256, 24, 14, 7, 33, 5
    buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=seed)
    eng = drb.engine(buf)
    eng.start()
    rep = Backend("port").replay(1, K, cap, S, c, r, seed)
    spec = stream_spec(K, 1, b, S, steps_per_task=10**9, seed=seed)
    rings = []
    for x in range(3):
        rd = np.stack([spec.payload(0, 100 * x + k) for k in range(ring)])
        rl = np.stack([spec.labels(0, 100 * x + k) for k in range(ring)])
        rings.append((rd, rl, dev(rd, rl)))
    torch.cuda.synchronize()
    s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    eng.run(rings[0][2][0], rings[0][2][1], 9, stream=s1)
    eng.run(rings[1][2][0], rings[1][2][1], 7, first=2, stream=s2)
    g = eng.prepare_run(rings[2][2][0], rings[2][2][1], 11, first=1)
    g.launch(s3)
    for x, (steps, first) in enumerate(((9, 0), (7, 2), (11, 1))):
        rd, rl, _ = rings[x]
        for k in range(steps):
            rep.step(rd[(first + k) % ring][None], rl[(first + k) % ring][None])
    torch.cuda.synchronize()
    g.close()
    check_state(buf, rep, K, cap, "three runs on three streams")
    check_step(eng, rep, spec.payload(0, 999), spec.labels(0, 999), "step after")
    assert eng.device_error() == 0
    eng.shutdown()
