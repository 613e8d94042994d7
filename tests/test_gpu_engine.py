"""GPU engine (one fused launch per iteration) vs the synchronous-replay oracle, N=1.

Every augmented mini-batch m'_i = m_i ++ reps(i-1) must be bit-exact (bytes, labels, row
count) against oracle/drb_oracle.c's replay, itself pinned to the reference
(tests/test_oracle.py). Lifecycle errors follow proj/tests/test_engine.cpp:111-247.
"""
import numpy as np
import pytest
import torch

from oracle.py_oracle import Backend
from paper_2406_03285_b200.workload import stream_spec

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["resident", "three-kernel"])
def drb(request, monkeypatch):
    import paper_2406_03285_b200 as drb
    monkeypatch.setenv("DRB_PERSIST", "1" if request.param == "resident" else "0")
    return drb


def dev(data, labels):
    return (torch.from_numpy(np.ascontiguousarray(data)).cuda(),
            torch.from_numpy(np.ascontiguousarray(labels).astype(np.int32)).cuda())


def run_parity(drb, K, cap, S, b, c, r, seed, steps, spec=None, n_of=None, host=False, inplace=False):
    buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=seed)
    eng = drb.engine(buf)
    eng.start()
    rep = Backend("port").replay(1, K, cap, S, c, r, seed)
    spec = spec or stream_spec(K, 1, b, S, steps_per_task=10**9, seed=seed)
    if host:
        out = np.zeros((b + r, S), np.uint8)
        out_l = np.zeros(b + r, np.uint32)
        cnt = np.zeros(1, np.uint32)
    for i in range(steps):
        n = n_of(i) if n_of else b
        lab = spec.labels(0, i, n)
        data = spec.payload(0, i, n)
        o, ol, oc = rep.step(data[None], lab[None])
        if host and inplace:  # m' assembled in the caller's batch buffer (capacity n + r rows)
            slot = np.zeros((n + r, S), np.uint8)
            slot_l = np.zeros(n + r, np.uint32)
            slot[:n], slot_l[:n] = data, lab
            eng.update_host(slot[:n], slot_l[:n], slot, slot_l, cnt)
            eng.synchronize()
            got, got_l, got_c = slot[: cnt[0]], slot_l[: cnt[0]].astype(np.int64), int(cnt[0])
        elif host:
            eng.update_host(data, lab, out, out_l, cnt)
            eng.synchronize()
            got, got_l, got_c = out[: cnt[0]], out_l[: cnt[0]].astype(np.int64), int(cnt[0])
        else:
            aug = eng.update(dev(data, lab))
            d, l = aug.tensors()
            got, got_l, got_c = d.cpu().numpy(), l.cpu().numpy().astype(np.int64), aug.count()
        assert got_c == int(oc[0]), i
        assert np.array_equal(got_l, ol[0, :got_c].astype(np.int64)), i
        assert np.array_equal(got, o[0, :got_c]), i
    eng.shutdown()
    return buf


def test_kat6_config1(drb):
    """KAT6: K=10, cap=100, b=64, c=14, r=8, seed=1; sample j of round i has
    label (64i+j)%10 and features[0] = 64i+j."""
    K, cap, b, c, r, S = 10, 100, 64, 14, 8, 12288
    buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=1)
    eng = drb.engine(buf)
    eng.start()
    f0 = {}
    for i in range(201):
        feats = np.zeros((b, S // 4), np.float32)
        feats[:, 0] = 64 * i + np.arange(b)
        lab = ((64 * i + np.arange(b)) % 10).astype(np.uint32)
        aug = eng.update(dev(feats.view(np.uint8).reshape(b, S), lab))
        if i in (1, 200):
            reps, _ = aug.reps()
            f0[i] = reps.cpu().numpy()[:, :4].copy().view(np.float32)[:, 0].astype(int).tolist()
    assert f0[1] == [49, 11, 57, 45, 63, 56, 26, 20]
    assert f0[200] == [10625, 6439, 10000, 12388, 6326, 9761, 8648, 878]
    eng.shutdown()


@pytest.mark.parametrize("K,cap,S,b,c,r,steps", [
    (10, 100, 12288, 64, 14, 8, 120),      # config 1 shape
    (4, 16, 12, 8, 4, 7, 60),              # engine_config of proj/tests/test_engine.cpp:17-27
    (50, 5, 256, 256, 14, 32, 80),         # config-5 ratios, small payload
    (3, 2, 16, 40, 40, 64, 40),            # r >= total (exhaustion) and c >= b
    (20, 4, 64, 33, 33, 33, 60),           # k > 32 and r > 32 general paths
    (8, 3, 32, 16, 6, 0, 20),              # r = 0
])
def test_engine_matches_replay(drb, K, cap, S, b, c, r, steps):
    run_parity(drb, K, cap, S, b, c, r, seed=K + cap, steps=steps)


def test_engine_short_and_empty_batches(drb):
    run_parity(drb, 12, 6, 64, 48, 14, 7, seed=3, steps=80, n_of=lambda i: [48, 17, 0, 1, 48][i % 5])


def test_engine_class_incremental_c2_full_size(drb):
    """BASELINE config 2 shape on one rank: 224x224x3 u8, K=100 (4 tasks), cap=48, b=56, r=7, c=14."""
    spec = stream_spec(100, 4, 56, 150528, steps_per_task=30, seed=1)
    run_parity(drb, 100, 48, 150528, 56, 14, 7, seed=1, steps=130, spec=spec)


def test_engine_host_path_in_place(drb):
    run_parity(drb, 10, 5, 96, 32, 14, 8, 4, 30, host=True, inplace=True,
               n_of=lambda i: [32, 7, 0, 32, 1][i % 5])


def test_engine_host_path(drb):
    run_parity(drb, 10, 8, 1024, 32, 14, 8, seed=4, steps=40, host=True)


def test_iteration0_and_steady_state_rep_counts(drb):  # test_engine.cpp:237-247
    buf = drb.rehearsal_buffer(4, 16, 12, max_batch=8, candidate_count=4, rep_count=7, seed=77)
    eng = drb.engine(buf)
    eng.start()
    spec = stream_spec(4, 1, 8, 12, 10**9, 77)
    a0 = eng.update(dev(spec.payload(0, 0), spec.labels(0, 0)))
    assert a0.count() == 8  # iteration 0: no representatives
    a1 = eng.update(dev(spec.payload(0, 1), spec.labels(0, 1)))
    assert a1.count() == 8 + 4  # only c=4 stored after round 0
    a2 = eng.update(dev(spec.payload(0, 2), spec.labels(0, 2)))
    assert a2.count() == 8 + 7
    eng.shutdown()


def test_engine_lifecycle_errors(drb):  # test_engine.cpp:174-193
    spec = stream_spec(4, 1, 8, 12, 10**9, 1)
    m = dev(spec.payload(0, 0), spec.labels(0, 0))
    buf = drb.rehearsal_buffer(4, 16, 12, max_batch=8)
    eng = drb.engine(buf)
    with pytest.raises(drb.usage_error):
        eng.update(m)
    with pytest.raises(drb.usage_error):
        eng.shutdown()
    eng.start()
    with pytest.raises(drb.usage_error):
        eng.start()
    eng.update(m)
    eng.shutdown()
    with pytest.raises(drb.usage_error):
        eng.update(m)
    with pytest.raises(drb.usage_error):
        eng.shutdown()


def test_engine_dies_on_bad_label(drb):
    buf = drb.rehearsal_buffer(4, 16, 12, max_batch=8)
    eng = drb.engine(buf)
    eng.start()
    spec = stream_spec(4, 1, 8, 12, 10**9, 1)
    eng.update(dev(spec.payload(0, 0), spec.labels(0, 0)))
    bad = spec.labels(0, 1)
    bad[3] = 9
    a = eng.update(dev(spec.payload(0, 1), bad))
    assert a.count() == 8 + 7  # m'_1 = m_1 ++ reps(0) is still delivered (round 0 was fine)
    with pytest.raises(drb.engine_error):
        eng.update(dev(spec.payload(0, 2), spec.labels(0, 2)))


@pytest.mark.parametrize("ring", [6, 70])
def test_split_streams_pipelined_parity(drb, ring):
    """update(m_i, stream=loader, consumer=trainer) (drb_rb_step_split): every post goes out on
    the loader stream back to back (the engine pipelines them); the trainer stream copies each
    m'_i right after its wait. With the smallest m' ring (6 slots) the engine may refill a slot
    only after the trainer released it — the copies must still equal the oracle's m'."""
    K, cap, S, b, c, r, steps = 20, 6, 4096, 40, 14, 9, 64
    buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=21, aug_ring=ring)
    eng = drb.engine(buf)
    eng.start()
    rep = Backend("port").replay(1, K, cap, S, c, r, 21)
    spec = stream_spec(K, 2, b, S, steps_per_task=25, seed=21)
    loader, trainer = torch.cuda.Stream(), torch.cuda.Stream()
    ins = [dev(spec.payload(0, i), spec.labels(0, i)) for i in range(steps)]
    torch.cuda.synchronize()
    got = []
    for i in range(steps):
        aug = eng.update(ins[i], stream=loader, consumer=trainer)
        with torch.cuda.stream(trainer):
            d, lab = aug.tensors_nowait()
            got.append((d.clone(), lab.clone(), aug))
    torch.cuda.synchronize()
    for i in range(steps):
        o, ol, oc = rep.step(spec.payload(0, i)[None], spec.labels(0, i)[None])
        d, lab, aug = got[i]
        cnt = int(oc[0])
        if ring > steps:  # (a 6-slot ring's row counts are rewritten by later steps by now)
            assert aug.count() == cnt, i
        assert np.array_equal(lab[:cnt].cpu().numpy().astype(np.uint32), ol[0, :cnt]), i
        assert np.array_equal(d[:cnt].cpu().numpy(), o[0, :cnt]), i
    assert eng.device_error() == 0
    eng.shutdown()


def test_drain_timings(drb):
    """engine::drain_timings (engine.hpp:43-50,93): one record per completed round since the
    last drain, from device stamps (resident engine; the three-kernel path records none)."""
    K, cap, S, b, c, r = 10, 8, 1024, 32, 14, 8
    buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=2, record_timings=True)
    eng = drb.engine(buf)
    eng.start()
    spec = stream_spec(K, 1, b, S, steps_per_task=10**9, seed=2)
    for i in range(30):
        eng.update(dev(spec.payload(0, i), spec.labels(0, i)))
    d_ring, l_ring = dev(np.stack([spec.payload(0, 30 + k) for k in range(4)]),
                         np.stack([spec.labels(0, 30 + k) for k in range(4)]))
    eng.run(d_ring, l_ring, 20)
    t = eng.drain_timings()
    resident = eng.engine_info()["resident"]
    if not resident:
        assert t == []
    else:
        assert [x["iteration"] for x in t] == list(range(50))
        for x in t:
            assert x["populate_ms"] > 0 and x["augment_ms"] > 0, x
            assert x["latency_ms"] >= x["augment_ms"], x
            assert x["latency_ms"] < 1000 and x["wait_ms"] == 0 and x["degraded"] == 0, x
        assert eng.drain_timings() == []
        eng.update(dev(spec.payload(0, 60), spec.labels(0, 60)))
        assert [x["iteration"] for x in eng.drain_timings()] == [50]
    eng.shutdown()


def test_instrumentation_counters_and_broadcast_sizes(drb):
    """engine::iterations / queue_depth / degraded_rounds / replanned_entries and
    broadcast_sizes (engine.hpp:82-92): iterations counts enqueued steps, queue_depth drains to
    0 once every m' is ready, nothing degrades or re-plans on a healthy engine, and
    broadcast_sizes (a no-op: rows are published every round) changes nothing."""
    K, cap, S, b, c, r, seed = 10, 4, 256, 24, 14, 7, 12
    buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=seed)
    eng = drb.engine(buf)
    eng.start()
    rep = Backend("port").replay(1, K, cap, S, c, r, seed)
    spec = stream_spec(K, 2, b, S, steps_per_task=5, seed=seed)
    assert eng.iterations() == 0 and eng.queue_depth() == 0
    for i in range(12):
        if i == 5:
            eng.broadcast_sizes()  # task boundary
        o, ol, oc = rep.step(spec.payload(0, i)[None], spec.labels(0, i)[None])
        aug = eng.update(dev(spec.payload(0, i), spec.labels(0, i)))
        assert eng.iterations() == i + 1
        d, l = aug.tensors()
        assert aug.count() == int(oc[0])
        assert np.array_equal(d.cpu().numpy(), o[0, :aug.count()])
    eng.synchronize()
    assert eng.queue_depth() == 0
    assert eng.degraded_rounds() == 0 and eng.replanned_entries() == 0
    eng.shutdown()
