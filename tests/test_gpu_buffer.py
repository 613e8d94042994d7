"""GPU rehearsal_buffer (update_buffer / read_slots / snapshot) — parity with the oracle and
the reference's own buffer tests (proj/tests/test_buffer.cpp) restated against the C ABI."""
import numpy as np
import pytest
import torch

from oracle.py_oracle import CANDIDATE, EVICTION, SLOT_SUBSTITUTE, OracleBuffer

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def drb():
    import paper_2406_03285_b200 as drb
    return drb


def dev_batch(data: np.ndarray, labels: np.ndarray):
    return (torch.from_numpy(np.ascontiguousarray(data)).cuda(),
            torch.from_numpy(np.ascontiguousarray(labels).astype(np.int32)).cuda())


def tagged(labels, base=0.0, S=8):
    """Samples {tag, tag+0.5} like make_sample (test_buffer.cpp:16-18), padded to S bytes."""
    n = len(labels)
    f = np.zeros((n, S // 4), np.float32)
    f[:, 0] = base + np.arange(n, dtype=np.float32)
    if S >= 8:
        f[:, 1] = f[:, 0] + 0.5
    return f.view(np.uint8).reshape(n, S), np.asarray(labels, np.uint32)


def stream(drb, salt):  # test_buffer.cpp:27-29
    return drb.rng_stream(1000 + salt, 0, CANDIDATE)


def test_empty_buffers_append_candidates(drb):  # test_buffer.cpp:33-45
    buf = drb.rehearsal_buffer(4, 10, 8, max_batch=8)
    cand, evict = stream(drb, 1), stream(drb, 2)
    d, l = tagged([i % 4 for i in range(8)])
    rep = buf.update_buffer(dev_batch(d, l), 2, cand, evict)
    assert rep.appends == 2 and rep.replacements == 0
    assert buf.total_stored() == 2
    assert buf.snapshot().version == 2


def test_short_batches_select_min_c(drb):  # :47-54
    buf = drb.rehearsal_buffer(2, 10, 8, max_batch=8)
    cand, evict = stream(drb, 3), stream(drb, 4)
    d, l = tagged([0, 0, 0])
    assert buf.update_buffer(dev_batch(d, l), 14, cand, evict).appends == 3
    empty = (torch.empty((0, 8), dtype=torch.uint8, device="cuda"), torch.empty(0, dtype=torch.int32, device="cuda"))
    ctr = cand.counter
    assert buf.update_buffer(empty, 14, cand, evict).appends == 0
    assert cand.counter == ctr  # empty batch: no draws


def test_labels_outside_k_rejected(drb):  # :56-61
    buf = drb.rehearsal_buffer(2, 4, 8, max_batch=8)
    cand, evict = stream(drb, 5), stream(drb, 6)
    d, l = tagged([7])
    with pytest.raises(drb.usage_error):
        buf.update_buffer(dev_batch(d, l), 1, cand, evict)
    assert cand.counter == 0 and buf.total_stored() == 0 and buf.snapshot().version == 0
    d, l = tagged([1])  # the buffer stays usable
    assert buf.update_buffer(dev_batch(d, l), 1, cand, evict).appends == 1


def test_class_incremental_never_evicts_across_classes(drb):  # :136-153
    buf = drb.rehearsal_buffer(6, 3, 8, max_batch=8)
    cand, evict = stream(drb, 10), stream(drb, 11)
    for base in range(0, 6, 2):
        for rnd in range(40):
            d, l = tagged([base + (i % 2) for i in range(8)], base=rnd * 8)
            buf.update_buffer(dev_batch(d, l), 4, cand, evict)
    assert buf.cross_class_evictions() == 0
    assert buf.snapshot().per_class == [3] * 6
    slab, slab_labels = buf.slab()
    assert (slab_labels.cpu().numpy() == np.arange(6)[:, None]).all()


def test_occupancy_bounds(drb):  # :155-175
    buf = drb.rehearsal_buffer(3, 5, 8, max_batch=10)
    cand, evict = stream(drb, 12), stream(drb, 13)
    for rnd in range(100):
        d, l = tagged([(rnd + i) % 3 for i in range(10)], base=rnd * 10)
        buf.update_buffer(dev_batch(d, l), 6, cand, evict)
        snap = buf.snapshot()
        assert all(o <= 5 for o in snap.per_class)
        assert snap.total() <= 15 and snap.total() == buf.total_stored()


def test_read_slots_cases(drb):  # :177-214
    buf = drb.rehearsal_buffer(3, 4, 8, max_batch=8)
    cand, evict = stream(drb, 14), stream(drb, 15)
    sub = drb.rng_stream(1, 0, SLOT_SUBSTITUTE)
    e = buf.read_slots([(0, 0)], sub)
    assert e[0].status == drb.rehearsal.READ_EMPTY
    d, l = tagged([1], base=42.0)
    buf.update_buffer(dev_batch(d, l), 1, cand, evict)
    e = buf.read_slots([(1, 0)], sub)
    assert e[0].status == drb.rehearsal.READ_EXACT
    assert e[0].value.cpu().numpy()[:4].view(np.float32)[0] == 42.0
    d, l = tagged([1] * 4, base=50.0)
    buf.update_buffer(dev_batch(d, l), 4, cand, evict)
    for _ in range(20):
        e = buf.read_slots([(1, 9)], sub)
        assert e[0].status == drb.rehearsal.READ_SUBSTITUTED and e[0].label == 1
    e = buf.read_slots([(2, 0)], sub)
    assert e[0].status == drb.rehearsal.READ_SUBSTITUTED and e[0].label == 1


def test_snapshot_and_insertion_report(drb):  # :315-340
    buf = drb.rehearsal_buffer(4, 8, 8, max_batch=8)
    s = buf.snapshot()
    assert s.per_class == [0, 0, 0, 0] and s.version == 0 and s.total() == 0
    cand, evict = stream(drb, 24), stream(drb, 25)
    d, l = tagged([2, 2, 2])
    buf.update_buffer(dev_batch(d, l), 3, cand, evict)
    s = buf.snapshot()
    assert s.per_class == [0, 0, 3, 0] and s.version == 3

    buf = drb.rehearsal_buffer(2, 2, 8, max_batch=8)
    cand, evict = stream(drb, 22), stream(drb, 23)
    r1 = buf.update_buffer(dev_batch(*tagged([0, 0])), 2, cand, evict)
    assert r1.per_class[0] == (2, 0)
    r2 = buf.update_buffer(dev_batch(*tagged([0, 0, 0], base=10.0)), 3, cand, evict)
    assert r2.per_class[0] == (0, 3)
    assert buf.snapshot().version == 5


@pytest.mark.parametrize("K,cap,S,nmax", [(4, 3, 8, 16), (10, 100, 12288, 64), (50, 5, 64, 256), (7, 1, 4, 40),
                                          (100, 48, 150528, 56)])
def test_update_buffer_matches_oracle(drb, K, cap, S, nmax):
    rng = np.random.default_rng(K * 1000 + cap)
    buf = drb.rehearsal_buffer(K, cap, S, max_batch=nmax)
    orc = OracleBuffer(K, cap, S)
    cand, evict = drb.rng_stream(9, 2, CANDIDATE), drb.rng_stream(9, 2, EVICTION)
    ocand, oevict = orc.stream(9, 2, CANDIDATE), orc.stream(9, 2, EVICTION)
    steps = 60 if S > 100000 else 150
    for i in range(steps):
        n = int(rng.integers(0, nmax + 1)) if i % 5 == 4 else nmax
        c = int(rng.choice([0, 1, 14, 32, 33, nmax]))
        lab = rng.integers(0, K, n).astype(np.uint32)
        data = rng.integers(0, 256, (n, S), dtype=np.uint8)
        rep = buf.update_buffer(dev_batch(data, lab), c, cand, evict)
        rc, app, rpl = orc.update_buffer(data, lab, c, ocand, oevict)
        assert rc == 0
        assert rep.appends == int(app.sum()) and rep.replacements == int(rpl.sum())
        assert {k: v for k, v in rep.per_class.items()} == {k: (int(app[k]), int(rpl[k])) for k in range(K) if app[k] or rpl[k]}
        assert cand.counter == ocand.ctr and evict.counter == oevict.ctr
    snap = buf.snapshot()
    assert snap.per_class == orc.occ.tolist() and snap.version == int(orc.version[0])
    slab, slab_labels = buf.slab()
    slab = slab.cpu().numpy()
    for k in range(K):
        o = orc.occ[k]
        assert np.array_equal(slab[k, :o], orc.slab[k, :o]), k
        assert np.array_equal(slab_labels.cpu().numpy()[k, :o], orc.slab_labels[k, :o])


def _read_slots_golden():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "read_slots.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", sorted(_read_slots_golden()))
def test_read_slots_substitute_stream_matches_reference(drb, name):
    """The substitute choices themselves (rehearsal_buffer.cpp:96-121): after the same update
    rounds, the device read_slots with the serve / slot substitute stream returns, per request,
    the status, label and bytes the reference's buffer returned, and leaves the stream where
    the reference left it (tests/golden/read_slots.json, generated from oracle/_ref)."""
    import hashlib

    from paper_2406_03285_b200.workload import stream_spec
    g = _read_slots_golden()[name]
    c = g["config"]
    buf = drb.rehearsal_buffer(c["K"], c["cap"], c["S"], max_batch=c["n"])
    spec = stream_spec(c["K"], c["T"], c["n"], c["S"], steps_per_task=10**9, seed=c["seed"])
    cand = drb.rng_stream(c["seed"], 0, CANDIDATE)
    evict = drb.rng_stream(c["seed"], 0, EVICTION)
    for i in range(c["rounds"]):
        buf.update_buffer(dev_batch(spec.payload(0, i, c["n"]), spec.labels(0, i, c["n"])), c["c"], cand, evict)
    assert buf.snapshot().per_class == g["occ"]
    if c["keyed"]:
        sub = drb.rng_stream.keyed(c["seed"], 0, c["purpose"], c["k1"], c["k2"])
    else:
        sub = drb.rng_stream(c["seed"], 0, c["purpose"])
    got = buf.read_slots([tuple(x) for x in g["requests"]], sub)
    assert [e.status for e in got] == g["status"]
    assert [e.label for e in got] == g["labels"]
    data = np.stack([e.value.cpu().numpy() for e in got])
    assert hashlib.sha256(np.ascontiguousarray(data).tobytes()).hexdigest() == g["bytes_sha256"]
    assert hex(int(sub.next_u64()[0])) == g["sub_next_u64"]
