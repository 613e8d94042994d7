"""CPU: pin the C restatement (oracle/drb_oracle.c) to the reference.

(1) tests/golden/*.json were generated from the reference itself (oracle/gen_golden.py over
    oracle/_ref/libdrb_ref.so, the unmodified reference sources); the port must reproduce
    every vector and every per-step m' digest.
(2) When oracle/_ref is built (this container), port and reference are compared directly
    on randomised configurations, including the multi-rank synchronous replay.
"""
import json
import os

import numpy as np
import pytest

from oracle.gen_golden import REPLAY_CONFIGS, digest
from oracle.py_oracle import Backend, CANDIDATE, EVICTION, GLOBAL_SAMPLING, have_reference
from paper_2406_03285_b200.workload import make_schedule, stream_spec

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def kat():
    return json.load(open(os.path.join(GOLD, "kat.json")))


@pytest.fixture(scope="module")
def port():
    return Backend("port")


def test_kat1_to_kat5(port, kat):
    assert [hex(int(x)) for x in port.rng_next(1, 0, CANDIDATE, 4)] == kat["kat1_next_u64_seed1_w0_candidate"]
    assert port.rng_bounded(1, 0, EVICTION, 100, 8).tolist() == kat["kat2_bounded100_seed1_w0_eviction"]
    assert port.swor(64, 14, 1).tolist() == kat["kat3_swor_64_14"]
    assert [hex(int(x)) for x in port.rng_next(1, 0, GLOBAL_SAMPLING, 2, keyed=True, k1=0x7E)] == kat["kat4_keyed_7e"]
    assert port.plan(8, np.array([[4, 0, 6], [10, 3, 0]]), 1).tolist() == kat["kat5_plan"]
    # the SURVEY.md §8c literal values (independent of the fixture file)
    assert kat["kat3_swor_64_14"] == [39, 22, 63, 46, 43, 26, 56, 11, 20, 49, 32, 45, 57, 44]
    assert kat["kat2_bounded100_seed1_w0_eviction"] == [35, 66, 61, 26, 88, 2, 66, 17]


def test_rejection_heavy_bounds(port, kat):
    for bd, vals in kat["bounded_big"].items():
        assert [str(int(x)) for x in port.rng_bounded(3, 1, GLOBAL_SAMPLING, int(bd), 64)] == vals


def test_swor_and_plan_vectors(port, kat):
    for v in kat["swor_random"]:
        assert port.swor(v["n"], v["k"], v["seed"]).tolist() == v["out"]
    for v in kat["plan_random"]:
        got = port.plan(v["want"], np.array(v["occ"], np.uint32), v["seed"], 0, GLOBAL_SAMPLING, rounds=3)
        assert [g.tolist() for g in got] == v["rounds"]


def test_kat6_config1(port, kat):
    K, cap, b, c, r, S = 10, 100, 64, 14, 8, 16
    rp = port.replay(1, K, cap, S, c, r, 1)
    for i in range(200):
        feats = np.zeros((b, S // 4), np.float32)
        feats[:, 0] = 64 * i + np.arange(b)
        lab = ((64 * i + np.arange(b)) % 10).astype(np.uint32)
        aug, al, cnt = rp.step(feats.view(np.uint8).reshape(1, b, S), lab[None])
        assert rp.last_plan(0)[:, 1:].tolist() == kat["kat6_plans_cls_slot"][i]
        if i > 0:
            assert aug[0, b:cnt[0], :4].copy().view(np.float32)[:, 0].astype(int).tolist() == kat["kat6_reps_f0"][i - 1]
    assert kat["kat6_reps_f0"][0] == [49, 11, 57, 45, 63, 56, 26, 20]
    assert kat["kat6_reps_f0"][199] == [10625, 6439, 10000, 12388, 6326, 9761, 8648, 878]


@pytest.mark.parametrize("cfg", REPLAY_CONFIGS, ids=[c[0] for c in REPLAY_CONFIGS])
def test_replay_digests(port, cfg):
    gold = json.load(open(os.path.join(GOLD, "replay.json")))[cfg[0]]["digests"]
    name, N, K, cap, S, b, c, r, seed, T, spt, steps, pattern = cfg
    spec = stream_spec(K, T, b, S, steps_per_task=spt, seed=seed)
    rp = port.replay(N, K, cap, S, c, r, seed)
    for i in range(steps):
        n = pattern[i % len(pattern)] if pattern else b
        data = np.stack([spec.payload(w, i, n) for w in range(N)])
        labs = np.stack([spec.labels(w, i, n) for w in range(N)])
        aug, al, cnt = rp.step(data, labs)
        assert [digest(aug[w], al[w], int(cnt[w])) for w in range(N)] == gold[i], (name, i)


def test_bad_label_is_usage_error_before_any_draw(port):
    rp = port.replay(1, 4, 2, 8, 3, 2, 1)
    with pytest.raises(ValueError):
        rp.step(np.zeros((1, 4, 8), np.uint8), np.array([[0, 1, 9, 2]], np.uint32))
    assert rp.counters(0).tolist() == [0, 0, 0]


@pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built (no /root/reference here)")
def test_port_equals_reference_randomised():
    P, R = Backend("port"), Backend("reference")
    rng = np.random.default_rng(2024)
    for trial in range(25):
        N, K, cap = int(rng.integers(1, 6)), int(rng.integers(1, 14)), int(rng.integers(1, 9))
        S, n = 4 * int(rng.integers(1, 6)), int(rng.integers(0, 24))
        c, r, seed = int(rng.integers(0, 30)), int(rng.integers(0, 40)), int(rng.integers(0, 10**6))
        a, b = P.replay(N, K, cap, S, c, r, seed), R.replay(N, K, cap, S, c, r, seed)
        for step in range(30):
            nn = n if step % 5 else int(rng.integers(0, n + 1))
            bat = rng.integers(0, 256, (N, nn, S), dtype=np.uint8)
            lab = rng.integers(0, K, (N, nn)).astype(np.uint32)
            for u, v in zip(a.step(bat, lab), b.step(bat, lab)):
                assert np.array_equal(u, v), (trial, step)
            for w in range(N):
                assert np.array_equal(a.last_plan(w), b.last_plan(w))
                for u, v in zip(a.last_report(w), b.last_report(w)):
                    assert np.array_equal(u, v)
        for w in range(N):
            oa, ob = a.dump(w), b.dump(w)
            assert np.array_equal(oa[0], ob[0]) and oa[1] == ob[1]
            assert np.array_equal(oa[2], ob[2]) and np.array_equal(oa[3], ob[3])


@pytest.mark.skipif(not have_reference(), reason="oracle/_ref not built")
def test_schedule_stream_matches_reference_rng():
    # make_schedule shuffles with keyed(seed, 0, data_shuffle, 0xabcd) (schedule.cpp:17-20)
    R = Backend("reference")
    from paper_2406_03285_b200.workload import _host_stream
    s = _host_stream(5, 0, 4, 0xABCD, 0)
    assert [s.bounded(97) for _ in range(50)] == R.rng_bounded(5, 0, 4, 97, 50, keyed=True, k1=0xABCD).tolist()
    sched = make_schedule(100, 4, 1)
    assert sorted(sum(sched, [])) == list(range(100)) and [len(t) for t in sched] == [25] * 4


def test_port_bias_counts_match_reference_golden():
    """The C restatement's bias-test counts (plan rounds on rank 0's stream) against the
    reference's, tests/golden/bias.json (oracle/gen_golden.py, bias.cpp:104-133)."""
    import hashlib
    from oracle.py_oracle import Backend, bias_counts, bias_view
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "bias.json")))["draws_2000"]
    be = Backend("port")
    for name, g in gold.items():
        occ = bias_view(g["N"], g["K"], g["fill"])
        assert occ.tolist() == g["occ"], name
        c = bias_counts(be, occ, g["r"], g["seed"], g["draws"], g["local_only"])
        assert hashlib.sha256(c.astype("<u8").tobytes()).hexdigest() == g["counts_sha256"], name


def _read_slots_golden():
    with open(os.path.join(os.path.dirname(__file__), "golden", "read_slots.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", sorted(_read_slots_golden()))
def test_port_read_slots_matches_reference_golden(name):
    """read_slots (rehearsal_buffer.cpp:88-142) of the C restatement after the same update
    rounds: statuses, labels, bytes and the substitute stream's position, as the reference's
    own buffer produced them (tests/golden/read_slots.json, oracle/gen_golden.py)."""
    import hashlib

    from oracle.py_oracle import OracleBuffer
    g = _read_slots_golden()[name]
    c = g["config"]
    ob = OracleBuffer(c["K"], c["cap"], c["S"])
    spec = stream_spec(c["K"], c["T"], c["n"], c["S"], steps_per_task=10**9, seed=c["seed"])
    cand = ob.stream(c["seed"], 0, CANDIDATE)
    evict = ob.stream(c["seed"], 0, EVICTION)
    for i in range(c["rounds"]):
        rc, _, _ = ob.update_buffer(spec.payload(0, i, c["n"]), spec.labels(0, i, c["n"]), c["c"], cand, evict)
        assert rc == 0
    assert ob.occ.tolist() == g["occ"]
    sub = ob.stream(c["seed"], 0, c["purpose"], bool(c["keyed"]), c["k1"], c["k2"])
    d, lab, st = ob.read_slots([tuple(x) for x in g["requests"]], sub)
    assert st.tolist() == g["status"]
    assert lab.tolist() == g["labels"]
    assert hashlib.sha256(np.ascontiguousarray(d).tobytes()).hexdigest() == g["bytes_sha256"]
    assert hex(ob.next_u64(sub)) == g["sub_next_u64"]
