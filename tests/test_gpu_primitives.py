"""GPU parity of the device RNG, selection and planning primitives against the CPU oracle
(oracle/drb_oracle.c, pinned to the reference by tests/test_oracle.py).

Bit-exact: every value, every index and the advanced stream counters.
"""
import numpy as np
import pytest

from oracle.py_oracle import Backend, CANDIDATE, EVICTION, GLOBAL_SAMPLING

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc():
    return Backend("port")


@pytest.fixture(scope="module")
def drb():
    import paper_2406_03285_b200 as drb
    return drb


def test_kat1_kat4_next_u64(drb):
    # KATs from SURVEY.md §8c, produced by the reference build.
    s = drb.rng_stream(1, 0, CANDIDATE)
    assert [hex(int(x)) for x in s.next_u64(4)] == [
        "0x825944e4c99d3327", "0x2175e91fe3cdcd23", "0xbf8c000bc894c96b", "0x4bd040e57361fda"]
    s = drb.rng_stream.keyed(1, 0, GLOBAL_SAMPLING, 0x7E, 0)
    assert [hex(int(x)) for x in s.next_u64(2)] == ["0xde53d8c3abe9003", "0x5a142724f691ceb1"]


def test_kat2_bounded(drb):
    s = drb.rng_stream(1, 0, EVICTION)
    assert s.bounded(100, 8).tolist() == [35, 66, 61, 26, 88, 2, 66, 17]
    assert s.counter == 8


@pytest.mark.parametrize("bound", [1, 2, 3, 7, 100, 150528, 2**32 - 5, 2**63 + 1, 2**64 - 3])
def test_bounded_rejection_semantics(drb, orc, bound):
    # bounds near 2^63 / 2^64 reject a large share of draws: counters must still match.
    rng = np.random.default_rng(bound % 1000)
    for _ in range(3):
        seed, worker = int(rng.integers(0, 2**40)), int(rng.integers(0, 8))
        s = drb.rng_stream(seed, worker, GLOBAL_SAMPLING)
        got = s.bounded(bound, 300)
        want = orc.rng_bounded(seed, worker, GLOBAL_SAMPLING, bound, 300)
        assert np.array_equal(got, want)


def test_kat3_sample_without_replacement(drb):
    s = drb.rng_stream(1, 0, CANDIDATE)
    assert drb.sample_without_replacement(64, 14, s).tolist() == [39, 22, 63, 46, 43, 26, 56, 11, 20, 49, 32, 45, 57, 44]
    assert s.counter == 14


def test_swor_random(drb, orc):
    rng = np.random.default_rng(7)
    cases = [(1, 1), (2, 5), (56, 14), (64, 32), (64, 33), (256, 14), (300, 100), (33, 33), (10, 0), (0, 4)]
    cases += [(int(rng.integers(1, 400)), int(rng.integers(0, 60))) for _ in range(40)]
    for n, k in cases:
        seed = int(rng.integers(0, 2**32))
        s = drb.rng_stream(seed, 3, CANDIDATE)
        got = drb.sample_without_replacement(n, k, s)
        want = orc.swor(n, k, seed, 3, CANDIDATE)
        assert got.tolist() == want.tolist(), (n, k)
        assert s.counter == min(n, k)


def test_kat5_plan(drb):
    s = drb.rng_stream(1, 0, GLOBAL_SAMPLING)
    p = drb.plan(8, np.array([[4, 0, 6], [10, 3, 0]]), s)
    assert p.entries.tolist() == [[0, 0, 0], [1, 0, 3], [1, 1, 1], [0, 2, 4], [1, 0, 0], [1, 0, 2], [0, 2, 1], [1, 0, 5]]


def test_plan_random_views(drb, orc):
    rng = np.random.default_rng(11)
    for trial in range(60):
        nw, nk = int(rng.integers(1, 9)), int(rng.integers(1, 60))
        occ = rng.integers(0, 6, (nw, nk)).astype(np.uint32)
        if trial % 7 == 0:
            occ[:] = 0
        want = int(rng.choice([0, 1, 7, 8, 14, 28, 32, 33, 64, 100]))
        seed, worker = int(rng.integers(0, 2**32)), int(rng.integers(0, nw))
        s = drb.rng_stream(seed, worker, GLOBAL_SAMPLING)
        want_rounds = orc.plan(want, occ, seed, worker, GLOBAL_SAMPLING, rounds=4)
        for rd in range(4):  # one stream, consecutive plans: counters must carry exactly
            got = drb.plan(want, occ, s)
            assert got.entries.tolist() == want_rounds[rd].tolist(), (trial, rd)
            assert not got.has_duplicates()


def test_plan_exhaustion_and_empty(drb):
    s = drb.rng_stream(5, 0, GLOBAL_SAMPLING)
    p = drb.plan(7, np.array([[3], [2]]), s)  # r >= total: all slots, flat order, no draws
    assert p.entries.tolist() == [[0, 0, 0], [0, 0, 1], [0, 0, 2], [1, 0, 0], [1, 0, 1]]
    assert s.counter == 0
    assert len(drb.plan(0, np.array([[4, 6]]), s).entries) == 0
    assert len(drb.plan(7, np.array([[0], [0]]), s).entries) == 0


def test_plan_want_beyond_total_and_huge(drb, orc):
    """want far above the view's total (up to UINT32_MAX) returns every slot in flat order
    with no draws (sampler.cpp:45-51); the device scratch is sized by min(want, total), not
    by want. A large want below a larger total draws normally."""
    occ = np.array([[3, 0, 2], [1, 4, 0]], np.uint32)
    flat = [[w, k, s] for w in range(2) for k in range(3) for s in range(int(occ[w, k]))]
    for want in (11, 12, 13000, 2**31, 2**32 - 1):
        s = drb.rng_stream(9, 1, GLOBAL_SAMPLING)
        p = drb.plan(want, occ, s)
        assert p.entries.tolist() == flat, want
        assert s.counter == 0
    big = np.full((4, 250), 20, np.uint32)  # total 20000 > want 9000
    s = drb.rng_stream(3, 2, GLOBAL_SAMPLING)
    got = drb.plan(9000, big, s)
    assert got.entries.tolist() == orc.plan(9000, big, 3, 2, GLOBAL_SAMPLING).tolist()
    assert not got.has_duplicates()
