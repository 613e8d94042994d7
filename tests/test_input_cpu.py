"""Input side, CPU checks: the oracle restatement of the DRDS reader,
make_schedule, shard_batches and lockstep_batches against the reference's own outputs
(tests/golden/drds_*.drds written by the reference's write_dataset, tests/golden/input.json,
and oracle/_ref directly when it is built), and the product library's host-side schedule and
shard functions (C ABI, no device needed) against the same vectors. Error cases follow
proj/src/scenario/dataset.cpp:102-143 and schedule.cpp:13-15,44-45."""
import json
import os
import shutil

import numpy as np
import pytest

from oracle import py_input_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
FIXTURES = ["drds_small", "drds_odd"]
have_ref = os.path.exists(O.REF_LIB)


def _golden():
    return json.load(open(os.path.join(GOLD, "input.json")))


def _task_data(n):
    return np.arange(n, dtype=np.uint64) * 3 + 1


def broken_files(tmp_path):
    """(name, path) of malformed DRDS files; every one is an io_error in the reference."""
    src = open(os.path.join(GOLD, "drds_small.drds"), "rb").read()
    cases = {
        "bad_magic": b"DRDX" + src[4:],
        "short_magic": b"DR",
        "version2": src[:4] + (2).to_bytes(2, "little") + src[6:],
        "short_header": src[:13],
        "truncated_record": src[:len(src) - 10],
        "truncated_label": src[:len(src) - 2],
        "label_out_of_range": src[:22 + 13 * 3 * 4 - 4] + (5).to_bytes(4, "little") + src[22 + 13 * 3 * 4:],
        "label_oor_and_truncated": src[:22 + 13 * 4 - 4] + (99).to_bytes(4, "little") + src[22 + 13 * 4:len(src) - 7],
        "bad_split": src,
        "split_sum": src,
    }
    out = []
    for name, data in cases.items():
        p = tmp_path / f"{name}.drds"
        p.write_bytes(data)
        if name == "bad_split":
            (tmp_path / f"{name}.drds.split").write_text("train 35\nevil 5\n")
        elif name == "split_sum":
            (tmp_path / f"{name}.drds.split").write_text("train 35\neval 4\n")
        out.append((name, str(p)))
    out.append(("missing", str(tmp_path / "nope.drds")))
    return out


@pytest.mark.parametrize("name", FIXTURES)
def test_oracle_reads_the_reference_written_fixture(name):
    path = os.path.join(GOLD, name + ".drds")
    f, lab, k, tr, ev = O.load_dataset(path)
    assert f.dtype == np.float32 and lab.dtype == np.uint32
    assert len(lab) == tr + ev and int(lab.max()) < k
    # synth_dataset emits round-robin labels per block (dataset.cpp:189-201)
    assert lab[:k].tolist() == list(range(k))
    if have_ref:
        rf, rl, rk, rtr, rev = O.ref_load(path)
        assert (rk, rtr, rev) == (k, tr, ev)
        assert np.array_equal(rf.view(np.uint32), f.view(np.uint32)) and np.array_equal(rl, lab)


def test_oracle_writer_round_trips_through_the_reference(tmp_path):
    rng = np.random.default_rng(3)
    feats = rng.standard_normal((23, 9)).astype(np.float32)
    feats[0, 0] = np.nan
    labels = rng.integers(0, 4, 23).astype(np.uint32)
    p = str(tmp_path / "w.drds")
    O.write_dataset(p, feats, labels, 4, train=20, eval_count=3)
    f, lab, k, tr, ev = O.load_dataset(p)
    assert np.array_equal(f.view(np.uint32), feats.view(np.uint32)) and np.array_equal(lab, labels)
    assert (k, tr, ev) == (4, 20, 3)
    if have_ref:
        rf, rl, rk, rtr, rev = O.ref_load(p)
        assert np.array_equal(rf.view(np.uint32), feats.view(np.uint32)) and (rk, rtr, rev) == (4, 20, 3)


@pytest.mark.skipif(not have_ref, reason="oracle/_ref not built")
def test_oracle_load_errors_match_the_reference(tmp_path):
    for name, path in broken_files(tmp_path):
        with pytest.raises(O.io_error) as mine:
            O.load_dataset(path)
        with pytest.raises(O.io_error) as ref:
            O.ref_load(path)
        assert str(mine.value) == str(ref.value), name


@pytest.mark.parametrize("name", FIXTURES)
def test_oracle_indices_of_match_the_reference(name):
    if not have_ref:
        pytest.skip("oracle/_ref not built")
    path = os.path.join(GOLD, name + ".drds")
    _, lab, k, tr, _ = O.load_dataset(path)
    cases = [(c, ev) for c in ([0], [1, k - 1], list(range(k)), [k + 3], []) for ev in (0, 1)]
    res = O.ref_batch([{"op": "indices_of", "path": path, "classes": c, "eval": ev, "cap": len(lab)}
                       for c, ev in cases])
    for (classes, ev), r in zip(cases, res):
        assert r == O.indices_of(lab, tr, classes, bool(ev)).tolist(), (classes, ev)


def test_oracle_schedule_and_shards_match_golden():
    g = _golden()
    for s in g["schedules"]:
        tasks = O.make_schedule(s["K"], s["T"], s["seed"])
        assert sum(tasks, []) == s["classes"] and [len(t) for t in tasks] == s["sizes"]
    for s in g["shards"]:
        b = O.shard_batches(_task_data(s["n"]), s["worker"], s["n_workers"], s["batch"], s["seed"], s["task"],
                            s["epoch"])
        assert sum(b, []) == s["shard"] and len(b) == s["n_batches"]
    for s in g["lockstep"]:
        assert O.lockstep_batches(s["n"], s["n_workers"], s["batch"]) == s["batches"]


def test_product_schedule_and_shards_match_golden():
    from paper_2406_03285_b200 import dataset as D
    g = _golden()
    for s in g["schedules"]:
        sched = D.make_schedule(s["K"], s["T"], s["seed"])
        assert sum(sched.tasks, []) == s["classes"] and [len(t) for t in sched.tasks] == s["sizes"]
    for s in g["shards"]:
        b = D.shard_batches(_task_data(s["n"]), s["worker"], s["n_workers"], s["batch"], s["seed"], s["task"],
                            s["epoch"])
        assert len(b) == s["n_batches"] and all(len(x) <= s["batch"] for x in b)
        assert (np.concatenate(b).tolist() if b else []) == s["shard"]
    for s in g["lockstep"]:
        assert D.lockstep_batches(s["n"], s["n_workers"], s["batch"]) == s["batches"]


def test_product_shards_partition_the_task_and_errors():
    from paper_2406_03285_b200 import _lib
    from paper_2406_03285_b200 import dataset as D
    td = _task_data(1001)
    for nw in (1, 2, 3, 8):
        shards = [np.concatenate(D.shard_batches(td, w, nw, 56, 7, 2, 3)) for w in range(nw)]
        allv = np.concatenate(shards)
        assert len(allv) == len(td) and set(allv.tolist()) == set(td.tolist())
        assert D.lockstep_batches(len(td), nw, 56) == (len(td) // nw + 55) // 56
    assert D.shard_batches([], 0, 4, 8, 1, 0, 0) == []
    with pytest.raises(_lib.usage_error):
        D.shard_batches(td, 4, 4, 8, 1, 0, 0)
    with pytest.raises(_lib.config_error):
        D.make_schedule(10, 0, 1)
    with pytest.raises(_lib.config_error):
        D.make_schedule(10, 11, 1)


@pytest.mark.skipif(not have_ref, reason="oracle/_ref not built")
def test_product_shards_match_the_reference_on_random_cases():
    from paper_2406_03285_b200 import dataset as D
    rng = np.random.default_rng(11)
    cases = []
    for _ in range(40):
        n = int(rng.integers(0, 3000))
        nw = int(rng.integers(1, 9))
        cases.append({"op": "shard", "task_data": rng.integers(0, 2**50, n).tolist(), "worker": int(rng.integers(0, nw)),
                      "n_workers": nw, "batch": int(rng.integers(1, 300)), "seed": int(rng.integers(0, 2**40)),
                      "task": int(rng.integers(0, 2**40)), "epoch": int(rng.integers(0, 2**40))})
    for c, r in zip(cases, O.ref_batch(cases)):
        assert r["rc"] == 0
        mine = D.shard_batches(np.asarray(c["task_data"], np.uint64), c["worker"], c["n_workers"], c["batch"],
                               c["seed"], c["task"], c["epoch"])
        assert len(mine) == r["n_batches"]
        assert (np.concatenate(mine).tolist() if mine else []) == r["shard"]


def test_copy_of_fixture_keeps_split(tmp_path):
    # the sidecar travels with the file: a copy without it reads as all-train
    p = tmp_path / "c.drds"
    shutil.copy(os.path.join(GOLD, "drds_small.drds"), p)
    _, lab, _, tr, ev = O.load_dataset(str(p))
    assert (tr, ev) == (len(lab), 0)


def test_product_load_header_errors_before_touching_the_gpu(tmp_path):
    """drb_ds_load rejects a missing file and bad headers before any device work, with the
    reference's io_error messages (dataset.cpp:103-111) — callable without a GPU."""
    from paper_2406_03285_b200 import _lib
    from paper_2406_03285_b200 import dataset as D
    early = {"missing", "bad_magic", "short_magic", "version2", "short_header"}
    for name, path in broken_files(tmp_path):
        if name not in early:
            continue
        with pytest.raises(O.io_error) as mine:
            O.load_dataset(path)
        with pytest.raises(_lib.io_error) as prod:
            D.load_dataset(path, 0)
        assert str(prod.value).split("] ", 1)[1] == str(mine.value), name
    with pytest.raises(_lib.invalid_argument):
        _lib.check(_lib.lib.drb_ds_load(None, 0, None))
