"""Input side on the GPU, through the C ABI (drb_ds_*): a DRDS file
loaded into HBM, its device features/labels, train/eval_indices_of, the device gather that
produces m, and load_dataset's io_error cases — all bit-exact against the oracle
restatement (oracle/py_input_oracle.py, pinned to the reference in test_input_cpu.py) on the
reference-written fixtures tests/golden/drds_*.drds and on larger seeded files (multi-chunk
streaming, 16 B and 4 B row paths). Ends with gather -> engine step parity: a batch gathered
on the device drives the rehearsal buffer exactly like the same bytes built on the host."""
import os

import numpy as np
import pytest

from oracle import py_input_oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def _D():
    from paper_2406_03285_b200 import dataset as D
    return D


def _check_loaded(ds, path):
    f, lab, k, tr, ev = O.load_dataset(path)
    assert (ds.size(), ds.feature_dim, ds.n_classes, ds.train_count, ds.eval_count) == (len(lab), f.shape[1], k, tr, ev)
    assert np.array_equal(ds.features().cpu().numpy().view(np.uint32), f.view(np.uint32))
    assert np.array_equal(ds.labels().cpu().numpy().astype(np.uint32), lab)
    return f, lab, k, tr


@pytest.mark.parametrize("name", ["drds_small", "drds_odd"])
def test_load_fixture_and_gather(name):
    import torch
    D = _D()
    path = os.path.join(GOLD, name + ".drds")
    ds = D.load_dataset(path, 0)
    f, lab, k, tr = _check_loaded(ds, path)
    for classes in ([0], [1, k - 1], list(range(k)), [k + 7], []):
        assert np.array_equal(ds.train_indices_of(classes), O.indices_of(lab, tr, classes, False))
        assert np.array_equal(ds.eval_indices_of(classes), O.indices_of(lab, tr, classes, True))
    rng = np.random.default_rng(5)
    for n in (0, 1, 7, 56, 300):
        idx = rng.integers(0, len(lab), n)
        m, ml = ds.gather(idx)
        torch.cuda.synchronize()
        of, ol = O.gather(f, lab, idx)
        assert np.array_equal(m.cpu().numpy().view(np.uint32).reshape(n, f.shape[1]), of.view(np.uint32).reshape(n, f.shape[1]))
        assert np.array_equal(ml.cpu().numpy().astype(np.uint32), ol)
    assert ds.device_error() == 0


@pytest.mark.parametrize("dim,count", [(3072, 6000), (37, 20011), (1, 5)])
def test_load_large_and_gather(tmp_path, dim, count):
    """(3072, 6000): 73 MB, two 64 MB staging chunks; (37, 20011): 4 B rows; (1, 5): tiny."""
    import torch
    D = _D()
    rng = np.random.default_rng(dim)
    feats = rng.standard_normal((count, dim)).astype(np.float32)
    labels = rng.integers(0, 100, count).astype(np.uint32)
    p = str(tmp_path / "big.drds")
    O.write_dataset(p, feats, labels, 100, train=count - count // 7, eval_count=count // 7)
    ds = D.load_dataset(p, 0)
    _check_loaded(ds, p)
    idx = torch.randint(0, count, (256,), device="cuda:0")
    out = torch.full((256, dim * 4), 0xAB, dtype=torch.uint8, device="cuda:0")
    m, ml = ds.gather(idx, out=out)
    torch.cuda.synchronize()
    i = idx.cpu().numpy()
    assert np.array_equal(m.cpu().numpy().view(np.float32).view(np.uint32), feats[i].view(np.uint32))
    assert np.array_equal(ml.cpu().numpy().astype(np.uint32), labels[i])


def test_gather_out_of_range_index_sets_the_error_word():
    import torch
    D = _D()
    ds = D.load_dataset(os.path.join(GOLD, "drds_small.drds"), 0)
    out = torch.zeros((3, ds.sample_bytes), dtype=torch.uint8, device="cuda:0")
    ds.gather([0, ds.size(), 1], out=out)
    assert ds.device_error() == 1
    assert out[1].sum().item() == 0 and out[0].sum().item() != 0
    assert ds.device_error() == 0


def test_load_errors_match_the_oracle(tmp_path):
    from test_input_cpu import broken_files
    D = _D()
    for name, path in broken_files(tmp_path):
        with pytest.raises(O.io_error) as mine:
            O.load_dataset(path)
        with pytest.raises(D.io_error) as dev:
            D.load_dataset(path, 0)
        assert str(dev.value).split("] ", 1)[1] == str(mine.value), name


def test_gathered_batch_drives_the_buffer_like_host_bytes(tmp_path):
    """schedule -> shard -> device gather -> update_buffer: same occupancy, slab and reps as
    the same records copied from the host (the producer changes nothing downstream)."""
    import torch
    import paper_2406_03285_b200 as P
    D = _D()
    K, per_class, dim = 10, 60, 48
    rng = np.random.default_rng(9)
    feats = rng.standard_normal((K * per_class, dim)).astype(np.float32)
    labels = np.tile(np.arange(K, dtype=np.uint32), per_class)
    p = str(tmp_path / "t.drds")
    O.write_dataset(p, feats, labels, K)
    ds = D.load_dataset(p, 0)
    sched = D.make_schedule(K, 2, 1)
    task = ds.train_indices_of(sched.tasks[0])
    batches = D.shard_batches(task, 0, 1, 16, 1, 0, 0)
    S = dim * 4
    bufs = [P.rehearsal_buffer(K, 20, S, device=0, max_batch=16) for _ in range(2)]
    streams = [(P.rng_stream(1, 0, 1), P.rng_stream(1, 0, 2)) for _ in range(2)]
    for b in batches[:6]:
        m_dev, l_dev = ds.gather(b)
        m_host = torch.from_numpy(feats[b.astype(np.int64)].view(np.uint8).reshape(len(b), S)).cuda()
        l_host = torch.from_numpy(labels[b.astype(np.int64)].astype(np.int32)).cuda()
        r0 = bufs[0].update_buffer((m_dev, l_dev), 14, *streams[0])
        r1 = bufs[1].update_buffer((m_host, l_host), 14, *streams[1])
        assert (r0.appends, r0.replacements) == (r1.appends, r1.replacements)
    torch.cuda.synchronize()
    assert bufs[0].snapshot().per_class == bufs[1].snapshot().per_class
    s0, s1 = bufs[0].slab(), bufs[1].slab()
    occ = bufs[0].snapshot().per_class
    assert sum(occ) > 0
    for k in range(K):  # slots past occ[k] were never written (uninitialised HBM)
        assert torch.equal(s0[0][k, :occ[k]], s1[0][k, :occ[k]]) and torch.equal(s0[1][k, :occ[k]], s1[1][k, :occ[k]])


def test_epoch_batches_drive_the_engine_like_host_batches(tmp_path):
    """epoch_batches -> engine.update for a whole epoch gives the same m' sequence as the same
    records built on the host (trainer.cpp:94-113 with rehearse = true)."""
    import torch
    import paper_2406_03285_b200 as P
    D = _D()
    K, per_class, dim, b = 10, 80, 32, 16
    rng = np.random.default_rng(21)
    feats = rng.standard_normal((K * per_class, dim)).astype(np.float32)
    labels = np.tile(np.arange(K, dtype=np.uint32), per_class)
    p = str(tmp_path / "e.drds")
    O.write_dataset(p, feats, labels, K)
    ds = D.load_dataset(p, 0)
    sched = D.make_schedule(K, 2, 3)
    task = ds.train_indices_of(sched.tasks[1])
    host_batches = O.shard_batches(task.tolist(), 0, 1, b, 3, 1, 0)[:O.lockstep_batches(len(task), 1, b)]
    engines = []
    for _ in range(2):
        buf = P.rehearsal_buffer(K, 12, dim * 4, max_batch=b, candidate_count=14, rep_count=5, seed=3, device=0)
        eng = P.engine(buf)
        eng.start()
        engines.append((buf, eng))
    got = []
    for step, m in enumerate(D.epoch_batches(ds, task, 0, 1, b, 3, 1, 0)):
        idx = np.asarray(host_batches[step], np.int64)
        m_host = (torch.from_numpy(feats[idx].view(np.uint8).reshape(len(idx), dim * 4)).cuda(),
                  torch.from_numpy(labels[idx].astype(np.int32)).cuda())
        a0 = engines[0][1].update(m)
        a1 = engines[1][1].update(m_host)
        x0, y0 = a0.tensors()
        x1, y1 = a1.tensors()
        assert torch.equal(x0, x1) and torch.equal(y0, y1), step
        got.append(len(y0))
    assert len(got) == len(host_batches) and max(got) > b  # reps arrived after the first round
    for buf, eng in engines:
        eng.shutdown()


@pytest.mark.parametrize("name,args", [("drds_small", (5, 8, 12, 4.0, 11)), ("drds_odd", (3, 6, 7, 3.0, 12))])
def test_synth_dataset_is_bit_identical_to_the_reference(name, args):
    """synth_dataset(K, per_class, dim, separation, seed) in HBM equals the file the reference's
    own synth_dataset + write_dataset produced for the same arguments (oracle/gen_golden_input.py)."""
    from paper_2406_03285_b200 import _lib
    D = _D()
    ds = D.synth_dataset(*args, device=0)
    _check_loaded(ds, os.path.join(GOLD, name + ".drds"))
    with pytest.raises(_lib.config_error):
        D.synth_dataset(3, 5, 4, 0.0, 1)
