"""Multi-rank engine on several GPUs vs the synchronous-replay oracle.

Single process, one rehearsal_buffer per device (peer access over NVLink); every rank's
augmented batch must be bit-exact against oracle/drb_oracle.c's N-rank replay, including
the cross-GPU pushes of representatives owned by other ranks.
"""
import numpy as np
import pytest
import torch

from oracle.py_oracle import Backend
from paper_2406_03285_b200.workload import stream_spec

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def make_world(drb, N, K, cap, S, b, c, r, seed):
    bufs = [drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=seed, rank=w,
                                 world=N, device=w) for w in range(N)]
    blobs = [bf.export_handle() for bf in bufs]
    for bf in bufs:
        bf.connect(blobs)
    engs = [drb.engine(bf) for bf in bufs]
    for e in engs:
        e.start()
    return bufs, engs


def run_multi(drb, N, K, cap, S, b, c, r, seed, steps, T=1, spt=10**9, pattern=None, ring_run=False):
    bufs, engs = make_world(drb, N, K, cap, S, b, c, r, seed)
    spec = stream_spec(K, T, b, S, steps_per_task=spt, seed=seed)
    rep = Backend("port").replay(N, K, cap, S, c, r, seed)
    streams = [torch.cuda.Stream(device=w) for w in range(N)]
    for i in range(steps):
        n = pattern[i % len(pattern)] if pattern else b
        data = np.stack([spec.payload(w, i, n) for w in range(N)])
        labs = np.stack([spec.labels(w, i, n) for w in range(N)])
        o, ol, oc = rep.step(data, labs)
        augs = []
        for w in range(N):  # enqueue every rank before waiting on any (they rendezvous)
            with torch.cuda.device(w):
                m = (torch.from_numpy(data[w]).cuda(w), torch.from_numpy(labs[w].astype(np.int32)).cuda(w))
                torch.cuda.synchronize(w)
                augs.append(engs[w].update(m, stream=streams[w]))
        for w in range(N):
            d, l = augs[w].tensors()
            cnt = augs[w].count()
            assert cnt == int(oc[w]), (i, w)
            assert np.array_equal(l.cpu().numpy().astype(np.uint32), ol[w, :cnt]), (i, w)
            assert np.array_equal(d.cpu().numpy(), o[w, :cnt]), (i, w)
    for e in engs:
        e.shutdown()
    return bufs


def ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("N", [2, 4, 8])
def test_multi_rank_parity_small(N):
    if ngpu() < N:
        pytest.skip(f"needs {N} GPUs")
    import paper_2406_03285_b200 as drb
    run_multi(drb, N, K=12, cap=5, S=64, b=24, c=14, r=7, seed=5, steps=40, T=3, spt=10)


def test_multi_rank_parity_c2_shape():
    if ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    import paper_2406_03285_b200 as drb
    run_multi(drb, 2, K=100, cap=48, S=150528, b=56, c=14, r=7, seed=1, steps=60, T=4, spt=15)


def test_multi_rank_short_batches_and_exhaustion():
    if ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    import paper_2406_03285_b200 as drb
    run_multi(drb, 2, K=6, cap=3, S=16, b=12, c=5, r=40, seed=11, steps=30, pattern=[12, 3, 0, 12, 1])


@pytest.mark.parametrize("N", [2, 4])
def test_multi_process_ipc_parity(N):
    """torchrun, one process per GPU, regions mapped with CUDA IPC handles."""
    if ngpu() < N:
        pytest.skip(f"needs {N} GPUs")
    import os
    import socket
    import subprocess
    import sys
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    worker = os.path.join(os.path.dirname(__file__), "mp", "ipc_parity_worker.py")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={N}",
           "--master-addr=127.0.0.1", f"--master-port={port}", worker]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]


def test_stalled_peer_times_out_without_hanging(monkeypatch):
    """A peer that stops calling update: the reference degrades after its
    rendezvous timeout (size_table.cpp:66-100); here every cross-rank wait is bounded
    (DRB_TIMEOUT_MS), the round fails with a sticky transport error, the next augmented batch
    reports it, the engine is dead for later updates (engine.cpp:67-68,74-80), and shutdown
    still drains — the GPU is not left spinning."""
    if ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    import time

    import paper_2406_03285_b200 as drb
    monkeypatch.setenv("DRB_TIMEOUT_MS", "300")
    K, cap, S, b, c, r = 8, 4, 64, 16, 6, 5
    bufs, engs = make_world(drb, 2, K, cap, S, b, c, r, seed=3)
    spec = stream_spec(K, 1, b, S, steps_per_task=10**9, seed=3)
    streams = [torch.cuda.Stream(device=w) for w in range(2)]

    def upd(w, i):
        with torch.cuda.device(w):
            m = (torch.from_numpy(spec.payload(w, i)).cuda(w),
                 torch.from_numpy(spec.labels(w, i).astype(np.int32)).cuda(w))
            return engs[w].update(m, stream=streams[w])
    for i in range(4):  # healthy rounds
        a = [upd(w, i) for w in range(2)]
        assert [x.count() for x in a] == [b + r if i else b] * 2
    t0 = time.time()
    # rank 1 stalls: never enqueues round 4. update(m_4) returns m_4 ++ reps(3), which the
    # peer's round 3 already delivered — as the reference's update(m_4) returns the reps
    # fetched in round 3 (engine.cpp:62-106) — so it completes; round 4's rendezvous (the
    # peer's occupancy row 5) is what times out, and update(m_5) reports it.
    lone = upd(0, 4)
    assert lone.count() == b + r
    nxt = upd(0, 5)
    try:
        got = nxt.count()
    except drb.engine_error:
        got = None
    assert got is None, ("m'_5 completed without the stalled peer", got, engs[0].device_error(),
                         engs[0].engine_info(), engs[1].engine_info(), time.time() - t0)
    assert time.time() - t0 < 30
    with pytest.raises(drb.engine_error):
        upd(0, 6)
    assert engs[0].device_error() != 0
    for e in engs:
        e.shutdown()


@pytest.mark.parametrize("persist", ["1", "0"])
def test_multi_rank_ring_runs(monkeypatch, persist):
    """Multi-iteration runs over device rings on every rank (the bench path, persistent kernel
    and three-kernel graph path): after the runs, every rank's later update() steps — whose
    representative rows the runs' last pushes delivered — are bit-exact vs the N-rank replay."""
    if ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    import paper_2406_03285_b200 as drb
    monkeypatch.setenv("DRB_PERSIST", persist)
    monkeypatch.setenv("DRB_TIMEOUT_MS", "5000")
    N = min(ngpu(), 4)
    K, cap, S, b, c, r, seed, ring, steps = 12, 5, 1024, 24, 14, 7, 13, 5, 60
    bufs, engs = make_world(drb, N, K, cap, S, b, c, r, seed)
    spec = stream_spec(K, 3, b, S, steps_per_task=10, seed=seed)
    rep = Backend("port").replay(N, K, cap, S, c, r, seed)
    rd = [np.stack([spec.payload(w, 500 + x) for x in range(ring)]) for w in range(N)]
    rl = [np.stack([spec.labels(w, 500 + x) for x in range(ring)]) for w in range(N)]
    rings = []
    for w in range(N):
        with torch.cuda.device(w):
            rings.append((torch.from_numpy(rd[w]).cuda(w), torch.from_numpy(rl[w].astype(np.int32)).cuda(w)))
    for w in range(N):  # every rank's run in flight at once (they rendezvous on the device)
        with torch.cuda.device(w):
            engs[w].run(rings[w][0], rings[w][1], steps, first=1)
    for k in range(steps):
        rep.step(np.stack([rd[w][(1 + k) % ring] for w in range(N)]),
                 np.stack([rl[w][(1 + k) % ring] for w in range(N)]))
    for w in range(N):
        torch.cuda.synchronize(w)
    streams = [torch.cuda.Stream(device=w) for w in range(N)]
    for i in range(3):
        data = np.stack([spec.payload(w, i) for w in range(N)])
        labs = np.stack([spec.labels(w, i) for w in range(N)])
        o, ol, oc = rep.step(data, labs)
        augs = []
        for w in range(N):
            with torch.cuda.device(w):
                m = (torch.from_numpy(data[w]).cuda(w), torch.from_numpy(labs[w].astype(np.int32)).cuda(w))
                torch.cuda.synchronize(w)
                augs.append(engs[w].update(m, stream=streams[w]))
        for w in range(N):
            d, l = augs[w].tensors()
            cnt = augs[w].count()
            assert cnt == int(oc[w]), (i, w)
            assert np.array_equal(l.cpu().numpy().astype(np.uint32), ol[w, :cnt]), (i, w)
            assert np.array_equal(d.cpu().numpy(), o[w, :cnt]), (i, w)
    for e in engs:
        assert e.device_error() == 0
        e.shutdown()
