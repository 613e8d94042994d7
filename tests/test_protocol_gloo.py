"""CPU, world_size 2 (gloo): the host-side multi-rank logic.

1. exchange_blobs: the handle all-gather used to wire ranks (dist.py).
2. A CPU model of the distributed protocol the kernels implement: every
   rank keeps only its own buffer, exchanges occupancy rows, replicates every requester's
   global-sampling stream to plan for all of them, derives its PUSH list (every entry of
   any requester's plan(i) whose slot it owns), resolves each slot's version-(i+1) bytes
   the way copy(i) does — the winning candidate's batch row if round i wrote the slot
   (W_i), else the slab row untouched by round i — and sends exactly those rows to their
   requesters (standing in for the NVLink stores) — and must reproduce the N-rank
   synchronous replay oracle bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

M64 = (1 << 64) - 1
PHI = 0x9E3779B97F4A7C15


def mix64(z):
    z = (z + PHI) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class stream:  # rng_stream(seed, worker, purpose) (rng.cpp:19-53), test-only Python port
    def __init__(self, seed, worker, purpose):
        k = mix64(seed)
        k = mix64(k ^ ((worker * 0xD1342543DE82EF95) & M64))
        k = mix64(k ^ ((purpose * 0xAF251AF3B0F025B5) & M64))
        k = mix64(k ^ 0)
        self.key, self.ctr = mix64(k ^ 0), 0

    def bounded(self, n):
        thr = ((1 << 64) - n) % n
        while True:
            self.ctr += 1
            v = mix64(self.key ^ ((self.ctr * PHI) & M64))
            if v >= thr:
                return v % n


def plan(want, occ, s):  # sampler.cpp:39-68 + size_table.cpp:29-39
    flat = occ.reshape(-1)
    total = int(flat.sum())
    if total == 0 or want == 0:
        return []
    pre = np.concatenate([[0], np.cumsum(flat)])
    locate = lambda f: (int(np.searchsorted(pre, f, side="right") - 1))
    K = occ.shape[1]
    fs = list(range(total)) if want >= total else []
    seen = set()
    while len(fs) < want and want < total:
        f = s.bounded(total)
        if f not in seen:
            seen.add(f)
            fs.append(f)
    out = []
    for f in fs:
        i = locate(f)
        out.append((i // K, i % K, f - int(pre[i])))
    return out


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        from oracle.py_oracle import Backend, CANDIDATE, EVICTION, OracleBuffer
        from paper_2406_03285_b200.dist import exchange_blobs
        from paper_2406_03285_b200.workload import stream_spec

        # 1) blob exchange
        blobs = exchange_blobs(bytes([rank]) * 40 + b"rank%02d" % rank)
        assert [b[:1] for b in blobs] == [bytes([w]) for w in range(world)]

        # 2) protocol model vs replay oracle
        K, cap, S, b, c, r, seed, steps = 10, 4, 32, 16, 6, 9, 21, 40
        spec = stream_spec(K, 2, b, S, steps_per_task=12, seed=seed)
        buf = OracleBuffer(K, cap, S)
        cand, evict = buf.stream(seed, rank, CANDIDATE), buf.stream(seed, rank, EVICTION)
        # shadow buffer, same decisions (same labels and streams), payload = (round, batch row)
        # tags: the slots it shows written in round i are W_i (last writer per slot)
        tag = OracleBuffer(K, cap, 8)
        tcand, tevict = type(cand).from_buffer_copy(cand), type(evict).from_buffer_copy(evict)
        samp = [stream(seed, w, 3) for w in range(world)]  # every requester, replicated
        replay = Backend("port").replay(world, K, cap, S, c, r, seed)
        reps, rep_labels = [], []  # reps(i-1): the rows of m'_i pushed during round i-1
        bad = 0
        for i in range(steps):
            data = np.stack([spec.payload(w, i) for w in range(world)])
            labs = np.stack([spec.labels(w, i) for w in range(world)])
            o, ol, oc = replay.step(data, labs)
            # m'_i = m_i ++ reps(i-1)
            got = np.concatenate([data[rank]] + ([np.stack(reps)] if reps else []))
            got_l = np.concatenate([labs[rank], np.array(rep_labels, np.uint32)])
            n = int(oc[rank])
            if not (len(got) == n and np.array_equal(got, o[rank, :n]) and np.array_equal(got_l, ol[rank, :n])):
                bad += 1
            # (a) round-i update of the own buffer only (copy(i) reads the slab as it was)
            before = buf.slab.copy()
            rc, _, _ = buf.update_buffer(data[rank], labs[rank], c, cand, evict)
            assert rc == 0
            tags = np.zeros((len(labs[rank]), 8), np.uint8)
            tags[:, :4] = np.arange(len(labs[rank]), dtype=np.uint32).view(np.uint8).reshape(-1, 4)
            tags[:, 4:] = np.full(len(labs[rank]), i + 1, np.uint32).view(np.uint8).reshape(-1, 4)
            rc, _, _ = tag.update_buffer(tags, labs[rank], c, tcand, tevict)
            assert rc == 0
            tv = tag.slab.view(np.uint32).reshape(K, cap, 2)
            # (b) occupancy rows v = i+1 (the size rendezvous)
            rows = [None] * world
            dist.all_gather_object(rows, buf.occ.copy())
            view = np.stack(rows).astype(np.uint32)
            # (c) plan(i) for every requester; push every owned entry at version i+1
            plans = [plan(r, view, samp[w]) for w in range(world)]
            out = {}
            for w in range(world):
                for j, (ow, cl, sl) in enumerate(plans[w]):
                    if ow != rank:
                        continue
                    won = tv[cl, sl, 1] == i + 1
                    src = data[rank][tv[cl, sl, 0]] if won else before[cl, sl]
                    out.setdefault(w, []).append((j, src.copy()))
            gathered = [None] * world
            dist.all_gather_object(gathered, out)
            mine = {}
            for g in gathered:
                for j, row in g.get(rank, []):
                    mine[j] = row
            assert sorted(mine) == list(range(len(plans[rank])))
            reps = [mine[j] for j in range(len(plans[rank]))]
            rep_labels = [cl for (_, cl, _) in plans[rank]]
        t = torch.tensor([bad])
        dist.all_reduce(t)
        q.put((rank, int(t.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_push_protocol_model_matches_replay(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(w, world, port, q)) for w in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    results = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert results == {w: 0 for w in range(world)}
