"""CPU, world_size 2 and 3 (gloo): the input side's multi-rank contract
(proj/src/scenario/schedule.cpp:37-69, used by trainer.cpp:94-99). Every rank derives its
shard for (task, epoch) locally through the product C ABI (drb_shard_batches) with no
communication; all-gathered, the shards must partition the task data exactly once, every
rank must agree on the schedule and on lockstep_batches, and the shards must equal the
oracle restatement's (pinned to the reference in test_input_cpu.py)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bad = 0
    try:
        import numpy as np
        from oracle import py_input_oracle as O
        from paper_2406_03285_b200 import dataset as D

        K, T, seed, b = 100, 4, 1, 56
        sched = D.make_schedule(K, T, seed)
        mine = [sum(sched.tasks, [])]
        every = [None] * world
        dist.all_gather_object(every, mine)
        bad += any(e != mine for e in every)
        # a synthetic class-incremental labelling: record i has label i % K
        labels = np.arange(13001, dtype=np.uint32) % K
        for t, classes in enumerate(sched.tasks):
            task = np.nonzero(np.isin(labels, classes))[0].astype(np.uint64)
            for epoch in range(2):
                shard = D.shard_batches(task, rank, world, b, seed, t, epoch)
                flat = np.concatenate(shard).tolist() if shard else []
                bad += flat != sum(O.shard_batches(task.tolist(), rank, world, b, seed, t, epoch), [])
                steps = D.lockstep_batches(len(task), world, b)
                bad += len(shard) < steps
                got = [None] * world
                dist.all_gather_object(got, (flat, steps))
                allv = sum((g[0] for g in got), [])
                bad += sorted(allv) != sorted(task.tolist())
                bad += len(set(g[1] for g in got)) != 1
    except Exception as e:  # noqa: BLE001
        print(f"rank {rank}: {e!r}")
        bad += 1000
    finally:
        q.put((rank, bad))
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shards_partition_every_task_across_ranks(world):
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
