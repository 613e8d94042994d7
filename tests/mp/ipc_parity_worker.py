"""torchrun worker: one process per GPU, CUDA-IPC-mapped peer regions (the bench / training
deployment path). Every rank checks its own m'_i bit-exactly against the N-rank replay
oracle (each process replays all ranks; small config). Exit code 0 = parity."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2406_03285_b200 as drb  # noqa: E402
from oracle.py_oracle import Backend  # noqa: E402
from paper_2406_03285_b200.workload import stream_spec  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo", init_method="env://")
    K, cap, S, b, c, r, seed, steps = 16, 6, 256, 32, 14, 9, 3, 60
    spec = stream_spec(K, 2, b, S, steps_per_task=20, seed=seed)
    run_steps = int(os.environ.get("DRB_PIN_RUN", "50"))  # then one run(), every m' of it pinned
    buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=seed, rank=rank,
                               world=world, device=local, aug_ring=max(6, run_steps + 1))
    from paper_2406_03285_b200.dist import connect_world
    connect_world(buf)
    eng = drb.engine(buf)
    eng.start()
    rep = Backend("port").replay(world, K, cap, S, c, r, seed)
    bad = 0
    for i in range(steps):
        data = np.stack([spec.payload(w, i) for w in range(world)])
        labs = np.stack([spec.labels(w, i) for w in range(world)])
        o, ol, oc = rep.step(data, labs)
        m = (torch.from_numpy(data[rank]).cuda(local), torch.from_numpy(labs[rank].astype(np.int32)).cuda(local))
        aug = eng.update(m)
        d, l = aug.tensors()
        cnt = aug.count()
        ok = cnt == int(oc[rank]) and np.array_equal(l.cpu().numpy().astype(np.uint32), ol[rank, :cnt]) and \
            np.array_equal(d.cpu().numpy(), o[rank, :cnt])
        if not ok:
            bad += 1
            print(f"rank {rank} step {i}: mismatch (count {cnt} vs {oc[rank]})", flush=True)
    # the benchmarked path: one multi-step run over a device ring, every rank's m'_k read back
    # from the deep m' ring after the run and compared step by step
    if run_steps:
        first = steps
        rd = np.stack([np.stack([spec.payload(w, first + k) for w in range(world)]) for k in range(run_steps)])
        rl = np.stack([np.stack([spec.labels(w, first + k) for w in range(world)]) for k in range(run_steps)])
        d_ring = torch.from_numpy(np.ascontiguousarray(rd[:, rank])).cuda(local)
        l_ring = torch.from_numpy(rl[:, rank].astype(np.int32)).cuda(local)
        eng.run(d_ring, l_ring, run_steps)
        torch.cuda.synchronize()
        for k in range(run_steps):
            o, ol, oc = rep.step(rd[k], rl[k])
            aug = eng.aug_slot(first + k, b)
            d, l = aug.tensors()
            cnt = aug.count()
            ok = cnt == int(oc[rank]) and np.array_equal(l.cpu().numpy().astype(np.uint32), ol[rank, :cnt]) and \
                np.array_equal(d.cpu().numpy(), o[rank, :cnt])
            if not ok:
                bad += 1
                print(f"rank {rank} run step {first + k}: mismatch (count {cnt} vs {oc[rank]})", flush=True)
        # every rank is done reading its peers' pushes before any rank tears down
        dist.barrier()
    eng.shutdown()
    t = torch.tensor([bad])
    dist.all_reduce(t)
    dist.destroy_process_group()
    if rank == 0:
        print(f"ipc parity: {world} ranks x ({steps} update steps + a {run_steps}-step run), "
              f"mismatching rank-steps: {int(t.item())}", flush=True)
    sys.exit(1 if int(t.item()) else 0)


if __name__ == "__main__":
    main()
