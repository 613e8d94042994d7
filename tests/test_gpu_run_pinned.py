"""Every m' of a multi-step drb_rb_run — the call bench.py times — pinned to the oracle.

A run keeps its m'_i only in the engine's m' ring, which the next steps overwrite; created
with a deep ring (aug_ring >= steps) the handle keeps all of them, so each m'_k of the
benchmarked kernel (rows, labels, row count) is compared with the synchronous-replay oracle
after the run: the batch rows the A engine copied (m_k) and the representative rows pushed
by B(k-1) (reps(k-1) drawn at version k, sampler.cpp:234-240, engine.cpp:62-106). The
persistent cooperative kernel (the default) and the three-kernel path (DRB_PERSIST=0) run
the same cases. Inputs: the BASELINE c2 shape (224x224x3 u8, K=100, cap 48, b=56, r=7,
c=14) over 240 steps that cross two class-incremental task boundaries, plus short batches.
"""
import numpy as np
import pytest
import torch

from oracle.py_oracle import Backend
from paper_2406_03285_b200.workload import stream_spec

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["persistent", "three-kernel"])
def drb(request, monkeypatch):
    import paper_2406_03285_b200 as drb
    monkeypatch.setenv("DRB_PERSIST", "1" if request.param == "persistent" else "0")
    return drb


def pinned_run(drb, K, cap, S, b, c, r, seed, T, spt, runs, n=None, pre=0):
    """runs: list of step counts; each run gets distinct batches (one ring slot per step),
    so the labels follow the task schedule across the run."""
    n = b if n is None else n
    total = pre + sum(runs)
    buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=seed,
                               aug_ring=max(6, max(runs) + 1))
    eng = drb.engine(buf)
    eng.start()
    rep = Backend("port").replay(1, K, cap, S, c, r, seed)
    spec = stream_spec(K, T, b, S, steps_per_task=spt, seed=seed)
    i = 0
    for _ in range(pre):  # single steps before the first run (state carried into the run)
        data, lab = spec.payload(0, i, n), spec.labels(0, i, n)
        o, ol, oc = rep.step(data[None], lab[None])
        aug = eng.update((torch.from_numpy(data).cuda(), torch.from_numpy(lab.astype(np.int32)).cuda()))
        assert aug.count() == int(oc[0])
        i += 1
    for steps in runs:
        rd = np.stack([spec.payload(0, i + k, n) for k in range(steps)])
        rl = np.stack([spec.labels(0, i + k, n) for k in range(steps)])
        d_ring = torch.from_numpy(rd).cuda()
        l_ring = torch.from_numpy(rl.astype(np.int32)).cuda()
        eng.run(d_ring, l_ring, steps)
        torch.cuda.synchronize()
        bad = []
        for k in range(steps):
            o, ol, oc = rep.step(rd[k][None], rl[k][None])
            aug = eng.aug_slot(i + k, n)
            cnt = aug.count()
            d, lab = aug.tensors()
            ok = cnt == int(oc[0])
            ok = ok and np.array_equal(lab.cpu().numpy().astype(np.uint32), ol[0, :cnt])
            ok = ok and np.array_equal(d.cpu().numpy(), o[0, :cnt])
            if not ok:
                bad.append(i + k)
        assert not bad, f"m' differs from the oracle at steps {bad[:10]} ({len(bad)} of {steps})"
        i += steps
        del d_ring, l_ring
    assert i == total
    assert eng.device_error() == 0
    eng.shutdown()
    buf.close()


def test_run_every_step_c2_across_task_boundaries(drb):
    # 240 steps, tasks of 100 steps: appends, then replacements, then the next task's classes
    pinned_run(drb, K=100, cap=48, S=150528, b=56, c=14, r=7, seed=1, T=4, spt=100, runs=[240])


def test_run_every_step_short_batches_and_two_runs(drb):
    # n < max_batch inside a run (batch rows right-aligned in m'), single steps before, two runs
    pinned_run(drb, K=20, cap=5, S=4096, b=40, c=14, r=9, seed=5, T=2, spt=30, runs=[70, 45], n=31, pre=3)


def test_run_every_step_replacement_heavy_small(drb):
    # tiny capacity: reps pushed from slots rewritten in the same round (winner batch rows)
    pinned_run(drb, K=4, cap=2, S=64, b=16, c=12, r=5, seed=9, T=1, spt=10**9, runs=[200])
