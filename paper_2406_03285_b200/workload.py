"""Synthetic class-incremental input streams of the BASELINE.json shapes (input producer,
not the hot path).

Task split follows make_schedule (proj/src/scenario/schedule.cpp:10-35): classes shuffled
by a keyed data_shuffle stream (k1=0xabcd), then cut into T near-equal contiguous chunks.
Within a task, labels are uniform over the task's classes; payload bytes are seeded noise.
Everything is deterministic in (seed, rank, step), so the GPU run and the CPU oracle see
the same bytes.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

import numpy as np

_PHI = 0x9E3779B97F4A7C15
_M = (1 << 64) - 1


def _mix64(z: int) -> int:
    z = (z + _PHI) & _M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M
    return z ^ (z >> 31)


class _host_stream:
    """Host splitmix stream keyed like rng_stream::keyed (rng.cpp:19-39); input generation only."""

    def __init__(self, seed, worker, purpose, k1, k2):
        k = _mix64(seed & _M)
        k = _mix64(k ^ ((worker * 0xD1342543DE82EF95) & _M))
        k = _mix64(k ^ ((purpose * 0xAF251AF3B0F025B5) & _M))
        k = _mix64(k ^ ((k1 + 1) & _M))
        self.key = _mix64(k ^ ((k2 + 1) & _M))
        self.ctr = 0

    def bounded(self, n: int) -> int:
        thr = ((1 << 64) - n) % n
        while True:
            self.ctr += 1
            v = _mix64(self.key ^ ((self.ctr * _PHI) & _M))
            if v >= thr:
                return v % n


def make_schedule(n_classes: int, n_tasks: int, seed: int) -> List[List[int]]:
    if n_tasks == 0 or n_tasks > n_classes:
        raise ValueError("make_schedule: need 1 <= T <= K")
    classes = list(range(n_classes))
    rng = _host_stream(seed, 0, 4, 0xABCD, 0)
    for i in range(n_classes, 1, -1):
        j = rng.bounded(i)
        classes[i - 1], classes[j] = classes[j], classes[i - 1]
    base, extra = divmod(n_classes, n_tasks)
    out, cur = [], 0
    for t in range(n_tasks):
        size = base + (1 if t < extra else 0)
        out.append(classes[cur:cur + size])
        cur += size
    return out


@dataclass
class stream_spec:
    n_classes: int
    n_tasks: int
    batch: int
    sample_bytes: int
    steps_per_task: int
    seed: int = 1

    def schedule(self) -> List[List[int]]:
        if not hasattr(self, "_sched"):
            self._sched = make_schedule(self.n_classes, self.n_tasks, self.seed)
        return self._sched

    def task_of(self, step: int) -> int:
        return (step // self.steps_per_task) % self.n_tasks

    def labels(self, rank: int, step: int, n: int | None = None) -> np.ndarray:
        n = self.batch if n is None else n
        cls = np.asarray(self.schedule()[self.task_of(step)], np.uint32)
        g = np.random.default_rng([self.seed, rank, step, 1])
        return cls[g.integers(0, len(cls), n)].astype(np.uint32)

    def payload(self, rank: int, step: int, n: int | None = None) -> np.ndarray:
        n = self.batch if n is None else n
        g = np.random.default_rng([self.seed, rank, step, 2])
        return g.integers(0, 256, (n, self.sample_bytes), dtype=np.uint8)


def device_ring(spec: stream_spec, rank: int, n_batches: int, device, first_step: int = 0):
    """GPU-resident ring of n_batches batches (torch, generated on device; bench inputs).
    Returns (data uint8 [B, n, S], labels int32 [B, n]). Labels follow spec.labels."""
    import torch
    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(spec.seed * 1000003 + rank)
    data = torch.empty((n_batches, spec.batch, spec.sample_bytes), dtype=torch.uint8, device=dev)
    for b in range(n_batches):  # per batch to bound the int64 temporary of randint
        data[b] = torch.randint(0, 256, (spec.batch, spec.sample_bytes), generator=g, device=dev,
                                dtype=torch.uint8)
    labels = torch.from_numpy(
        np.stack([spec.labels(rank, first_step + b) for b in range(n_batches)]).astype(np.int32)).to(dev)
    return data, labels
