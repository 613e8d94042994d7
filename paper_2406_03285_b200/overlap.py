"""Asynchronous overlap of the rehearsal engine with a real training step.

The reference measures this with `run_overlap_bench` (proj/src/runner/overlap.cpp:39-120,
acceptance criterion 5 of proj/tests/acceptance.cpp:229-256): calibrate the background round
cost, run a training stub of >= 10x that cost after every `engine.update(m)`, and require the
mean time the trainer waits for its augmented batch to stay under 5% of the iteration.

Here the trainer is a real GPU training step (forward, backward and SGD update of a small
convolutional classifier on m'_i, bf16 autocast) on its own CUDA stream, next to the
resident engine on its partition of the SMs. update(m_{i+1}) posts m_{i+1} on the loader's
stream right after step i is enqueued, so round i+1's selection, sampling and copy run while
step i trains; the train stream only waits for m'_{i+1} behind step i. Everything is timed on
the device:
  background_ms      engine alone, device time per update
  train_ms           the training step alone on a resident batch
  iteration_ms       the overlapped loop, per iteration (train stream events)
  wait_ms            the train stream blocked on m'_i (the reference's wait_ms: time
                     update() blocks, engine.cpp:82-90)
  slowdown_ms        iteration_ms - train_ms: what the trainer lost overall (waiting for
                     m'_i, and SM / HBM contention with the engine)
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.nn as nn


@dataclass
class overlap_result:  # overlap_stats (proj/include/drb.h:70-77)
    train_cost_ms: float
    background_ms: float
    mean_wait_ms: float        # the train stream blocked on m'_i (engine.cpp:82-90 wait_ms)
    mean_iteration_ms: float
    iterations: int
    mean_slowdown_ms: float = 0.0  # iteration - training alone: blocking + SM / HBM contention

    @property
    def wait_fraction(self) -> float:
        return self.mean_wait_ms / self.mean_iteration_ms if self.mean_iteration_ms > 0 else 0.0

    @property
    def slowdown_fraction(self) -> float:
        return self.mean_slowdown_ms / self.mean_iteration_ms if self.mean_iteration_ms > 0 else 0.0


class conv_classifier(nn.Module):
    """The consumer: a small CNN over H x W x C uint8 samples (channels-last bytes)."""

    def __init__(self, hw: int, ch: int, n_classes: int, width: int = 64, depth: int = 4):
        super().__init__()
        self.hw, self.ch = hw, ch
        layers, c = [], ch
        for i in range(depth):
            layers += [nn.Conv2d(c, width * (2 ** min(i, 2)), 3, stride=2, padding=1), nn.ReLU(inplace=True)]
            c = width * (2 ** min(i, 2))
        self.body = nn.Sequential(*layers)
        self.head = nn.Linear(c, n_classes)

    def forward(self, x_u8: torch.Tensor) -> torch.Tensor:
        x = x_u8.view(-1, self.hw, self.hw, self.ch).permute(0, 3, 1, 2).float().div_(255.0)
        x = x.contiguous(memory_format=torch.channels_last)
        return self.head(self.body(x).mean(dim=(2, 3)))


def make_train_step(model: nn.Module, lr: float = 0.01):
    opt = torch.optim.SGD(model.parameters(), lr=lr, momentum=0.9)
    loss_fn = nn.CrossEntropyLoss()

    def step(data_u8: torch.Tensor, labels: torch.Tensor) -> torch.Tensor:
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = loss_fn(model(data_u8), labels.long())
        opt.zero_grad(set_to_none=True)
        loss.backward()
        opt.step()
        return loss

    return step


def run_overlap_bench(eng, data_ring: torch.Tensor, label_ring: torch.Tensor, train_step, iterations: int,
                      calib: int = 60) -> overlap_result:
    """eng: a started engine; data_ring [B, n, S] u8 / label_ring [B, n] int32 on its device."""
    dev = data_ring.device
    B = data_ring.shape[0]
    s_eng = torch.cuda.Stream(device=dev)
    s_train = torch.cuda.Stream(device=dev)

    def ev():
        return torch.cuda.Event(enable_timing=True)

    # background: engine alone (device time per update, steady state)
    with torch.cuda.stream(s_eng):
        for i in range(calib):
            eng.update((data_ring[i % B], label_ring[i % B]), stream=s_eng)
    torch.cuda.synchronize(dev)
    e0, e1 = ev(), ev()
    e0.record(s_eng)
    for i in range(calib):
        eng.update((data_ring[i % B], label_ring[i % B]), stream=s_eng)
    e1.record(s_eng)
    torch.cuda.synchronize(dev)
    background_ms = e0.elapsed_time(e1) / calib

    # training step alone, on a resident augmented batch
    aug = eng.update((data_ring[0], label_ring[0]), stream=s_eng)
    d, l = aug.tensors()
    d, l = d.clone(), l.clone()
    torch.cuda.synchronize(dev)
    with torch.cuda.stream(s_train):
        for _ in range(5):
            train_step(d, l)
    torch.cuda.synchronize(dev)
    e0.record(s_train)
    with torch.cuda.stream(s_train):
        for _ in range(min(iterations, 100)):
            train_step(d, l)
    e1.record(s_train)
    torch.cuda.synchronize(dev)
    train_ms = e0.elapsed_time(e1) / min(iterations, 100)

    # overlapped loop (the reference's trainer, trainer.cpp:109-113, with the loader on its own
    # stream): after step i is enqueued on the train stream, update(m_{i+1}) posts m_{i+1} on
    # the engine stream — round i+1 runs on the device while step i trains — and the train
    # stream releases m'_i and waits for m'_{i+1} behind step i (drb_rb_step_split)
    aug = eng.update((data_ring[0], label_ring[0]), stream=s_eng, consumer=s_train)
    torch.cuda.synchronize(dev)
    w0 = [ev() for _ in range(iterations)]
    w1 = [ev() for _ in range(iterations)]
    e0.record(s_train)
    for i in range(iterations):
        with torch.cuda.stream(s_train):
            dd, ll = aug.tensors_nowait()
            train_step(dd, ll)
        w0[i].record(s_train)  # step i done; from here the train stream waits for m'_{i+1}
        aug = eng.update((data_ring[(i + 1) % B], label_ring[(i + 1) % B]), stream=s_eng, consumer=s_train)
        w1[i].record(s_train)
    e1.record(s_train)
    torch.cuda.synchronize(dev)
    iteration_ms = e0.elapsed_time(e1) / iterations
    wait_ms = sum(w0[i].elapsed_time(w1[i]) for i in range(iterations)) / iterations
    return overlap_result(train_ms, background_ms, wait_ms, iteration_ms, iterations,
                          max(0.0, iteration_ms - train_ms))
