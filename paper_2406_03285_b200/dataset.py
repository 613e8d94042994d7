"""Input side of the hot path: the producer of m.

Python mirror of the reference's scenario API over the C ABI (include/drb_rb.h, drb_ds_* /
drb_make_schedule / drb_shard_batches / drb_lockstep_batches):

  dataset, load_dataset        proj/src/scenario/dataset.hpp:10-40, dataset.cpp:102-143
  synth_dataset                proj/src/scenario/dataset.cpp:145-205
  dataset.train_indices_of     proj/src/scenario/dataset.cpp:48-55
  dataset.eval_indices_of      proj/src/scenario/dataset.cpp:57-64
  dataset.gather               proj/src/scenario/dataset.cpp:66-72 (on the device: returns
                               the rehearsal buffer's m layout, u8 [n, S] + int32 labels [n])
  task_schedule, make_schedule proj/src/scenario/schedule.hpp:10-25, schedule.cpp:10-35
  shard_batches                proj/src/scenario/schedule.cpp:37-62
  lockstep_batches             proj/src/scenario/schedule.cpp:64-69

The dataset lives in HBM after load_dataset; a training loop gathers each batch on the
device and hands it straight to engine.update / rehearsal_buffer.update_buffer.
Errors: io_error for every load failure (dataset.cpp's io_error), config_error from
make_schedule, usage_error from shard_batches (schedule.cpp:44-45).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .rehearsal import _stream_arg, _view

io_error = _lib.io_error


class dataset:
    """A DRDS dataset resident in HBM: features [count][feature_dim] f32 (SoA) + u32 labels."""

    def __init__(self, handle: C.c_void_p, device: int):
        self._h = handle
        self.device = device
        cnt, tr, ev = C.c_uint64(), C.c_uint64(), C.c_uint64()
        dim, k = C.c_uint32(), C.c_uint32()
        check(lib.drb_ds_info(self._h, C.byref(cnt), C.byref(dim), C.byref(k), C.byref(tr), C.byref(ev)))
        self.feature_dim, self.n_classes = dim.value, k.value
        self.train_count, self.eval_count = tr.value, ev.value
        self._count = cnt.value

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and lib is not None:
            lib.drb_ds_destroy(h)

    def size(self) -> int:
        return self._count

    @property
    def sample_bytes(self) -> int:
        return self.feature_dim * 4

    def features(self) -> torch.Tensor:
        """Zero-copy view of the device features, f32 [count, feature_dim]."""
        fp, lp = C.c_void_p(), C.c_void_p()
        check(lib.drb_ds_device_views(self._h, C.byref(fp), C.byref(lp)))
        return _view(fp.value or 0, (self._count, self.feature_dim), "<f4", self.device, self)

    def labels(self) -> torch.Tensor:
        fp, lp = C.c_void_p(), C.c_void_p()
        check(lib.drb_ds_device_views(self._h, C.byref(fp), C.byref(lp)))
        return _view(lp.value or 0, (self._count,), "<i4", self.device, self)

    def _indices_of(self, classes: Sequence[int], eval_set: int) -> np.ndarray:
        cls = np.ascontiguousarray(np.asarray(list(classes), dtype=np.uint32))
        n = C.c_uint64()
        check(lib.drb_ds_indices_of(self._h, cls.ctypes.data, len(cls), eval_set, None, 0, C.byref(n)))
        out = np.empty(n.value, np.uint64)
        check(lib.drb_ds_indices_of(self._h, cls.ctypes.data, len(cls), eval_set, out.ctypes.data, n.value,
                                    C.byref(n)))
        return out

    def train_indices_of(self, classes: Sequence[int]) -> np.ndarray:
        return self._indices_of(classes, 0)

    def eval_indices_of(self, classes: Sequence[int]) -> np.ndarray:
        return self._indices_of(classes, 1)

    def gather(self, indices, out: torch.Tensor = None, out_labels: torch.Tensor = None):
        """m = records `indices` in order: (u8 [n, S], int32 labels [n]) on this dataset's
        device, ordered on the current stream. indices: host sequence or device int64/uint64."""
        dev = torch.device("cuda", self.device)
        if isinstance(indices, torch.Tensor) and indices.is_cuda:
            idx = indices.to(torch.int64).contiguous()
        else:
            idx = torch.as_tensor(np.asarray(indices, dtype=np.int64).reshape(-1)).to(dev, non_blocking=True)
        n = idx.numel()
        if out is None:
            out = torch.empty((n, self.sample_bytes), dtype=torch.uint8, device=dev)
        if out_labels is None:
            out_labels = torch.empty(n, dtype=torch.int32, device=dev)
        if out.numel() < n * self.sample_bytes or out_labels.numel() < n:
            raise _lib.usage_error("gather: output buffers too small")
        stream = torch.cuda.current_stream(dev)
        check(lib.drb_ds_gather(self._h, C.c_void_p(idx.data_ptr()), n, C.c_void_p(out.data_ptr()),
                                C.c_void_p(out_labels.data_ptr()), _stream_arg(stream)))
        idx.record_stream(stream)
        return out, out_labels

    def device_error(self) -> int:
        e = C.c_uint32()
        check(lib.drb_ds_device_error(self._h, C.byref(e)))
        return e.value


def load_dataset(path: str, device: int = 0) -> dataset:
    h = C.c_void_p()
    check(lib.drb_ds_load(str(path).encode(), device, C.byref(h)))
    return dataset(h, device)


def synth_dataset(n_classes: int, per_class: int, feature_dim: int, separation: float, seed: int,
                  device: int = 0) -> dataset:
    """synth_dataset (proj/src/scenario/dataset.cpp:145-205), bit-identical, resident in HBM."""
    h = C.c_void_p()
    check(lib.drb_ds_synth(n_classes, per_class, feature_dim, float(separation), seed, device, C.byref(h)))
    return dataset(h, device)


@dataclass
class task_schedule:
    tasks: List[List[int]] = field(default_factory=list)
    epochs_per_task: int = 1


def make_schedule(n_classes: int, n_tasks: int, seed: int, epochs_per_task: int = 1) -> task_schedule:
    classes = np.empty(max(n_classes, 1), np.uint32)
    sizes = np.empty(max(n_tasks, 1), np.uint32)
    check(lib.drb_make_schedule(n_classes, n_tasks, seed, classes.ctypes.data, sizes.ctypes.data))
    tasks, cur = [], 0
    for t in range(n_tasks):
        tasks.append([int(c) for c in classes[cur:cur + sizes[t]]])
        cur += int(sizes[t])
    return task_schedule(tasks, epochs_per_task)


def shard_batches(task_data, worker: int, n_workers: int, batch_size: int, seed: int, task_index: int,
                  epoch: int) -> List[np.ndarray]:
    td = np.ascontiguousarray(np.asarray(task_data, dtype=np.uint64).reshape(-1))
    cap = (len(td) + n_workers - 1) // n_workers if n_workers else 0
    out = np.empty(max(cap, 1), np.uint64)
    n = C.c_uint64()
    check(lib.drb_shard_batches(td.ctypes.data, len(td), worker, n_workers, batch_size, seed, task_index, epoch,
                                out.ctypes.data, cap, C.byref(n)))
    shard = out[:n.value]
    return [shard[s:s + batch_size] for s in range(0, len(shard), batch_size)]


def lockstep_batches(task_size: int, n_workers: int, batch_size: int) -> int:
    out = C.c_uint64()
    check(lib.drb_lockstep_batches(task_size, n_workers, batch_size, C.byref(out)))
    return out.value


def epoch_batches(ds: dataset, task_data, worker: int, n_workers: int, batch_size: int, seed: int,
                  task_index: int, epoch: int):
    """The producer side of epoch_driver::run (proj/src/trainer/trainer.cpp:94-106): this
    worker's shard for (task, epoch), lockstep_batches steps, each yielded as a device m
    (u8 [n, S], int32 labels [n]) ready for engine.update. The shard's indices go to HBM
    once per epoch; every step is one device gather into a fresh pair of tensors."""
    batches = shard_batches(task_data, worker, n_workers, batch_size, seed, task_index, epoch)
    steps = lockstep_batches(len(task_data), n_workers, batch_size)
    if steps == 0:
        return
    dev = torch.device("cuda", ds.device)
    flat = torch.as_tensor(np.concatenate(batches[:steps]).astype(np.int64)).to(dev)
    pos = 0
    for b in batches[:steps]:
        yield ds.gather(flat[pos:pos + len(b)])
        pos += len(b)
