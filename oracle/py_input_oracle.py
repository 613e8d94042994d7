"""TEST INFRASTRUCTURE — CPU restatement of the input side.

Checker only (tests/ may import it; the product path never does). Restates, in numpy and
plain Python:
  * load_dataset / DRDS parsing  proj/src/scenario/dataset.cpp:102-143 (format: dataset.hpp:10-17)
  * train/eval_indices_of        proj/src/scenario/dataset.cpp:48-64
  * gather                       proj/src/scenario/dataset.cpp:66-72
  * make_schedule                proj/src/scenario/schedule.cpp:10-35
  * shard_batches                proj/src/scenario/schedule.cpp:37-62
  * lockstep_batches             proj/src/scenario/schedule.cpp:64-69
Parity status: pinned — tests/test_input_cpu.py checks every function here against the
reference itself (oracle/_ref/libdrb_ref.so, built from the unmodified sources) and the
committed fixture tests/golden/drds_small.* written by the reference's write_dataset.
"""
from __future__ import annotations

import os
from typing import List, Optional, Tuple

import numpy as np

_PHI = 0x9E3779B97F4A7C15
_M = (1 << 64) - 1
DATA_SHUFFLE = 4  # rng.hpp purpose::data_shuffle


class io_error(Exception):
    pass


def _mix64(z: int) -> int:
    z = (z + _PHI) & _M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M
    return z ^ (z >> 31)


class keyed_stream:
    """rng_stream::keyed(seed, worker, purpose, k1, k2) (rng.cpp:19-53)."""

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


def load_dataset(path: str):
    """Returns (features f32 [count, dim], labels u32 [count], n_classes, train, eval)."""
    try:
        raw = open(path, "rb").read()
    except OSError:
        raise io_error(f"cannot open dataset file: {path}")
    if len(raw) < 4 or raw[:4] != b"DRDS":
        raise io_error(f"not a dataset file (bad magic): {path}")
    if len(raw) < 6:
        raise io_error(f"truncated dataset file: {path}")
    version = int.from_bytes(raw[4:6], "little")
    if version != 1:
        raise io_error(f"unsupported dataset version {version}: {path}")
    if len(raw) < 22:
        raise io_error(f"truncated dataset file: {path}")
    count = int.from_bytes(raw[6:14], "little")
    dim = int.from_bytes(raw[14:18], "little")
    n_classes = int.from_bytes(raw[18:22], "little")
    rec = (dim + 1) * 4
    avail = min(count, (len(raw) - 22) // rec)
    words = np.frombuffer(raw, dtype="<u4", count=avail * (dim + 1), offset=22).reshape(avail, dim + 1)
    labels = words[:, dim].astype(np.uint32)
    bad = np.nonzero(labels >= n_classes)[0]
    if len(bad):
        raise io_error(f"dataset label out of range at record {int(bad[0])}: {path}")
    if avail < count:
        raise io_error(f"truncated dataset file: {path}")
    features = words[:, :dim].copy().view(np.float32)
    train, ev = count, 0
    if os.path.exists(path + ".split"):
        tok = open(path + ".split").read().split()
        try:
            ok = len(tok) >= 4 and tok[0] == "train" and tok[2] == "eval"
            train, ev = int(tok[1]), int(tok[3])
            ok = ok and train + ev == count
        except ValueError:
            ok = False
        if not ok:
            raise io_error(f"bad split sidecar: {path}.split")
    return features, labels, n_classes, train, ev


def indices_of(labels: np.ndarray, train: int, classes, eval_set: bool) -> np.ndarray:
    lo, hi = (train, len(labels)) if eval_set else (0, train)
    sel = np.isin(labels[lo:hi], np.asarray(list(classes), dtype=np.uint32))
    return (np.nonzero(sel)[0] + lo).astype(np.uint64)


def gather(features: np.ndarray, labels: np.ndarray, idx) -> Tuple[np.ndarray, np.ndarray]:
    idx = np.asarray(idx, dtype=np.int64)
    return features[idx], labels[idx]


def make_schedule(n_classes: int, n_tasks: int, seed: int) -> List[List[int]]:
    if n_tasks == 0 or n_tasks > n_classes:
        raise ValueError("make_schedule: need 1 <= T <= K")
    classes = list(range(n_classes))
    rng = keyed_stream(seed, 0, DATA_SHUFFLE, 0xABCD, 0)
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


def shard_batches(task_data, worker: int, n_workers: int, batch: int, seed: int, task_index: int,
                  epoch: int) -> List[List[int]]:
    if worker >= n_workers:
        raise ValueError("shard_batches: worker id out of range")
    order = [int(x) for x in task_data]
    rng = keyed_stream(seed, 0, DATA_SHUFFLE, task_index + 1, epoch + 1)
    for i in range(len(order), 1, -1):
        j = rng.bounded(i)
        order[i - 1], order[j] = order[j], order[i - 1]
    shard = order[worker::n_workers]
    return [shard[s:s + batch] for s in range(0, len(shard), batch)]


def lockstep_batches(task_size: int, n_workers: int, batch: int) -> int:
    return (task_size // n_workers + batch - 1) // batch


def write_dataset(path: str, features: np.ndarray, labels: np.ndarray, n_classes: int,
                  train: Optional[int] = None, eval_count: int = 0) -> None:
    """write_dataset (dataset.cpp:74-100) restated: test-input writer."""
    features = np.ascontiguousarray(features, dtype=np.float32)
    count, dim = features.shape
    rec = np.empty((count, dim + 1), dtype="<u4")
    rec[:, :dim] = features.view(np.uint32)
    rec[:, dim] = labels
    with open(path, "wb") as f:
        f.write(b"DRDS" + (1).to_bytes(2, "little") + count.to_bytes(8, "little") +
                dim.to_bytes(4, "little") + n_classes.to_bytes(4, "little"))
        f.write(rec.tobytes())
    with open(path + ".split", "w") as f:
        f.write(f"train {count if train is None else train}\neval {eval_count}\n")


# ---- the reference itself (oracle/_ref), for pinning this restatement ----
#
# The reference .so resolves its C++ runtime symbols from the process; once numpy's bundled
# libraries are loaded first, its iostream parsing and libm draws misbehave (a bad-split
# verdict on a valid sidecar, a crash in synth_dataset). Every reference call therefore runs
# in a child process that loads the .so BEFORE numpy (oracle/ref_input_child.py).

REF_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref", "libdrb_ref.so")
_CHILD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_input_child.py")


def ref_batch(requests):
    """Run [{"op": ..., ...}, ...] through the reference in a child; returns the results."""
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, _CHILD], input=json.dumps(requests), capture_output=True, text=True,
                         check=True).stdout
    return json.loads(out)


def ref_load(path: str):
    """The reference's load_dataset: (features, labels, n_classes, train, eval) or io_error."""
    r = ref_batch([{"op": "load", "path": path}])[0]
    if "io_error" in r:
        raise io_error(r["io_error"])
    feats = np.frombuffer(bytes.fromhex(r["features"]), dtype="<f4").reshape(r["count"], r["dim"])
    return feats, np.asarray(r["labels"], np.uint32), r["n_classes"], r["train"], r["eval"]
