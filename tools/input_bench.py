"""Input-side throughput: DRDS file -> HBM load, and the device gather that
produces m (c2 shape: rows of 150528 B = 37632 f32, b = 56), timed with CUDA events on the
gather's stream; the dataset (602 MB) is larger than L2, indices are fresh random draws."""
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_03285_b200 import dataset as D  # noqa: E402


def write_dataset(path, features, labels, n_classes):
    """A DRDS file (proj/src/scenario/dataset.hpp:10-17) of the synthetic input, all train."""
    count, dim = features.shape
    rec = np.empty((count, dim + 1), dtype="<u4")
    rec[:, :dim] = features.view(np.uint32)
    rec[:, dim] = labels
    with open(path, "wb") as f:
        f.write(b"DRDS" + (1).to_bytes(2, "little") + count.to_bytes(8, "little") + dim.to_bytes(4, "little") +
                n_classes.to_bytes(4, "little"))
        f.write(rec.tobytes())

count, dim, b, iters = 4000, 37632, 56, 200
rng = np.random.default_rng(0)
feats = rng.integers(0, 2**32, (count, dim), dtype=np.uint32).view(np.float32)
labels = rng.integers(0, 100, count).astype(np.uint32)
path = os.path.join(tempfile.mkdtemp(), "c2.drds")
write_dataset(path, feats, labels, 100)
fbytes = os.path.getsize(path)
os.system(f"cat {path} > /dev/null")
torch.zeros(1, device="cuda:0")  # CUDA context up before the load is timed  # page cache warm: time the parse + H2D + split, not the disk
t = time.perf_counter()
ds = D.load_dataset(path, 0)
load_s = time.perf_counter() - t
idx = [torch.randint(0, count, (b,), device="cuda:0") for _ in range(iters)]
out = torch.empty((b, dim * 4), dtype=torch.uint8, device="cuda:0")
lab = torch.empty(b, dtype=torch.int32, device="cuda:0")
for i in range(5):
    ds.gather(idx[i], out=out, out_labels=lab)
torch.cuda.synchronize()
# the gathers captured in one CUDA graph: the GPU time of the kernels, not Python's launch rate
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for i in range(iters):
            ds.gather(idx[i], out=out, out_labels=lab)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / iters
alg = 2 * b * dim * 4 + 8 * b + 8 * b  # row read + row write + index + labels
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
print(json.dumps({"load": {"file_bytes": fbytes, "seconds": round(load_s, 3), "GB_per_s": round(fbytes / load_s / 1e9, 2)},
                  "gather": {"rows": b, "row_bytes": dim * 4, "us_per_gather": round(us, 2),
                             "GB_per_s": round(alg / us / 1e3, 1), "algorithmic_bytes": alg},
                  "peaks": {k: v for k, v in peak.items() if "hbm" in k.lower() or "copy" in k.lower()}}))
assert ds.device_error() == 0
