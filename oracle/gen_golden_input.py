#!/usr/bin/env python3
"""TEST INFRASTRUCTURE: write the input-side fixtures from the REFERENCE itself.

Run here (the reference is not on the GPU box):  python oracle/gen_golden_input.py
Outputs (the reference's own synth_dataset + write_dataset, proj/src/scenario/dataset.cpp):
  tests/golden/drds_small.drds(+.split)   K=5, 8 per class, feature_dim 12 (48 B rows)
  tests/golden/drds_odd.drds(+.split)     K=3, 6 per class, feature_dim 7 (28 B rows)
  tests/golden/input.json                 the reference's make_schedule / shard_batches /
                                          lockstep_batches outputs for a few cases
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.py_input_oracle import ref_batch  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
SCHEDULES = [(10, 4, 1), (100, 4, 1), (1000, 4, 7), (7, 7, 3)]
SHARDS = [(97, 0, 4, 8, 1, 0, 0), (97, 3, 4, 8, 1, 2, 5), (1000, 1, 2, 56, 9, 1, 1), (5, 4, 8, 2, 1, 0, 0)]
LOCKSTEP = [(97, 4, 8), (1000, 8, 56), (3, 4, 2)]


def main() -> None:
    req = [{"op": "synth", "path": os.path.join(OUT, "drds_small.drds"), "K": 5, "per_class": 8, "dim": 12,
            "sep": 4.0, "seed": 11},
           {"op": "synth", "path": os.path.join(OUT, "drds_odd.drds"), "K": 3, "per_class": 6, "dim": 7,
            "sep": 3.0, "seed": 12}]
    req += [{"op": "schedule", "K": K, "T": T, "seed": s} for K, T, s in SCHEDULES]
    req += [{"op": "shard", "task_data": [i * 3 + 1 for i in range(n)], "worker": w, "n_workers": nw, "batch": b,
             "seed": s, "task": t, "epoch": e} for n, w, nw, b, s, t, e in SHARDS]
    req += [{"op": "lockstep", "n": n, "n_workers": nw, "batch": b} for n, nw, b in LOCKSTEP]
    res = ref_batch(req)
    assert res[0]["rc"] == 0 and res[1]["rc"] == 0
    res = res[2:]
    out = {"schedules": [], "shards": [], "lockstep": []}
    for (K, T, seed), r in zip(SCHEDULES, res):
        out["schedules"].append({"K": K, "T": T, "seed": seed, **r})
    res = res[len(SCHEDULES):]
    for (n, w, nw, b, seed, t, e), r in zip(SHARDS, res):
        assert r["rc"] == 0
        out["shards"].append({"task_data": "arange(n)*3+1", "n": n, "worker": w, "n_workers": nw, "batch": b,
                              "seed": seed, "task": t, "epoch": e, "shard": r["shard"], "n_batches": r["n_batches"]})
    res = res[len(SHARDS):]
    for (n, nw, b), r in zip(LOCKSTEP, res):
        out["lockstep"].append({"n": n, "n_workers": nw, "batch": b, "batches": r})
    with open(os.path.join(OUT, "input.json"), "w") as f:
        json.dump(out, f, indent=0)


if __name__ == "__main__":
    main()
