#!/usr/bin/env python3
"""Overlap of the rehearsal engine with a real training step on one GPU (
the reference's overlap bench, proj/src/runner/overlap.cpp:39-120, criterion 5 of
proj/tests/acceptance.cpp:229-256). Prints one JSON line.
Usage: python tools/overlap_bench.py [--config c2] [--iters 600] [--width 64]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2406_03285_b200 as drb  # noqa: E402
from paper_2406_03285_b200.overlap import conv_classifier, make_train_step, run_overlap_bench  # noqa: E402
from paper_2406_03285_b200.workload import device_ring, stream_spec  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--iters", type=int, default=600)
    ap.add_argument("--width", type=int, default=64)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    K, cap, S, b, r, c = cfg["K"], cfg["cap"], cfg["S"], cfg["b"], cfg["r"], cfg["c"]
    hw, ch = (224, 3) if S == 224 * 224 * 3 else (int(round((S // 3) ** 0.5)), 3)
    spec = stream_spec(K, cfg["T"], b, S, steps_per_task=100, seed=9)
    buf = drb.rehearsal_buffer(K, cap, S, max_batch=b, candidate_count=c, rep_count=r, seed=9)
    eng = drb.engine(buf)
    eng.start()
    data, lab = device_ring(spec, 0, 16, "cuda:0")
    eng.run(data, lab, 400)  # fill the buffers first (steady state: m' has b + r rows)
    torch.cuda.synchronize()
    model = conv_classifier(hw, ch, K, width=a.width).cuda().to(memory_format=torch.channels_last)
    res = run_overlap_bench(eng, data, lab, make_train_step(model), a.iters)
    eng.shutdown()
    print(json.dumps({"bench": "overlap", "config": cfg["workload"], "iterations": res.iterations,
                      "train_cost_ms": res.train_cost_ms, "background_ms": res.background_ms,
                      "mean_wait_ms": res.mean_wait_ms, "mean_iteration_ms": res.mean_iteration_ms,
                      "wait_fraction": res.wait_fraction,
                      "train_over_background": res.train_cost_ms / res.background_ms,
                      "criterion": "wait < 5% of the iteration with train >= 10x background "
                                   "(acceptance.cpp:229-256)"}))


if __name__ == "__main__":
    main()
