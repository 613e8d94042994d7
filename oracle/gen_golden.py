#!/usr/bin/env python3
"""TEST INFRASTRUCTURE: regenerate tests/golden/*.json from the REFERENCE itself
(oracle/_ref/libdrb_ref.so = the unmodified /root/reference sources + ref_capi.cpp).

Run here (the reference is not on the GPU box):  python oracle/gen_golden.py
Outputs:
  tests/golden/kat.json     KAT1-KAT6 + extra rng/swor/plan vectors
  tests/golden/replay.json  per-step sha256 of every rank's m'_i (bytes ++ labels ++ count)
                            under the synchronous replay, for small configs at N = 1, 2, 4, 8
  tests/golden/bias.json    the bias test of proj/tests/acceptance.cpp:205-227 (K=10, r=7,
                            seed=5, 1e5 draws; N=2 fill 40, N=4 fill 80, local-only control):
                            sha256 of the reference's per-slot counts, its chi-square
                            statistic and p-value (make_bias_report)
  tests/golden/read_slots.json  read_slots of the reference's rehearsal_buffer after update
                            rounds: statuses, labels, sha256 of the returned bytes, and the
                            substitute stream's next draw (exact / substituted / empty paths)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.py_oracle import Backend, CANDIDATE, EVICTION, GLOBAL_SAMPLING  # noqa: E402
from paper_2406_03285_b200.workload import stream_spec  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

# (name, N, K, cap, S, b, c, r, seed, T, steps_per_task, steps, short-batch pattern or None)
REPLAY_CONFIGS = [
    ("c1_like_n1", 1, 10, 100, 256, 64, 14, 8, 1, 1, 10**9, 220, None),
    ("engine_cfg_n2", 2, 4, 16, 12, 8, 4, 7, 77, 1, 10**9, 80, None),
    ("ci_n2", 2, 20, 6, 64, 56, 14, 7, 3, 4, 15, 120, None),
    ("ci_n4", 4, 12, 5, 32, 24, 14, 7, 5, 3, 10, 100, None),
    ("ci_n8", 8, 16, 4, 16, 16, 6, 9, 9, 2, 12, 90, None),
    ("short_n2", 2, 6, 3, 16, 12, 5, 6, 11, 1, 10**9, 60, [12, 3, 0, 12, 1]),
    ("exhaust_n4", 4, 3, 2, 8, 4, 4, 40, 13, 1, 10**9, 30, None),
    ("big_r_n2", 2, 8, 8, 16, 40, 33, 33, 17, 2, 20, 60, None),
]


def digest(aug: np.ndarray, lab: np.ndarray, count: int) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(aug[:count]).tobytes())
    h.update(np.ascontiguousarray(lab[:count].astype(np.uint32)).tobytes())
    h.update(np.uint32(count).tobytes())
    return h.hexdigest()


def replay_digests(be: Backend, cfg):
    name, N, K, cap, S, b, c, r, seed, T, spt, steps, pattern = cfg
    spec = stream_spec(K, T, b, S, steps_per_task=spt, seed=seed)
    rp = be.replay(N, K, cap, S, c, r, seed)
    out = []
    for i in range(steps):
        n = pattern[i % len(pattern)] if pattern else b
        data = np.stack([spec.payload(w, i, n) for w in range(N)])
        labs = np.stack([spec.labels(w, i, n) for w in range(N)])
        aug, al, cnt = rp.step(data, labs)
        out.append([digest(aug[w], al[w], int(cnt[w])) for w in range(N)])
    return out


def kat(be: Backend):
    k = {}
    k["kat1_next_u64_seed1_w0_candidate"] = [hex(int(x)) for x in be.rng_next(1, 0, CANDIDATE, 4)]
    k["kat2_bounded100_seed1_w0_eviction"] = be.rng_bounded(1, 0, EVICTION, 100, 8).tolist()
    k["kat3_swor_64_14"] = be.swor(64, 14, 1).tolist()
    k["kat4_keyed_7e"] = [hex(int(x)) for x in be.rng_next(1, 0, GLOBAL_SAMPLING, 2, keyed=True, k1=0x7E)]
    k["kat5_plan"] = be.plan(8, np.array([[4, 0, 6], [10, 3, 0]]), 1).tolist()
    # extra vectors: rejection-heavy bounds, many (n,k), plans with carried counters
    k["bounded_big"] = {str(bd): [str(int(x)) for x in be.rng_bounded(3, 1, GLOBAL_SAMPLING, bd, 64)]
                        for bd in (2**63 + 1, 2**64 - 3, 3 * 2**62)}
    rng = np.random.default_rng(0)
    sw = []
    for _ in range(40):
        n, kk, seed = int(rng.integers(1, 300)), int(rng.integers(0, 50)), int(rng.integers(0, 2**31))
        sw.append({"n": n, "k": kk, "seed": seed, "out": be.swor(n, kk, seed).tolist()})
    k["swor_random"] = sw
    pl = []
    for _ in range(30):
        nw, nk = int(rng.integers(1, 9)), int(rng.integers(1, 30))
        occ = rng.integers(0, 6, (nw, nk)).astype(np.uint32)
        want, seed = int(rng.choice([1, 7, 8, 28, 33, 64])), int(rng.integers(0, 2**31))
        rounds = be.plan(want, occ, seed, 0, GLOBAL_SAMPLING, rounds=3)
        pl.append({"occ": occ.tolist(), "want": want, "seed": seed, "rounds": [x.tolist() for x in rounds]})
    k["plan_random"] = pl
    # KAT6: config-1 single rank, label (64i+j)%10, features[0] = 64i+j (float32)
    K, cap, b, c, r, S = 10, 100, 64, 14, 8, 16
    rp = be.replay(1, K, cap, S, c, r, 1)
    plans, f0 = [], []
    for i in range(200):
        feats = np.zeros((b, S // 4), np.float32)
        feats[:, 0] = 64 * i + np.arange(b)
        lab = ((64 * i + np.arange(b)) % 10).astype(np.uint32)
        aug, al, cnt = rp.step(feats.view(np.uint8).reshape(1, b, S), lab[None])
        plans.append(rp.last_plan(0)[:, 1:].tolist())
        if i > 0:
            f0.append(aug[0, b:cnt[0], :4].copy().view(np.float32)[:, 0].astype(int).tolist())
    feats = np.zeros((b, S // 4), np.float32)
    aug, al, cnt = rp.step(feats.view(np.uint8).reshape(1, b, S), np.zeros((1, b), np.uint32))
    f0.append(aug[0, b:cnt[0], :4].copy().view(np.float32)[:, 0].astype(int).tolist())
    k["kat6_plans_cls_slot"] = plans
    k["kat6_reps_f0"] = f0  # f0[i] = reps of round i (delivered in m'_{i+1})
    return k


BIAS_CONFIGS = [("n2", 2, 40, False), ("n4", 4, 80, False), ("control", 2, 40, True)]
BIAS_K, BIAS_R, BIAS_SEED = 10, 7, 5


def bias(be, draws):
    from oracle.py_oracle import bias_counts, bias_view, reference_bias_report
    out = {}
    for name, N, fill, control in BIAS_CONFIGS:
        occ = bias_view(N, BIAS_K, fill)
        counts = bias_counts(be, occ, BIAS_R, BIAS_SEED, draws, control)
        st, p = reference_bias_report(counts, BIAS_R, draws)
        out[name] = {"N": N, "K": BIAS_K, "r": BIAS_R, "seed": BIAS_SEED, "fill": fill, "local_only": control,
                     "draws": draws, "occ": occ.tolist(),
                     "counts_sha256": hashlib.sha256(counts.astype("<u8").tobytes()).hexdigest(),
                     "counts_head": counts[:16].tolist(), "statistic": st, "p_value": p}
    return out


# read_slots (rehearsal_buffer.cpp:88-142) against the reference's own buffer: (name, K, cap, S,
# rounds, n, c, seed, keyed, purpose, k1, k2). The requests of every scenario mix exact reads,
# stale indices (slot >= occupancy: a substitute drawn within the class), empty classes and
# classes >= K (the whole-buffer flat fallback), so every branch consumes the stream. The
# last field is the task count of the input stream (2: half the classes never stored).
READ_SLOTS_CONFIGS = [
    ("serve_subst_keyed", 6, 4, 32, 3, 8, 5, 11, 1, 6, 0x5E, 0, 1),  # engine.cpp:33-35 serve stream
    ("slot_subst_plain", 10, 3, 16, 6, 12, 9, 4, 0, 6, 0, 0, 1),      # engine.cpp:31 substitute stream
    ("full_classes", 4, 2, 48, 8, 16, 12, 7, 1, 6, 0x5E, 0, 1),
    ("half_empty", 8, 4, 32, 4, 8, 6, 13, 1, 6, 0x5E, 0, 2),
    ("nothing_stored", 5, 3, 16, 0, 8, 4, 2, 1, 6, 0x5E, 0, 1),
]


def read_slots_requests(K, cap, occ, seed):
    rng = np.random.default_rng(seed)
    req = []
    for k in range(K + 2):  # two classes past K
        for _ in range(3):
            o = int(occ[k]) if k < K else 0
            if o and rng.random() < 0.4:
                req.append((k, int(rng.integers(0, o))))           # exact
            else:
                req.append((k, int(rng.integers(o, cap + 3))))     # stale / empty / out of range
    return req


def read_slots_golden():
    from oracle.py_oracle import reference_read_slots
    out = {}
    for name, K, cap, S, rounds, n, c, seed, keyed, purpose, k1, k2, T in READ_SLOTS_CONFIGS:
        spec = stream_spec(K, T, n, S, steps_per_task=10**9, seed=seed)
        batches = np.stack([spec.payload(0, i, n) for i in range(rounds)]) if rounds else np.zeros((0, n, S), np.uint8)
        labels = np.stack([spec.labels(0, i, n) for i in range(rounds)]) if rounds else np.zeros((0, n), np.uint32)
        # occupancy first (a pass with no requests), then the requests built against it
        _, _, _, _, occ = reference_read_slots(K, cap, S, batches, labels, c, seed, keyed, purpose, k1, k2, [])
        req = read_slots_requests(K, cap, occ, seed)
        d, lab, st, nxt, occ = reference_read_slots(K, cap, S, batches, labels, c, seed, keyed, purpose, k1, k2, req)
        out[name] = {"config": dict(K=K, cap=cap, S=S, rounds=rounds, n=n, c=c, seed=seed, keyed=keyed,
                                    purpose=purpose, k1=k1, k2=k2, T=T),
                     "requests": req, "occ": occ.tolist(), "status": st.tolist(), "labels": lab.tolist(),
                     "bytes_sha256": hashlib.sha256(np.ascontiguousarray(d).tobytes()).hexdigest(),
                     "sub_next_u64": hex(nxt)}
    return out


def main():
    be = Backend("reference")
    os.makedirs(OUT, exist_ok=True)
    if len(sys.argv) > 1 and sys.argv[1] == "read_slots":
        with open(os.path.join(OUT, "read_slots.json"), "w") as f:
            json.dump(read_slots_golden(), f, indent=1)
        print("wrote read_slots.json")
        return
    with open(os.path.join(OUT, "kat.json"), "w") as f:
        json.dump(kat(be), f)
    rep = {}
    for cfg in REPLAY_CONFIGS:
        rep[cfg[0]] = {"config": dict(zip(["name", "N", "K", "cap", "S", "b", "c", "r", "seed", "T",
                                           "steps_per_task", "steps", "pattern"], cfg)),
                       "digests": replay_digests(be, cfg)}
    with open(os.path.join(OUT, "replay.json"), "w") as f:
        json.dump(rep, f)
    with open(os.path.join(OUT, "bias.json"), "w") as f:
        json.dump({"draws_1e5": bias(be, 100000), "draws_2000": bias(be, 2000)}, f, indent=1)
    with open(os.path.join(OUT, "read_slots.json"), "w") as f:
        json.dump(read_slots_golden(), f, indent=1)
    print("wrote", os.listdir(OUT))


if __name__ == "__main__":
    main()
