"""TEST INFRASTRUCTURE — numpy/ctypes wrapper over the CPU checkers.

Two interchangeable backends with identical signatures:
  * ``port``      — oracle/liboracle.so, the clean-room C restatement (drb_oracle.c);
                    always buildable, travels to the GPU box as a built .so.
  * ``reference`` — oracle/_ref/libdrb_ref.so, the unmodified reference sources compiled
                    by oracle/Makefile plus our harness ref_capi.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm may
import this module, and only as the checker or the CPU baseline — never as a product
path. Parity status: pinned (see drb_oracle.h and tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libdrb_ref.so")

# purposes, proj/src/core/rng.hpp:18-26
CANDIDATE, EVICTION, GLOBAL_SAMPLING, DATA_SHUFFLE, MODEL_INIT, SLOT_SUBSTITUTE, SYNTH = range(1, 8)

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def _nullable(nd):
    """An ndpointer argtype that also accepts None (NULL)."""
    return type(nd.__name__ + "_or_null", (nd,),
                {"from_param": classmethod(lambda cls, obj: None if obj is None else nd.from_param(obj))})


def _bind(lib, prefix):
    u32, u64, i32, vp = C.c_uint32, C.c_uint64, C.c_int, C.c_void_p
    sig = {
        "rng_next": (i32, [u64, u32, u32, i32, u64, u64, u64, _u64p]),
        "rng_bounded": (i32, [u64, u32, u32, i32, u64, u64, u64, u64, _u64p]),
        "swor": (i32, [u64, u64, u64, u32, u32, _u64p, _u64p]),
        "plan": (i32, [u64, u32, u32, _u32p, u64, u32, u32, u32, _u32p, _u64p]),
        "replay_create": (vp, [u32, u32, u32, u64, u32, u32, u64]),
        "replay_destroy": (None, [vp]),
        "replay_step": (i32, [vp, _u8p, _u32p, u32, _u8p, _u32p, _u32p]),
        "replay_last_plan": (u32, [vp, u32, _u32p]),
        "replay_last_report": (i32, [vp, u32, _u32p, _u32p, _u32p]),
        "replay_dump": (i32, [vp, u32, _u32p, _u64p, _nullable(_u8p), _nullable(_u32p)]),
    }
    fns = {}
    for name, (res, args) in sig.items():
        f = getattr(lib, prefix + name)
        f.restype = res
        f.argtypes = args
        fns[name] = f
    return fns


class Backend:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(f"{kind} oracle library missing: {path} (run `make -C oracle{' ref' if kind != 'port' else ''}`)")
        self.lib = C.CDLL(path)
        self.f = _bind(self.lib, "or_" if kind == "port" else "ref_")
        if kind == "reference":
            eb = self.lib.ref_engine_bench
            eb.restype = C.c_int
            eb.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32,
                           C.c_uint32, C.c_uint64, _u8p, _u32p, C.c_uint32, C.c_uint32, C.c_uint32,
                           C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        else:
            rc = self.lib.or_replay_counters
            rc.restype = C.c_int
            rc.argtypes = [C.c_void_p, C.c_uint32, _u64p]

    # --- S0 ---------------------------------------------------------------------------
    def rng_next(self, seed, worker, purpose, n, keyed=False, k1=0, k2=0):
        out = np.zeros(n, np.uint64)
        self.f["rng_next"](seed, worker, purpose, int(keyed), k1, k2, n, out)
        return out

    def rng_bounded(self, seed, worker, purpose, bound, n, keyed=False, k1=0, k2=0):
        out = np.zeros(n, np.uint64)
        self.f["rng_bounded"](seed, worker, purpose, int(keyed), k1, k2, bound, n, out)
        return out

    # --- S1 ---------------------------------------------------------------------------
    def swor(self, n, k, seed, worker=0, purpose=CANDIDATE):
        out = np.zeros(max(n, 1), np.uint64)
        kk = np.zeros(1, np.uint64)
        self.f["swor"](n, k, seed, worker, purpose, out, kk)
        return out[: int(kk[0])]

    # --- S4 ---------------------------------------------------------------------------
    def plan(self, want, occ, seed, worker=0, purpose=GLOBAL_SAMPLING, rounds=1):
        occ = np.ascontiguousarray(occ, dtype=np.uint32)
        nw, nk = occ.shape
        total = int(occ.sum())
        cap = max(1, min(want, total)) * rounds
        out = np.zeros(cap * 3, np.uint32)
        counts = np.zeros(rounds, np.uint64)
        self.f["plan"](want, nw, nk, occ.ravel(), seed, worker, purpose, rounds, out, counts)
        res, pos = [], 0
        for c in counts:
            c = int(c)
            res.append(out[pos: pos + 3 * c].reshape(c, 3).copy())
            pos += 3 * c
        return res if rounds > 1 else res[0]

    # --- S5 replay ----------------------------------------------------------------------
    def replay(self, N, K, cap, S, c, r, seed):
        return Replay(self, N, K, cap, S, c, r, seed)

    def engine_bench(self, N, K, cap, S, n, c, r, seed, batches, labels, warmup, iters):
        """Reference arm: the real async engine (N in-process workers over loopback)."""
        assert self.kind == "reference"
        batches = np.ascontiguousarray(batches, np.uint8).reshape(-1)
        labels = np.ascontiguousarray(labels, np.uint32).reshape(-1)
        n_batches = labels.size // (N * n)
        secs = C.c_double(0)
        samples = C.c_uint64(0)
        rc = self.lib.ref_engine_bench(N, K, cap, S, n, c, r, seed, batches, labels, n_batches,
                                       warmup, iters, C.byref(secs), C.byref(samples))
        if rc:
            raise RuntimeError(f"ref_engine_bench failed rc={rc}")
        return secs.value, samples.value


class Replay:
    def __init__(self, be: Backend, N, K, cap, S, c, r, seed):
        self.be, self.N, self.K, self.cap, self.S, self.c, self.r = be, N, K, cap, S, c, r
        self.h = be.f["replay_create"](N, K, cap, S, c, r, seed)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.be.f["replay_destroy"](h)
            self.h = None

    def step(self, batches: np.ndarray, labels: np.ndarray):
        """batches [N, n, S] u8, labels [N, n] u32 -> (aug [N, n+r, S], aug_labels, counts)."""
        N, n = labels.shape
        out = np.zeros((N, n + self.r, self.S), np.uint8)
        out_l = np.zeros((N, n + self.r), np.uint32)
        counts = np.zeros(N, np.uint32)
        rc = self.be.f["replay_step"](self.h, np.ascontiguousarray(batches, np.uint8).reshape(-1),
                                      np.ascontiguousarray(labels, np.uint32).reshape(-1), n,
                                      out.reshape(-1), out_l.reshape(-1), counts)
        if rc:
            raise ValueError(f"replay step failed rc={rc}")
        return out, out_l, counts

    def last_plan(self, w):
        out = np.zeros(max(self.r, 1) * 3, np.uint32)
        c = self.be.f["replay_last_plan"](self.h, w, out)
        return out[: 3 * c].reshape(c, 3).copy()

    def last_report(self, w):
        a = np.zeros(self.K, np.uint32)
        rp = np.zeros(self.K, np.uint32)
        t = np.zeros(2, np.uint32)
        self.be.f["replay_last_report"](self.h, w, a, rp, t)
        return a, rp, t

    def dump(self, w, occupancy_only=False):
        occ = np.zeros(self.K, np.uint32)
        ver = np.zeros(1, np.uint64)
        if occupancy_only:
            assert self.be.kind == "port"
            self.be.f["replay_dump"](self.h, w, occ, ver, None, None)
            return occ, int(ver[0]), None, None
        slab = np.zeros(self.K * self.cap * self.S, np.uint8)
        sl = np.zeros(self.K * self.cap, np.uint32)
        self.be.f["replay_dump"](self.h, w, occ, ver, slab, sl)
        return occ, int(ver[0]), slab.reshape(self.K, self.cap, self.S), sl.reshape(self.K, self.cap)

    def counters(self, w):
        assert self.be.kind == "port"
        out = np.zeros(3, np.uint64)
        self.be.lib.or_replay_counters(self.h, w, out)
        return out


class _or_stream(C.Structure):
    _fields_ = [("key", C.c_uint64), ("ctr", C.c_uint64)]


class OracleBuffer:
    """One rank's rehearsal_buffer restated in C (drb_oracle.c or_update_buffer)."""

    def __init__(self, K, cap, S):
        self.lib = Backend("port").lib
        f = self.lib.or_update_buffer
        f.restype = C.c_int
        f.argtypes = [_u8p, _u32p, _u32p, _u64p, C.c_uint32, C.c_uint32, C.c_uint64, _u8p, _u32p, C.c_uint32,
                      C.c_uint32, C.POINTER(_or_stream), C.POINTER(_or_stream), _u32p, _u32p]
        mk = self.lib.or_stream_make
        mk.restype = _or_stream
        mk.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, C.c_uint64, C.c_uint64]
        self.K, self.cap, self.S = K, cap, S
        self.slab = np.zeros((K, cap, S), np.uint8)
        self.slab_labels = np.zeros((K, cap), np.uint32)
        self.occ = np.zeros(K, np.uint32)
        self.version = np.zeros(1, np.uint64)

    def stream(self, seed, worker, purpose, keyed=False, k1=0, k2=0):
        return self.lib.or_stream_make(seed, worker, purpose, int(keyed), k1, k2)

    def update_buffer(self, batch, labels, c, cand, evict):
        n = int(labels.shape[0])
        app = np.zeros(self.K, np.uint32)
        rep = np.zeros(self.K, np.uint32)
        b = np.ascontiguousarray(batch, np.uint8).reshape(-1) if n else np.zeros(1, np.uint8)
        l = np.ascontiguousarray(labels, np.uint32) if n else np.zeros(1, np.uint32)
        rc = self.lib.or_update_buffer(self.slab.reshape(-1), self.slab_labels.reshape(-1), self.occ, self.version,
                                       self.K, self.cap, self.S, b, l, n, c, C.byref(cand), C.byref(evict), app, rep)
        return rc, app, rep


    def read_slots(self, requests, sub):
        """read_slots (rehearsal_buffer.cpp:88-142) with the substitute stream `sub`
        (or_read_slots). Returns (bytes [count, S], labels, status)."""
        f = self.lib.or_read_slots
        f.restype = C.c_int
        f.argtypes = [_u8p, _u32p, _u32p, C.c_uint32, C.c_uint32, C.c_uint64, _u32p, C.c_uint32,
                      C.POINTER(_or_stream), _u8p, _u32p, _u8p]
        cnt = len(requests)
        req = np.ascontiguousarray(np.asarray(requests, np.uint32).reshape(-1)) if cnt else np.zeros(2, np.uint32)
        out = np.zeros((max(cnt, 1), self.S), np.uint8)
        out_l = np.zeros(max(cnt, 1), np.uint32)
        st = np.zeros(max(cnt, 1), np.uint8)
        f(self.slab.reshape(-1), self.slab_labels.reshape(-1), self.occ, self.K, self.cap, self.S, req, cnt,
          C.byref(sub), out.reshape(-1), out_l, st)
        return out[:cnt], out_l[:cnt], st[:cnt]

    def next_u64(self, s):
        f = self.lib.or_next_u64
        f.restype = C.c_uint64
        f.argtypes = [C.POINTER(_or_stream)]
        return int(f(C.byref(s)))


def reference_read_slots(K, cap, S, batches, labels, c, seed, keyed, purpose, k1, k2, requests):
    """The reference's own rehearsal_buffer: len(batches) update_buffer rounds, then one
    read_slots with the given substitute stream (ref_read_slots_scenario). Returns (bytes,
    labels, status, the substitute stream's next draw, occupancy)."""
    lib = C.CDLL(REF_LIB)
    f = lib.ref_read_slots_scenario
    f.restype = C.c_int
    f.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, _u8p, _u32p, C.c_uint32, C.c_uint32, C.c_uint64,
                  C.c_int, C.c_uint32, C.c_uint64, C.c_uint64, _u32p, C.c_uint32, _u8p, _u32p, _u8p, _u64p, _u32p]
    rounds, n = int(labels.shape[0]), int(labels.shape[1])
    cnt = len(requests)
    req = np.ascontiguousarray(np.asarray(requests, np.uint32).reshape(-1)) if cnt else np.zeros(2, np.uint32)
    out = np.zeros((max(cnt, 1), S), np.uint8)
    out_l = np.zeros(max(cnt, 1), np.uint32)
    st = np.zeros(max(cnt, 1), np.uint8)
    nxt = np.zeros(1, np.uint64)
    occ = np.zeros(K, np.uint32)
    b = np.ascontiguousarray(batches, np.uint8).reshape(-1) if rounds * n else np.zeros(1, np.uint8)
    l = np.ascontiguousarray(labels, np.uint32).reshape(-1) if rounds * n else np.zeros(1, np.uint32)
    rc = f(K, cap, S, rounds, b, l, n, c, seed, int(keyed), purpose, k1, k2, req, cnt, out.reshape(-1), out_l, st,
           nxt, occ)
    if rc:
        raise RuntimeError(f"ref_read_slots_scenario failed rc={rc}")
    return out[:cnt], out_l[:cnt], st[:cnt], int(nxt[0]), occ


# ---- global-sampling bias test (proj/src/runner/bias.cpp:35-154), test infrastructure -----
def bias_view(N: int, K: int, fill: int) -> np.ndarray:
    """Frozen occupancy after the fill phase (bias.cpp:42-45,84-89): rank w inserts
    fill/N (+1 for w < fill % N) samples labelled i % K, all appended (capacity covers it)."""
    occ = np.zeros((N, K), np.uint32)
    for w in range(N):
        here = fill // N + (1 if w < fill % N else 0)
        for c in range(K):
            occ[w, c] = here // K + (1 if c < here % K else 0)
    return occ


def bias_counts(be: "Backend", occ: np.ndarray, r: int, seed: int, draws: int, local_only: bool) -> np.ndarray:
    """Per-slot hit counts of `draws` plans on rank 0's global-sampling stream (bias.cpp:
    104-133); the biased control plans over rank 0's own slots only (plan_local_only,
    sampler.cpp:70-83 == plan over the one-row view). Slots are counted in flat order."""
    total = int(occ.sum())
    view = occ[:1] if local_only else occ
    plans = be.plan(r, view, seed, 0, GLOBAL_SAMPLING, rounds=draws)
    pre = np.concatenate([[0], np.cumsum(occ.reshape(-1).astype(np.int64))])
    K = occ.shape[1]
    flat = np.concatenate([pre[p[:, 0].astype(np.int64) * K + p[:, 1]] + p[:, 2] for p in plans if len(p)])
    return np.bincount(flat, minlength=total).astype(np.uint64)


def reference_bias_report(counts: np.ndarray, r: int, draws: int):
    """make_bias_report of the reference itself (metrics.cpp:90-107) -> (statistic, p)."""
    lib = C.CDLL(REF_LIB)
    f = lib.ref_bias_report
    f.restype = C.c_int
    f.argtypes = [_u64p, C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    st, p = C.c_double(0), C.c_double(0)
    rc = f(np.ascontiguousarray(counts, np.uint64), len(counts), r, draws, C.byref(st), C.byref(p))
    if rc:
        raise ValueError("make_bias_report failed")
    return st.value, p.value


def have_reference() -> bool:
    return os.path.exists(REF_LIB)
