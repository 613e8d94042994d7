"""Python mirror of the reference's hot-path C++ API over the sm_100a C ABI.

Names, argument meaning and error behaviour follow the reference:
  rng_stream                      proj/src/core/rng.hpp:16-51
  sample_without_replacement      proj/src/buffer/rehearsal_buffer.hpp:130-132
  rehearsal_buffer                proj/src/buffer/rehearsal_buffer.hpp:60-128
  plan / augment                  proj/src/sampler/sampler.hpp:33-61
  engine                          proj/src/engine/engine.hpp:41-145
A mini-batch is a pair (data, labels) of CUDA tensors: data uint8 [n, S] (any payload
dtype viewed as bytes), labels int32/int64/uint32 [n]. Everything runs on the GPU through
libdrb_b200.so; torch only provides device memory and streams.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import check, lib

CANDIDATE_SELECTION, EVICTION, GLOBAL_SAMPLING, DATA_SHUFFLE, MODEL_INIT, SLOT_SUBSTITUTE, SYNTH = range(1, 8)


# --------------------------------------------------------------------------------------
# device-pointer plumbing
class _cai:
    """Minimal __cuda_array_interface__ holder to view engine-owned memory as a tensor."""

    def __init__(self, ptr: int, shape, typestr: str, owner):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 2, "strides": None}
        self._owner = owner


_CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy


def _stream_arg(s: torch.cuda.Stream) -> C.c_void_p:
    """The handle to pass for a torch stream. torch's default stream reports handle 0, which the
    C ABI reads as "the engine's own stream" (unordered with the caller's work), so the legacy
    default stream is passed explicitly."""
    return C.c_void_p(s.cuda_stream or _CUDA_STREAM_LEGACY)


def _view(ptr: int, shape, typestr: str, device: int, owner) -> torch.Tensor:
    return torch.as_tensor(_cai(ptr, shape, typestr, owner), device=f"cuda:{device}")


def _as_bytes(data: torch.Tensor) -> torch.Tensor:
    if not data.is_cuda:
        raise _lib.usage_error("mini-batch data must be a CUDA tensor")
    data = data.contiguous()
    return data.view(torch.uint8).reshape(data.shape[0], -1) if data.dim() > 0 else data


def _as_labels(labels: torch.Tensor) -> torch.Tensor:
    if not labels.is_cuda:
        raise _lib.usage_error("labels must be a CUDA tensor")
    if labels.dtype in (torch.int32, torch.uint32):
        return labels.contiguous()
    return labels.to(torch.int32).contiguous()


# --------------------------------------------------------------------------------------
class rng_stream:
    """Counter-based stream; state (key, ctr) lives on the host, draws run on the GPU."""

    purpose = type("purpose", (), dict(candidate_selection=1, eviction=2, global_sampling=3, data_shuffle=4,
                                       model_init=5, slot_substitute=6, synth=7))

    def __init__(self, seed: int, worker: int, purpose: int, _raw: Optional[_lib.drb_rng] = None):
        self.s = _lib.drb_rng()
        if _raw is not None:
            self.s = _raw
        else:
            check(lib.drb_rng_init(C.byref(self.s), seed, worker, purpose))

    @staticmethod
    def keyed(seed: int, worker: int, purpose: int, k1: int, k2: int = 0) -> "rng_stream":
        s = _lib.drb_rng()
        check(lib.drb_rng_keyed(C.byref(s), seed, worker, purpose, k1, k2))
        return rng_stream(0, 0, 0, _raw=s)

    @property
    def counter(self) -> int:
        return int(self.s.ctr)

    def next_u64(self, n: int = 1, device: int = 0) -> np.ndarray:
        out = np.zeros(max(n, 1), np.uint64)
        check(lib.drb_rng_draw(C.byref(self.s), 0, n, out.ctypes.data, device))
        return out[:n]

    def bounded(self, bound: int, n: int = 1, device: int = 0) -> np.ndarray:
        if bound == 0:
            raise _lib.usage_error("bounded: n must be nonzero")
        out = np.zeros(max(n, 1), np.uint64)
        check(lib.drb_rng_draw(C.byref(self.s), bound, n, out.ctypes.data, device))
        return out[:n]


def sample_without_replacement(n: int, k: int, rng: rng_stream, device: int = 0) -> np.ndarray:
    out = np.zeros(max(min(n, k), 1), np.uint32)
    got = C.c_uint32(0)
    check(lib.drb_sample_without_replacement(n, k, C.byref(rng.s), out.ctypes.data, C.byref(got), device))
    return out[: got.value]


@dataclass
class sampling_plan:
    entries: np.ndarray  # [m, 3] (owner, cls, slot) in draw order

    def has_duplicates(self) -> bool:
        return len({tuple(e) for e in self.entries.tolist()}) != len(self.entries)

    def distinct_owners(self) -> List[int]:
        return sorted(set(int(o) for o in self.entries[:, 0])) if len(self.entries) else []


def plan(want: int, view: np.ndarray, rng: rng_stream, device: int = 0) -> sampling_plan:
    """plan(want, view, rng): view is occupancy[n_workers][n_classes] (sampler.cpp:65-68)."""
    view = np.ascontiguousarray(view, np.uint32)
    nw, nk = view.shape
    total = int(view.sum())
    out = np.zeros((max(1, min(want, total)), 3), np.uint32)
    got = C.c_uint32(0)
    check(lib.drb_plan(want, nw, nk, view.ctypes.data, C.byref(rng.s), out.ctypes.data, C.byref(got), device))
    return sampling_plan(out[: got.value].copy())


@dataclass
class bias_report:
    statistic: float
    p_value: float
    counts: np.ndarray  # per-slot hits, flat worker-major order


def bias_test(n_workers: int, n_classes: int, rep_count: int, seed: int, draws: int, fill: int,
              biased_control: bool = False, device: int = 0) -> bias_report:
    """drb_bias_test (drb.h:91-97, bias.cpp:35-154) with the plans drawn on the GPU."""
    counts = np.zeros(max(fill, 1), np.uint64)
    st, p = C.c_double(0), C.c_double(0)
    check(lib.drb_rb_bias_test(n_workers, n_classes, rep_count, seed, draws, fill, 1 if biased_control else 0,
                               counts.ctypes.data, C.byref(st), C.byref(p), device))
    return bias_report(float(st.value), float(p.value), counts[:fill])


def augment(m: Tuple[torch.Tensor, torch.Tensor], reps: Tuple[torch.Tensor, torch.Tensor]):
    """m then reps (sampler.cpp:234-240). The engine already produces this layout in place;
    this standalone form concatenates two device batches."""
    d = torch.cat([_as_bytes(m[0]), _as_bytes(reps[0])], 0) if len(reps[0]) else _as_bytes(m[0]).clone()
    l = torch.cat([_as_labels(m[1]), _as_labels(reps[1])], 0) if len(reps[1]) else _as_labels(m[1]).clone()
    return d, l


@dataclass
class insertion_report:
    per_class: dict = field(default_factory=dict)  # class -> (appends, replacements)
    appends: int = 0
    replacements: int = 0


@dataclass
class occupancy_snapshot:
    per_class: List[int]
    version: int

    def total(self) -> int:
        return int(sum(self.per_class))


READ_EXACT, READ_SUBSTITUTED, READ_EMPTY = 0, 1, 2


@dataclass
class read_entry:
    status: int
    value: torch.Tensor  # [S] uint8 on device
    label: int


# --------------------------------------------------------------------------------------
class rehearsal_buffer:
    """One rank's HBM-resident buffer (+ the engine state that drives it).

    rehearsal_buffer(n_classes, per_class_cap, sample_bytes, ...) mirrors
    rehearsal_buffer(K, cap) (rehearsal_buffer.cpp:28-35); config_error on K==0/cap==0.
    The engine parameters (c, r, seed, rank, world, max_batch) are fixed at construction
    because the device state of the asynchronous engine is allocated with the buffer.
    """

    def __init__(self, n_classes: int, per_class_cap: int, sample_bytes: int, *, max_batch: int = 64,
                 candidate_count: int = 14, rep_count: int = 7, seed: int = 1, rank: int = 0,
                 world: int = 1, device: int = 0, aug_ring: int = 0, engine_ctas: int = 0,
                 record_timings: bool = False):
        cfg = _lib.drb_rb_config(n_classes=n_classes, per_class_cap=per_class_cap, sample_bytes=sample_bytes,
                                 max_batch=max_batch, candidate_count=candidate_count, rep_count=rep_count,
                                 rank=rank, world=world, seed=seed, device=device,
                                 flags=_lib.FLAG_TIMINGS if record_timings else 0, aug_ring=aug_ring,
                                 engine_ctas=engine_ctas)
        self.h = C.c_void_p()
        check(lib.drb_rb_create(C.byref(cfg), C.byref(self.h)))
        self.K, self.cap, self.S = n_classes, per_class_cap, sample_bytes
        self.max_batch, self.c, self.r = max_batch, candidate_count, rep_count
        self.seed, self.rank, self.world, self.device = seed, rank, world, device
        self.aug_ring = aug_ring or _lib.AUG_RING

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            check(lib.drb_rb_destroy(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def n_classes(self) -> int:
        return self.K

    def per_class_cap(self) -> int:
        return self.cap

    # update_buffer(m, c, cand, evict) (rehearsal_buffer.cpp:37-86)
    def update_buffer(self, m, candidate_count: int, candidate_rng: rng_stream,
                      eviction_rng: rng_stream) -> insertion_report:
        data, labels = m
        n = int(labels.shape[0])
        data = _as_bytes(data) if n else data
        labels = _as_labels(labels) if n else labels
        app = (C.c_uint32 * self.K)()
        rep = (C.c_uint32 * self.K)()
        r = _lib.drb_insertion_report(C.cast(app, C.POINTER(C.c_uint32)), C.cast(rep, C.POINTER(C.c_uint32)), 0, 0)
        torch.cuda.current_stream(self.device).synchronize()
        check(lib.drb_rb_update_buffer(self.h, data.data_ptr() if n else None, labels.data_ptr() if n else None, n,
                                       candidate_count, C.byref(candidate_rng.s), C.byref(eviction_rng.s),
                                       C.byref(r)))
        per = {k: (app[k], rep[k]) for k in range(self.K) if app[k] or rep[k]}
        return insertion_report(per, r.appends, r.replacements)

    # read_slots(requests, substitute_rng) (rehearsal_buffer.cpp:88-142)
    def read_slots(self, requests: Sequence[Tuple[int, int]], substitute_rng: rng_stream) -> List[read_entry]:
        cnt = len(requests)
        req = (_lib.drb_read_request * max(cnt, 1))(*[_lib.drb_read_request(c, s) for c, s in requests])
        out = torch.empty((max(cnt, 1), self.S), dtype=torch.uint8, device=f"cuda:{self.device}")
        out_l = torch.empty(max(cnt, 1), dtype=torch.int32, device=f"cuda:{self.device}")
        status = (C.c_uint8 * max(cnt, 1))()
        check(lib.drb_rb_read_slots(self.h, req, cnt, C.byref(substitute_rng.s), out.data_ptr(), out_l.data_ptr(),
                                    status))
        labels = out_l.cpu().tolist()
        return [read_entry(int(status[i]), out[i], int(labels[i])) for i in range(cnt)]

    def snapshot(self) -> occupancy_snapshot:
        occ = np.zeros(self.K, np.uint32)
        ver = C.c_uint64(0)
        check(lib.drb_rb_snapshot(self.h, occ.ctypes.data, C.byref(ver)))
        return occupancy_snapshot(occ.tolist(), int(ver.value))

    def total_stored(self) -> int:
        v = C.c_uint64(0)
        check(lib.drb_rb_total_stored(self.h, C.byref(v)))
        return int(v.value)

    def cross_class_evictions(self) -> int:
        v = C.c_uint64(0)
        check(lib.drb_rb_cross_class_evictions(self.h, C.byref(v)))
        return int(v.value)

    def slab(self) -> Tuple[torch.Tensor, torch.Tensor]:
        """Zero-copy views of the HBM slab [K, cap, S] and slot labels [K, cap]."""
        s, l = C.c_void_p(), C.c_void_p()
        check(lib.drb_rb_device_views(self.h, C.byref(s), C.byref(l)))
        return (_view(s.value, (self.K, self.cap, self.S), "|u1", self.device, self),
                _view(l.value, (self.K, self.cap), "<i4", self.device, self))

    # multi-rank wiring
    def export_handle(self) -> bytes:
        n = lib.drb_rb_handle_size()
        buf = (C.c_uint8 * n)()
        ln = C.c_size_t(n)
        check(lib.drb_rb_export_handle(self.h, buf, C.byref(ln)))
        return bytes(buf)

    def connect(self, blobs: Sequence[bytes]) -> None:
        joined = b"".join(blobs)
        buf = (C.c_uint8 * len(joined)).from_buffer_copy(joined)
        check(lib.drb_rb_connect(self.h, buf, len(joined)))

    def launch_info(self):
        g, t, s = C.c_uint32(), C.c_uint32(), C.c_uint32()
        check(lib.drb_rb_launch_info(self.h, C.byref(g), C.byref(t), C.byref(s)))
        return int(g.value), int(t.value), int(s.value)


def _ring_args(buf: "rehearsal_buffer", data_ring: torch.Tensor, label_ring: torch.Tensor, what: str):
    """A device input ring as the C ABI takes it: bytes [B, n, S] (any payload dtype, row
    stride in BYTES) and uint32/int32 labels [B, n]."""
    if not data_ring.is_cuda or not label_ring.is_cuda:
        raise _lib.usage_error(f"{what}: rings must be CUDA tensors")
    if data_ring.dim() < 2 or label_ring.dim() != 2:
        raise _lib.usage_error(f"{what}: data ring [B, n, ...] and label ring [B, n] expected")
    B, n = int(data_ring.shape[0]), int(data_ring.shape[1])
    if tuple(label_ring.shape) != (B, n):
        raise _lib.usage_error(f"{what}: label ring must be [B, n] = [{B}, {n}]")
    if n > buf.max_batch:
        raise _lib.usage_error(f"{what}: batch of {n} rows exceeds max_batch {buf.max_batch}")
    data = data_ring.contiguous().view(torch.uint8).reshape(B, n, -1)
    if int(data.shape[2]) != buf.S:
        raise _lib.usage_error(f"{what}: samples are {int(data.shape[2])} bytes, the buffer holds {buf.S}")
    labels = label_ring if label_ring.dtype in (torch.int32, torch.uint32) else label_ring.to(torch.int32)
    labels = labels.contiguous()
    return data, labels, B, n


class augmented_batch:
    """m'_i = m_i ++ reps(i-1), engine-owned (valid until two more updates are enqueued)."""

    def __init__(self, eng: "engine", aug: _lib.drb_aug):
        self.eng, self.aug = eng, aug
        self._count: Optional[int] = None

    @property
    def n(self) -> int:
        return int(self.aug.n)

    def count(self) -> int:
        if self._count is None:
            c = C.c_uint32(0)
            check(lib.drb_rb_aug_count(self.eng.buffer.h, C.byref(self.aug), C.byref(c)))
            self._count = int(c.value)
        return self._count

    def tensors_nowait(self) -> Tuple[torch.Tensor, torch.Tensor]:
        """Views of the n + r rows m'_i has in steady state (the global buffer holds >= r
        slots), without waiting on the host: consumers order on the device (stream events)."""
        b = self.eng.buffer
        rows = self.n + b.r
        return (_view(self.aug.data, (rows, b.S), "|u1", b.device, self),
                _view(self.aug.labels, (rows,), "<i4", b.device, self))

    def tensors(self) -> Tuple[torch.Tensor, torch.Tensor]:
        b = self.eng.buffer
        cnt = self.count()
        d = _view(self.aug.data, (cnt, b.S), "|u1", b.device, self)
        l = _view(self.aug.labels, (cnt,), "<i4", b.device, self)
        return d, l

    def reps(self) -> Tuple[torch.Tensor, torch.Tensor]:
        d, l = self.tensors()
        return d[self.n:], l[self.n:]


class prepared_run:
    """A captured multi-iteration run (CUDA graph). Keeps its input rings alive."""

    def __init__(self, g: C.c_void_p, keep):
        self.g, self._keep = g, keep

    def launch(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream()
        check(lib.drb_rb_graph_launch(self.g, _stream_arg(s)))

    def close(self) -> None:
        if self.g and self.g.value:
            check(lib.drb_rb_graph_destroy(self.g))
            self.g = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class engine:
    """engine(cfg, rank, buffer, ...) (engine.hpp:53-93) over a rehearsal_buffer handle."""

    def __init__(self, buffer: rehearsal_buffer):
        self.buffer = buffer
        self.iteration = 0

    def start(self) -> None:
        check(lib.drb_rb_start(self.buffer.h))

    def shutdown(self) -> None:
        check(lib.drb_rb_shutdown(self.buffer.h))

    def update(self, m, stream: Optional[torch.cuda.Stream] = None,
               consumer: Optional[torch.cuda.Stream] = None) -> augmented_batch:
        """Enqueue round i for m_i and return m'_i = m_i ++ reps(i-1) (fused update+augment,
        trainer.cpp:109-113). Waits are deferred to first use of the result: `stream` waits
        for m'_i. With `consumer`, m_i is posted in `stream`'s order (its producer) and the
        consumer stream releases the m' it used so far, then waits for m'_i (drb_rb_step_split:
        back-to-back updates run pipelined in the engine)."""
        data, labels = m
        n = int(labels.shape[0])
        data = _as_bytes(data) if n else data
        labels = _as_labels(labels) if n else labels
        s = stream if stream is not None else torch.cuda.current_stream(self.buffer.device)
        aug = _lib.drb_aug()
        if consumer is None:
            check(lib.drb_rb_step(self.buffer.h, data.data_ptr() if n else None, labels.data_ptr() if n else None,
                                  n, _stream_arg(s), C.byref(aug)))
        else:
            check(lib.drb_rb_step_split(self.buffer.h, data.data_ptr() if n else None,
                                        labels.data_ptr() if n else None, n, _stream_arg(s), _stream_arg(consumer),
                                        C.byref(aug)))
            s = consumer
        if n:  # m_i is read until "m'_i ready", which `s` waits for: the caching allocator must
            # not hand m_i's blocks (or a converted label copy) to anyone before that point
            data.record_stream(s)
            labels.record_stream(s)
        self.iteration += 1
        return augmented_batch(self, aug)

    def update_host(self, data: np.ndarray, labels: np.ndarray, out: np.ndarray, out_labels: np.ndarray,
                    out_count: np.ndarray) -> None:
        """Host-buffer variant (reference-facing e2e path); call synchronize() before reading."""
        n = int(labels.shape[0])
        check(lib.drb_rb_step_host(self.buffer.h, data.ctypes.data, labels.ctypes.data, n, out.ctypes.data,
                                   out_labels.ctypes.data, out_count.ctypes.data))
        self.iteration += 1

    def run(self, data_ring: torch.Tensor, label_ring: torch.Tensor, steps: int, first: int = 0,
            stream: Optional[torch.cuda.Stream] = None, events=None) -> None:
        """`steps` iterations over a device ring: data [B, n, ...] (any dtype; each row is S
        bytes), labels [B, n] int32/int64/uint32; iteration i uses data[(first+i) % B] and
        labels[(first+i) % B]."""
        data_ring, label_ring, B, n = _ring_args(self.buffer, data_ring, label_ring, "run")
        s = stream if stream is not None else torch.cuda.current_stream(self.buffer.device)
        ev = None
        if events is not None:
            ev = (C.c_void_p * len(events))(*[e.cuda_event for e in events])
        check(lib.drb_rb_run(self.buffer.h, data_ring.data_ptr(), data_ring.stride(0), label_ring.data_ptr(),
                             label_ring.stride(0), B, n, steps, first, _stream_arg(s), ev))
        data_ring.record_stream(s)  # read until the run completes on `s`
        label_ring.record_stream(s)
        self.iteration += steps

    def prepare_run(self, data_ring: torch.Tensor, label_ring: torch.Tensor, steps: int,
                    first: int = 0, events=None) -> "prepared_run":
        """Capture `steps` iterations (as run()) into a CUDA graph; launch it once, in order.
        events: optional 2*steps torch.cuda.Event (timing) bracketing each copy kernel."""
        data_ring, label_ring, B, n = _ring_args(self.buffer, data_ring, label_ring, "prepare_run")
        ev = None
        if events is not None:
            ev = (C.c_void_p * len(events))(*[e.cuda_event for e in events])
        g = C.c_void_p()
        check(lib.drb_rb_graph_prepare(self.buffer.h, data_ring.data_ptr(), data_ring.stride(0),
                                       label_ring.data_ptr(), label_ring.stride(0), B, n, steps, first, ev,
                                       C.byref(g)))
        self.iteration += steps
        return prepared_run(g, (data_ring, label_ring))

    def aug_slot(self, step: int, n: int) -> augmented_batch:
        """m'_step as the engine's ring still holds it (one of the last aug_ring steps; its
        batch had n rows). With aug_ring >= steps every m' of a run() stays readable."""
        aug = _lib.drb_aug()
        check(lib.drb_rb_aug_slot(self.buffer.h, step, n, C.byref(aug)))
        return augmented_batch(self, aug)

    def engine_info(self) -> dict:
        """resident: the engine runs as a resident kernel; instances: launched so far (one per
        busy period, not per step); posted: work descriptors posted; grid: CTAs per instance."""
        r, g = C.c_uint32(), C.c_uint32()
        inst, posted = C.c_uint64(), C.c_uint64()
        check(lib.drb_rb_engine_info(self.buffer.h, C.byref(r), C.byref(inst), C.byref(posted), C.byref(g)))
        return {"resident": bool(r.value), "instances": int(inst.value), "posted": int(posted.value),
                "grid": int(g.value)}

    def synchronize(self) -> None:
        check(lib.drb_rb_synchronize(self.buffer.h))

    def drain_timings(self) -> List[dict]:
        """engine::drain_timings (engine.hpp:93): per-round timings since the last drain
        (device stamps; the buffer must be created with record_timings=True)."""
        cap = 4096
        arr = (_lib.drb_timing * cap)()
        n = C.c_uint32(0)
        check(lib.drb_rb_drain_timings(self.buffer.h, arr, cap, C.byref(n)))
        return [{"iteration": int(t.iteration), "populate_ms": t.populate_ms, "augment_ms": t.augment_ms,
                 "latency_ms": t.latency_ms, "wait_ms": t.wait_ms, "degraded": int(t.degraded)}
                for t in arr[: n.value]]

    def _counters(self):
        v = [C.c_uint64(0) for _ in range(4)]
        check(lib.drb_rb_engine_counters(self.buffer.h, *[C.byref(x) for x in v]))
        return [int(x.value) for x in v]

    def iterations(self) -> int:
        """engine::iterations (engine.hpp:88): steps enqueued."""
        return self._counters()[0]

    def queue_depth(self) -> int:
        """engine::queue_depth (engine.hpp:89): enqueued steps whose m' is not ready yet."""
        return self._counters()[1]

    def degraded_rounds(self) -> int:
        """engine::degraded_rounds (engine.hpp:90): always 0 (fail-stop)."""
        return self._counters()[2]

    def replanned_entries(self) -> int:
        """engine::replanned_entries (engine.hpp:91): always 0 (no unreachable owners)."""
        return self._counters()[3]

    def broadcast_sizes(self) -> None:
        """engine::broadcast_sizes (engine.hpp:82): a no-op, every round publishes the row."""
        check(lib.drb_rb_broadcast_sizes(self.buffer.h))

    def total_wait_ms(self) -> float:
        v = C.c_double(0)
        check(lib.drb_rb_total_wait_ms(self.buffer.h, C.byref(v)))
        return float(v.value)

    def device_error(self) -> int:
        v = C.c_uint32(0)
        check(lib.drb_rb_device_error(self.buffer.h, C.byref(v)))
        return int(v.value)
