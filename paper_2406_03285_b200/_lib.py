"""ctypes binding of the C ABI in include/drb_rb.h (libdrb_b200.so, built in-tree).

There is no fallback: if the CUDA library is missing this module raises ImportError.
Exceptions mirror the reference taxonomy (proj/src/core/errors.hpp:1-46) and the status
mapping of proj/src/capi/drb_capi.cpp:29-46.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DRB_LIB") or os.path.join(HERE, "libdrb_b200.so")  # DRB_LIB: A/B experiments

DRB_OK = 0
DRB_ERR_INVALID_ARGUMENT = 1
DRB_ERR_CONFIG = 2
DRB_ERR_IO = 3
DRB_ERR_TRANSPORT = 4
DRB_ERR_PROTOCOL = 5
DRB_ERR_TRAINING = 6
DRB_ERR_USAGE = 7
DRB_ERR_INTERNAL = 8
MAX_WORLD = 8
FLAG_TIMINGS = 1  # DRB_RB_FLAG_TIMINGS
AUG_RING = 32  # default m' ring depth (drb_rb_config.aug_ring = 0)


class drb_error(RuntimeError):
    status = DRB_ERR_INTERNAL


class invalid_argument(drb_error):
    status = DRB_ERR_INVALID_ARGUMENT


class config_error(drb_error):
    status = DRB_ERR_CONFIG


class transport_error(drb_error):
    status = DRB_ERR_TRANSPORT


class engine_error(drb_error):
    status = DRB_ERR_TRAINING


class usage_error(drb_error):
    status = DRB_ERR_USAGE


class io_error(drb_error):
    status = DRB_ERR_IO


_BY_STATUS = {c.status: c for c in (invalid_argument, config_error, io_error, transport_error, engine_error,
                                    usage_error)}


class drb_rng(C.Structure):
    _fields_ = [("key", C.c_uint64), ("ctr", C.c_uint64)]


class drb_rb_config(C.Structure):
    _fields_ = [
        ("n_classes", C.c_uint32),
        ("per_class_cap", C.c_uint32),
        ("sample_bytes", C.c_uint64),
        ("max_batch", C.c_uint32),
        ("candidate_count", C.c_uint32),
        ("rep_count", C.c_uint32),
        ("rank", C.c_uint32),
        ("world", C.c_uint32),
        ("seed", C.c_uint64),
        ("device", C.c_int32),
        ("flags", C.c_uint32),
        ("aug_ring", C.c_uint32),
        ("engine_ctas", C.c_uint32),
    ]


class drb_insertion_report(C.Structure):
    _fields_ = [
        ("per_class_appends", C.POINTER(C.c_uint32)),
        ("per_class_replacements", C.POINTER(C.c_uint32)),
        ("appends", C.c_uint32),
        ("replacements", C.c_uint32),
    ]


class drb_read_request(C.Structure):
    _fields_ = [("cls", C.c_uint32), ("slot", C.c_uint32)]


class drb_slot_ref(C.Structure):
    _fields_ = [("owner", C.c_uint32), ("cls", C.c_uint32), ("slot", C.c_uint32)]


class drb_timing(C.Structure):
    _fields_ = [("iteration", C.c_uint64), ("populate_ms", C.c_double), ("augment_ms", C.c_double),
                ("latency_ms", C.c_double), ("wait_ms", C.c_double), ("degraded", C.c_uint32),
                ("pad", C.c_uint32)]


class drb_aug(C.Structure):
    _fields_ = [
        ("data", C.c_void_p),
        ("labels", C.c_void_p),
        ("n", C.c_uint32),
        ("ring_slot", C.c_uint32),
        ("step", C.c_uint64),
    ]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a library first "
            "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    u32, u64, i32, vp, sz = C.c_uint32, C.c_uint64, C.c_int32, C.c_void_p, C.c_size_t
    st = C.c_int
    sigs = {
        "drb_rb_version": (C.c_char_p, []),
        "drb_rb_last_error": (C.c_char_p, []),
        "drb_rng_init": (st, [P(drb_rng), u64, u32, u32]),
        "drb_rng_keyed": (st, [P(drb_rng), u64, u32, u32, u64, u64]),
        "drb_rng_draw": (st, [P(drb_rng), u64, u64, vp, i32]),
        "drb_sample_without_replacement": (st, [u32, u32, P(drb_rng), vp, P(u32), i32]),
        "drb_plan": (st, [u32, u32, u32, vp, P(drb_rng), vp, P(u32), i32]),
        "drb_rb_create": (st, [P(drb_rb_config), P(vp)]),
        "drb_rb_destroy": (st, [vp]),
        "drb_rb_update_buffer": (st, [vp, vp, vp, u32, u32, P(drb_rng), P(drb_rng), P(drb_insertion_report)]),
        "drb_rb_read_slots": (st, [vp, vp, u32, P(drb_rng), vp, vp, vp]),
        "drb_rb_snapshot": (st, [vp, vp, P(u64)]),
        "drb_rb_total_stored": (st, [vp, P(u64)]),
        "drb_rb_cross_class_evictions": (st, [vp, P(u64)]),
        "drb_rb_device_views": (st, [vp, P(vp), P(vp)]),
        "drb_rb_export_handle": (st, [vp, vp, P(sz)]),
        "drb_rb_handle_size": (sz, []),
        "drb_rb_connect": (st, [vp, vp, sz]),
        "drb_rb_start": (st, [vp]),
        "drb_rb_shutdown": (st, [vp]),
        "drb_rb_step": (st, [vp, vp, vp, u32, vp, P(drb_aug)]),
        "drb_rb_step_split": (st, [vp, vp, vp, u32, vp, vp, P(drb_aug)]),
        "drb_rb_step_host": (st, [vp, vp, vp, u32, vp, vp, vp]),
        "drb_rb_run": (st, [vp, vp, u64, vp, u64, u32, u32, u64, u64, vp, vp]),
        "drb_rb_graph_prepare": (st, [vp, vp, u64, vp, u64, u32, u32, u64, u64, vp, P(vp)]),
        "drb_rb_graph_launch": (st, [vp, vp]),
        "drb_rb_graph_destroy": (st, [vp]),
        "drb_rb_aug_count": (st, [vp, P(drb_aug), P(u32)]),
        "drb_rb_aug_slot": (st, [vp, u64, u32, P(drb_aug)]),
        "drb_rb_engine_info": (st, [vp, P(u32), P(u64), P(u64), P(u32)]),
        "drb_rb_synchronize": (st, [vp]),
        "drb_rb_total_wait_ms": (st, [vp, P(C.c_double)]),
        "drb_rb_engine_counters": (st, [vp, P(u64), P(u64), P(u64), P(u64)]),
        "drb_rb_broadcast_sizes": (st, [vp]),
        "drb_rb_drain_timings": (st, [vp, P(drb_timing), u32, P(u32)]),
        "drb_rb_device_error": (st, [vp, P(u32)]),
        "drb_rb_launch_info": (st, [vp, P(u32), P(u32), P(u32)]),
        "drb_ds_load": (st, [C.c_char_p, i32, P(vp)]),
        "drb_ds_synth": (st, [u32, u32, u32, C.c_double, u64, i32, P(vp)]),
        "drb_ds_destroy": (st, [vp]),
        "drb_ds_info": (st, [vp, P(u64), P(u32), P(u32), P(u64), P(u64)]),
        "drb_ds_device_views": (st, [vp, P(vp), P(vp)]),  # uint32_t** as void**
        "drb_ds_indices_of": (st, [vp, vp, u32, i32, vp, u64, P(u64)]),
        "drb_ds_gather": (st, [vp, vp, u32, vp, vp, vp]),
        "drb_ds_device_error": (st, [vp, P(u32)]),
        "drb_make_schedule": (st, [u32, u32, u64, vp, vp]),
        "drb_shard_batches": (st, [vp, u64, u32, u32, u32, u64, u64, u64, vp, u64, P(u64)]),
        "drb_lockstep_batches": (st, [u64, u32, u32, P(u64)]),
        "drb_rb_bias_test": (st, [u32, u32, u32, u64, u64, u64, i32, vp, P(C.c_double), P(C.c_double), i32]),
        "drb_rb_trace_read": (st, [vp, vp]),
        "drb_rb_timeline_read": (st, [vp, vp, P(u32)]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    if status != DRB_OK:
        msg = lib.drb_rb_last_error().decode(errors="replace")
        raise _BY_STATUS.get(status, drb_error)(f"[{status}] {msg}")
