"""TEST INFRASTRUCTURE: runs input-side requests through the reference (oracle/_ref).

Loads libdrb_ref.so before numpy (see py_input_oracle.py), reads a JSON list of requests on
stdin, writes a JSON list of results on stdout. Never part of the product path.
"""
import ctypes as C
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
lib = C.CDLL(os.path.join(HERE, "_ref", "libdrb_ref.so"))
u32, u64, vp = C.c_uint32, C.c_uint64, C.c_void_p
P = C.POINTER
lib.ref_write_synth_dataset.argtypes = [C.c_char_p, u32, u32, u32, C.c_double, u64]
lib.ref_load_dataset.argtypes = [C.c_char_p, P(u64), P(u32), P(u32), P(u64), P(u64), vp, vp, C.c_char_p, C.c_size_t]
lib.ref_indices_of.argtypes = [C.c_char_p, vp, u32, C.c_int, vp, u64]
lib.ref_indices_of.restype = u64
lib.ref_make_schedule.argtypes = [u32, u32, u64, vp, vp]
lib.ref_shard_batches.argtypes = [vp, u64, u32, u32, u32, u64, u64, u64, vp, P(u64), P(u64)]
lib.ref_lockstep_batches.argtypes = [u64, u32, u32]
lib.ref_lockstep_batches.restype = u64

import numpy as np  # noqa: E402  (after the reference .so, on purpose)


def run(r):
    op = r["op"]
    if op == "synth":
        return {"rc": lib.ref_write_synth_dataset(r["path"].encode(), r["K"], r["per_class"], r["dim"],
                                                   float(r["sep"]), r["seed"])}
    if op == "load":
        cnt, tr, ev = u64(), u64(), u64()
        dim, k = u32(), u32()
        err = C.create_string_buffer(512)
        rc = lib.ref_load_dataset(r["path"].encode(), C.byref(cnt), C.byref(dim), C.byref(k), C.byref(tr),
                                  C.byref(ev), None, None, err, 512)
        if rc == 3:
            return {"io_error": err.value.decode()}
        f = np.empty((cnt.value, dim.value), np.float32)
        lab = np.empty(cnt.value, np.uint32)
        lib.ref_load_dataset(r["path"].encode(), C.byref(cnt), C.byref(dim), C.byref(k), C.byref(tr),
                             C.byref(ev), f.ctypes.data, lab.ctypes.data, err, 512)
        return {"count": cnt.value, "dim": dim.value, "n_classes": k.value, "train": tr.value, "eval": ev.value,
                "features": f.tobytes().hex(), "labels": lab.tolist()}
    if op == "indices_of":
        cls = np.asarray(r["classes"], np.uint32)
        out = np.empty(r["cap"], np.uint64)
        n = lib.ref_indices_of(r["path"].encode(), cls.ctypes.data, len(cls), r["eval"], out.ctypes.data, r["cap"])
        return out[:n].tolist()
    if op == "schedule":
        cls = np.empty(r["K"], np.uint32)
        sz = np.empty(r["T"], np.uint32)
        assert lib.ref_make_schedule(r["K"], r["T"], r["seed"], cls.ctypes.data, sz.ctypes.data) == 0
        return {"classes": cls.tolist(), "sizes": sz.tolist()}
    if op == "shard":
        td = np.asarray(r["task_data"], np.uint64)
        out = np.empty(max(len(td), 1), np.uint64)
        cnt, nb = u64(), u64()
        rc = lib.ref_shard_batches(td.ctypes.data, len(td), r["worker"], r["n_workers"], r["batch"], r["seed"],
                                   r["task"], r["epoch"], out.ctypes.data, C.byref(cnt), C.byref(nb))
        return {"rc": rc, "shard": out[:cnt.value].tolist(), "n_batches": nb.value}
    if op == "lockstep":
        return lib.ref_lockstep_batches(r["n"], r["n_workers"], r["batch"])
    raise ValueError(op)


json.dump([run(r) for r in json.load(sys.stdin)], sys.stdout)
