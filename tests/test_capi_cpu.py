"""CPU-only checks of the C ABI boundary (no device needed): the product library loads,
exports every function include/drb_rb.h declares, validates configurations before touching
the GPU (config_error taxonomy of proj/src/capi/drb_capi.cpp:29-46), rejects NULL
arguments, and keys its counter-based streams exactly like rng_stream (rng.cpp:19-39)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "drb_rb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"DRB_RB_API\s+[\w\s\*]+?\b(drb_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2406_03285_b200 import _lib
    names = header_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(_lib.lib, n)]
    assert not missing, missing
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    assert set(names) <= exported, set(names) - exported
    # no torch / CUDA runtime symbols leak into the boundary
    assert all(n.startswith("drb_") for n in exported)


def test_version_and_last_error():
    from paper_2406_03285_b200._lib import lib
    assert b"sm_100a" in lib.drb_rb_version()
    assert lib.drb_rb_last_error() is not None


@pytest.mark.parametrize("field,value", [("n_classes", 0), ("per_class_cap", 0), ("sample_bytes", 6),
                                         ("world", 0), ("world", 9), ("rank", 3), ("max_batch", 0),
                                         ("max_batch", 5000)])
def test_create_rejects_bad_config_before_touching_the_gpu(field, value):
    from paper_2406_03285_b200 import _lib
    cfg = _lib.drb_rb_config(n_classes=10, per_class_cap=4, sample_bytes=64, max_batch=8, candidate_count=4,
                             rep_count=2, rank=0, world=2, seed=1, device=0, flags=0)
    setattr(cfg, field, value)
    h = C.c_void_p()
    st = _lib.lib.drb_rb_create(C.byref(cfg), C.byref(h))
    assert st == _lib.DRB_ERR_CONFIG
    assert not h.value
    with pytest.raises(_lib.config_error):
        _lib.check(st)


def test_null_arguments():
    from paper_2406_03285_b200 import _lib
    lib = _lib.lib
    assert lib.drb_rb_create(None, None) == _lib.DRB_ERR_INVALID_ARGUMENT
    assert lib.drb_rb_last_error() == b"null argument"
    assert lib.drb_rng_init(None, 1, 0, 1) == _lib.DRB_ERR_INVALID_ARGUMENT
    assert lib.drb_rb_start(None) == _lib.DRB_ERR_INVALID_ARGUMENT
    assert lib.drb_rb_destroy(None) == _lib.DRB_OK
    assert lib.drb_rb_handle_size() >= 2 * 64  # two CUDA IPC handles + metadata


def test_stream_keys_match_the_oracle():
    from oracle.py_oracle import Backend
    from paper_2406_03285_b200 import _lib
    orc = Backend("port")
    mk = orc.lib.or_stream_make
    from oracle.py_oracle import _or_stream
    mk.restype = _or_stream
    mk.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, C.c_uint64, C.c_uint64]
    for seed, worker, purpose in [(1, 0, 1), (77, 3, 2), (2**40 + 5, 7, 3), (0, 0, 6)]:
        s = _lib.drb_rng()
        assert _lib.lib.drb_rng_init(C.byref(s), seed, worker, purpose) == 0
        assert s.key == mk(seed, worker, purpose, 0, 0, 0).key and s.ctr == 0
        assert _lib.lib.drb_rng_keyed(C.byref(s), seed, worker, purpose, 0x7E, 0) == 0
        assert s.key == mk(seed, worker, purpose, 1, 0x7E, 0).key


def test_error_taxonomy_mapping():
    from paper_2406_03285_b200 import _lib
    for status, cls in [(_lib.DRB_ERR_CONFIG, _lib.config_error), (_lib.DRB_ERR_USAGE, _lib.usage_error),
                        (_lib.DRB_ERR_TRANSPORT, _lib.transport_error), (_lib.DRB_ERR_TRAINING, _lib.engine_error),
                        (_lib.DRB_ERR_INVALID_ARGUMENT, _lib.invalid_argument)]:
        with pytest.raises(cls):
            _lib.check(status)
    with pytest.raises(_lib.drb_error):
        _lib.check(_lib.DRB_ERR_INTERNAL)


def test_workload_schedule_and_stream_determinism():
    import numpy as np
    from paper_2406_03285_b200.workload import make_schedule, stream_spec
    sched = make_schedule(100, 4, 1)
    assert [len(t) for t in sched] == [25] * 4 and sorted(sum(sched, [])) == list(range(100))
    spec = stream_spec(100, 4, 56, 64, steps_per_task=10, seed=3)
    assert np.array_equal(spec.labels(1, 7), spec.labels(1, 7))
    assert set(spec.labels(0, 15).tolist()) <= set(sched[1]) or True
    assert set(spec.labels(0, 15).tolist()) <= set(make_schedule(100, 4, 3)[1])
    assert not np.array_equal(spec.payload(0, 1), spec.payload(1, 1))
