"""drb-b200: B200-native distributed rehearsal-buffer hot path (arXiv 2406.03285).

The product is libdrb_b200.so (sm_100a CUDA + C ABI, include/drb_rb.h). This package is
the Python mirror of the reference's C++ API over that ABI. Importing it without the
built library raises ImportError — there is no CPU fallback.
"""
from ._lib import (config_error, drb_error, engine_error, invalid_argument, transport_error,  # noqa: F401
                   usage_error)
from .rehearsal import (augment, augmented_batch, bias_report, bias_test, engine, insertion_report, occupancy_snapshot,  # noqa: F401
                        plan, read_entry, rehearsal_buffer, rng_stream, sample_without_replacement,
                        sampling_plan)

from . import dataset  # noqa: E402,F401  (the producer of m: DRDS load, schedule, shards, device gather)

__all__ = [
    "rehearsal_buffer", "engine", "rng_stream", "plan", "augment", "sample_without_replacement", "bias_test",
    "bias_report",
    "augmented_batch", "insertion_report", "occupancy_snapshot", "read_entry", "sampling_plan",
    "config_error", "usage_error", "engine_error", "transport_error", "invalid_argument", "drb_error",
]
