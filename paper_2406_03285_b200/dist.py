"""Multi-rank wiring over torch.distributed (plumbing only: the data path is the CUDA
kernels pushing over NVLink). Replaces the reference's worker_mesh roster/connect step
(proj/src/runner/mesh.cpp:12-81): every rank all-gathers the opaque handle blobs of the
peer-shareable regions (CUDA IPC) and maps them."""
from __future__ import annotations

from typing import List, Optional

import torch
import torch.distributed as dist


def exchange_blobs(blob: bytes, group: Optional[dist.ProcessGroup] = None) -> List[bytes]:
    """All-gather one fixed-size byte blob per rank, in rank order (any backend)."""
    world = dist.get_world_size(group)
    t = torch.frombuffer(bytearray(blob), dtype=torch.uint8)
    backend = dist.get_backend(group)
    if backend == "nccl":
        t = t.cuda()
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [bytes(o.cpu().numpy().tobytes()) for o in out]


def connect_world(buffer, group: Optional[dist.ProcessGroup] = None) -> None:
    """Map every rank's region + slab into `buffer` (a rehearsal_buffer with world > 1)."""
    blobs = exchange_blobs(buffer.export_handle(), group)
    if len(blobs) != buffer.world:
        raise ValueError(f"process group has {len(blobs)} ranks, buffer was created for {buffer.world}")
    buffer.connect(blobs)
