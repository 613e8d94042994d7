"""Practical ceiling: device-to-device copies of the per-step byte volume, graph-captured
back to back (no launch gaps), timed with CUDA events."""
import torch
dev = torch.device("cuda:0")
S = 224 * 224 * 3
for rows in (14, 56, 63, 77, 200, 1000, 7000):
    nbytes = rows * S
    ring = max(2, (512 << 20) // nbytes)
    src = torch.randint(0, 255, (ring, nbytes), dtype=torch.uint8, device=dev)
    dst = torch.empty((ring, nbytes), dtype=torch.uint8, device=dev)
    steps = 200
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for i in range(3):
            dst[i % ring].copy_(src[i % ring])
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for i in range(steps):
                dst[i % ring].copy_(src[i % ring])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s); g.replay(); e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / steps
    print(f"copy {nbytes/1e6:8.2f} MB: {us:7.2f} us/copy, {2*nbytes/us/1e3:7.1f} GB/s (read+write)")
