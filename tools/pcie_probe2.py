"""PCIe copy bandwidth from pinned host memory with the copy split into C chunks on C streams per
direction (both directions at once): does more than one DMA stream per direction help?"""
import json

import torch

n = 673 * 1024 * 1024 // 8
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]


def run(chunks, both=True):
    step = (n + chunks - 1) // chunks
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for c in range(chunks):
        lo, hi = c * step, min(n, (c + 1) * step)
        with torch.cuda.stream(streams[c % 4]):
            d_a[lo:hi].copy_(h_in[lo:hi], non_blocking=True)
        if both:
            with torch.cuda.stream(streams[4 + c % 4]):
                h_out[lo:hi].copy_(d_b[lo:hi], non_blocking=True)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


gb = n * 8 / 1e9
out = {}
for chunks in (1, 2, 4, 8, 16):
    best = min(run(chunks) for _ in range(5))
    out[f"both_each_GBps_{chunks}chunks"] = gb / (best * 1e-3)
    best1 = min(run(chunks, both=False) for _ in range(5))
    out[f"h2d_only_GBps_{chunks}chunks"] = gb / (best1 * 1e-3)
print(json.dumps(out))
