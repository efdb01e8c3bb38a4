"""Pinned host->device copy bandwidth on this box (the e2e input path's bound):
one 77.6 MB AlexNet shard (128x224x224x3 fp32) per copy, alone and while the GPU computes."""
import time

import torch

n = 128 * 224 * 224 * 3
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
for label, busy in (("idle", False), ("under compute", True)):
    a = torch.randn(8192, 8192, device="cuda")
    torch.cuda.synchronize()
    if busy:
        for _ in range(200):
            a @ a  # keep the default stream busy
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(10):
            d.copy_(h, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"H2D {label}: {ms:.3f} ms per 77.6 MB = {n * 4 / ms / 1e6:.1f} GB/s")
t0 = time.perf_counter()
hd = torch.empty(n, dtype=torch.float32).pin_memory()
e0.record()
for _ in range(10):
    hd.copy_(d, non_blocking=True)
e1.record()
torch.cuda.synchronize()
print(f"D2H: {n * 4 / (e0.elapsed_time(e1) / 10) / 1e6:.1f} GB/s")
