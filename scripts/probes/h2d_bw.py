"""Pinned host -> device copy bandwidth on this box (context for the e2e number)."""
import json
import torch

x = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
y = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for _ in range(3):
    y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    y.copy_(x, non_blocking=True)
e1.record()
torch.cuda.synchronize()
h2d = 10 * x.numel() / (e0.elapsed_time(e1) / 1e3) / 1e9
e0.record()
for _ in range(10):
    x.copy_(y, non_blocking=True)
e1.record()
torch.cuda.synchronize()
d2h = 10 * x.numel() / (e0.elapsed_time(e1) / 1e3) / 1e9
print(json.dumps({"h2d_GBps": h2d, "d2h_GBps": d2h}))
