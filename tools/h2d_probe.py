"""Pinned host -> device copy bandwidth (the e2e floor for host-resident A)."""
import torch

for gb in (1.536, 8.0):
    n = int(gb * 1e9 / 8)
    h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    h.fill_(1.0)
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"H2D {gb:.2f} GB: {ms:.2f} ms  {gb / ms * 1e3:.1f} GB/s")
    h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
    e0.record()
    h2.copy_(d, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"D2H {gb:.2f} GB: {ms:.2f} ms  {gb / ms * 1e3:.1f} GB/s")
    del h, h2, d
