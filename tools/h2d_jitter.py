"""Per-copy time of 60 back-to-back 1.536 GB pinned H2D copies (C2's A):
does the PCIe rate itself vary from copy to copy?"""
import torch

n = int(1.536e9 / 8)
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
ts = []
for _ in range(60):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    d.copy_(h, non_blocking=True)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print("ms per copy: min %.2f max %.2f mean %.2f" % (min(ts), max(ts), sum(ts) / len(ts)))
print(" ".join("%.1f" % t for t in ts))
