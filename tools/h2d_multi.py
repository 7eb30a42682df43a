"""Does splitting one H2D copy across 1, 2 or 4 streams (copy engines) raise
the pinned host -> device rate?"""
import torch

gb = 1.536
n = int(gb * 1e9 / 8)
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    parts = [(i * n // k, (i + 1) * n // k) for i in range(k)]

    def go():
        for s, (a, b) in zip(streams, parts):
            with torch.cuda.stream(s):
                d[a:b].copy_(h[a:b], non_blocking=True)
        for s in streams:
            s.synchronize()
    go()
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    for _ in range(3):
        go()
    ms = (time.perf_counter() - t0) / 3 * 1e3
    print(f"{k} stream(s): {ms:.2f} ms  {gb / ms * 1e3:.1f} GB/s")
