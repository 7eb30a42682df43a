"""H2D bandwidth from pinned host memory with 1, 2 and 4 concurrent copy
streams (is one DMA stream the PCIe limit?)."""
import torch

n = 4 * 2**30 // 8
src = torch.empty(n, dtype=torch.float64, pin_memory=True)
src.fill_(1.0)
dst = torch.empty(n, dtype=torch.float64, device="cuda")
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in streams:
            s.wait_event(e0)
        chunk = n // k
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dst[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            e1.wait(s) if False else torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
    print(f"{k} stream(s): {n * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s", flush=True)
