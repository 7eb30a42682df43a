"""GPU idle gaps inside one rangefinder + solve call (CUPTI timeline via
torch.profiler): the sum of kernel/memcpy busy time vs the wall span, and
the largest gaps with the kernel that follows each."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14783_b200 import configs, qlra as Q  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
method = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ctx = Q.Context(0)
a = configs.build_matrix(cfg, ctx=ctx)
o = Q.resolve_defaults(Q.OnePassOptions(r=cfg.s - 5, s=cfg.s, l=cfg.l, rangefinder=method, embedding=cfg.kind))
st = Q.make_sketch(a, o.r, o.s, o.l, o.omega_seed, o.psi_seed, o.embedding, o.density, ctx)
for _ in range(2):
    Q.qb_stage(st, method, ctx=ctx)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    Q.qb_stage(st, method, ctx=ctx)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end, e.name[:50]) for e in ev)
busy, last_end, gaps = 0.0, None, []
span0, span1 = iv[0][0], max(e for _, e, _ in iv)
merged_end = iv[0][0]
for s0, s1, nm in iv:
    if s0 > merged_end:
        gaps.append((s0 - merged_end, nm))
    busy += max(0.0, s1 - max(s0, merged_end))
    merged_end = max(merged_end, s1)
print("span %.1f us  busy %.1f us  idle %.1f us  kernels %d" % (span1 - span0, busy, span1 - span0 - busy, len(iv)))
for g, nm in sorted(gaps, reverse=True)[:15]:
    print("  gap %7.1f us before %s" % (g, nm.replace("qlra_dev::(anonymous namespace)::", "")))
