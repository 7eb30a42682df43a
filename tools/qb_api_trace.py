"""CUDA runtime API calls (CUPTI, via the torch profiler) of one QB stage:
where the host time at the start of the call goes.
usage: python tools/qb_api_trace.py C5 [method]"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14783_b200 import configs, qlra as Q  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
method = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ctx = Q.Context(0)
a = configs.build_matrix(cfg, ctx=ctx)
st = Q.make_sketch(a, cfg.s - 5, cfg.s, cfg.l, 1, 2, kind=cfg.kind, ctx=ctx)
for _ in range(3):
    Q.qb_stage(st, method, ctx=ctx)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    Q.qb_stage(st, method, ctx=ctx)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type != torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev[:80]:
    d = e.time_range.end - e.time_range.start
    print("%9.1f %8.1f %s" % (e.time_range.start - t0, d, e.name[:60]))
