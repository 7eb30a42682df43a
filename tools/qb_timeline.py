"""Kernel timeline (start offset, duration, stream) of one QB stage call.

usage: python tools/qb_timeline.py C2 [method] [split]
"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14783_b200 import configs, qlra as Q  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
method = int(sys.argv[2]) if len(sys.argv) > 2 else 0
split = len(sys.argv) > 3 and sys.argv[3] == "split"
ctx = Q.Context(0)
a = configs.build_matrix(cfg, ctx=ctx)
st = Q.make_sketch(a, cfg.s - 5, cfg.s, cfg.l, 1, 2, kind=cfg.kind, ctx=ctx)
for _ in range(3):
    Q.qb_stage(st, method, ctx=ctx, split=split)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    Q.qb_stage(st, method, ctx=ctx, split=split)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start if ev else 0
end = 0
for e in ev:
    s, d = e.time_range.start - t0, e.time_range.end - e.time_range.start
    end = max(end, s + d)
    print("%9.1f %8.1f  %-4s %s" % (s, d, getattr(e, "device_resource_id", "?"), e.name[:70]))
print("span %.1f us" % end)
