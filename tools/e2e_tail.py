"""Kernel timeline of the last ~120 ms of one host-in/host-out one-pass call
(qlra_one_pass_qb_host): what runs after the last chunk of A arrives.
usage: python tools/e2e_tail.py C4"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14783_b200 import configs, qlra as Q  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
ctx = Q.Context(0)
a = configs.build_matrix(cfg, ctx=ctx)
a_host = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
a_host.copy_(a)
del a
torch.cuda.empty_cache()
opts = Q.OnePassOptions(r=cfg.s - 5, s=cfg.s, l=cfg.l, embedding=cfg.kind)
h_host = torch.empty((4, cfg.m, cfg.s), dtype=torch.float64, pin_memory=True)
x_host = torch.empty((4, cfg.s, cfg.n), dtype=torch.float64, pin_memory=True)
for _ in range(2):
    Q.one_pass_qb_host(a_host, opts, ctx=ctx, h_out=h_host, x_out=x_host)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    Q.one_pass_qb_host(a_host, opts, ctx=ctx, h_out=h_host, x_out=x_host)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
end = max(e.time_range.end for e in ev)
last_h2d = max((e.time_range.end for e in ev if "HtoD" in e.name), default=t0)
print("span %.1f ms, last H2D ends at %.1f ms" % ((end - t0) / 1e3, (last_h2d - t0) / 1e3))
for e in ev:
    if e.time_range.end >= last_h2d - 5000 and (e.time_range.end - e.time_range.start) > 150:
        print("%9.1f %8.1f %-4s %s" % ((e.time_range.start - t0) / 1e3, (e.time_range.end - e.time_range.start) / 1e3,
                                      getattr(e, "device_resource_id", "?"), e.name[:70]))
