"""Per-stream timeline of one one_pass_qb_host call (A in pinned memory):
busy time per stream and kernel/memcpy class, plus the span.

usage: python tools/host_timeline.py C5 [method]
"""
import collections
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
a_host = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
a_host.copy_(a)
del a
torch.cuda.empty_cache()
h_host = torch.empty((4, cfg.m, cfg.s), dtype=torch.float64, pin_memory=True)
x_host = torch.empty((4, cfg.s, cfg.n), dtype=torch.float64, pin_memory=True)
opts = Q.OnePassOptions(r=cfg.s - 5, s=cfg.s, l=cfg.l, rangefinder=method, embedding=cfg.kind)
import time
for _ in range(int(os.environ.get("REPS", "2"))):
    t0 = time.perf_counter()
    Q.one_pass_qb_host(a_host, opts, ctx=ctx, h_out=h_host, x_out=x_host)
    torch.cuda.synchronize()
    print("wall %.1f ms" % (1e3 * (time.perf_counter() - t0)))
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    Q.one_pass_qb_host(a_host, opts, ctx=ctx, h_out=h_host, x_out=x_host)
    torch.cuda.synchronize()
    print("profiled wall %.1f ms" % (1e3 * (time.perf_counter() - t0)))
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
busy = collections.defaultdict(float)
first = {}
last = {}
for e in ev:
    key = (getattr(e, "device_resource_id", "?"), e.name.split("(")[0][-40:])
    busy[key] += e.time_range.end - e.time_range.start
    first.setdefault(key, e.time_range.start - t0)
    last[key] = e.time_range.end - t0
for k in sorted(busy, key=lambda k: first[k]):
    print("stream %-4s %-42s busy %9.1f us  [%9.1f .. %9.1f]" % (k[0], k[1], busy[k], first[k], last[k]))
print("span %.1f us" % (max(last.values())))
