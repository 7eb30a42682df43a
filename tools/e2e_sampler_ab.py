"""Back-to-back one_pass_qb_host calls on C2 with and without bench.py's
NVML ClockSampler thread running: does the sampler cause e2e jitter?"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2404_14783_b200 import configs, qlra as Q  # noqa: E402

cfg = configs.CONFIGS["C2"]
ctx = Q.Context(0)
a = configs.build_matrix(cfg, ctx=ctx)
a_host = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
a_host.copy_(a)
del a
torch.cuda.empty_cache()
h_host = torch.empty((4, cfg.m, cfg.s), dtype=torch.float64, pin_memory=True)
x_host = torch.empty((4, cfg.s, cfg.n), dtype=torch.float64, pin_memory=True)
opts = Q.OnePassOptions(r=cfg.s - 5, s=cfg.s, l=cfg.l, embedding=cfg.kind)


def run(n):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        Q.one_pass_qb_host(a_host, opts, ctx=ctx, h_out=h_host, x_out=x_host)
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    return ts


run(3)
for label in ("plain", "sampler", "plain", "sampler"):
    if label == "sampler":
        with bench.ClockSampler(0):
            ts = run(40)
    else:
        ts = run(40)
    print("%-8s mean %.2f max %.2f  n>+1ms %d" % (label, sum(ts) / len(ts), max(ts), sum(t > min(ts) + 1 for t in ts)))
