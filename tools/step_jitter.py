"""Per-step times of the device-resident one-pass and of the host API, to
expose run-to-run jitter (bench.py reports means)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14783_b200 import configs, qlra as Q  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ctx = Q.Context(0)
a = configs.build_matrix(cfg, ctx=ctx)
torch.cuda.synchronize()
torch.cuda.empty_cache()
o = Q.resolve_defaults(Q.OnePassOptions(r=cfg.s - 5, s=cfg.s, l=cfg.l, embedding=cfg.kind))
dev, host = [], []
for i in range(n):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = Q.make_sketch(a, o.r, o.s, o.l, o.omega_seed, o.psi_seed, o.embedding, ctx=ctx)
    Q.qb_stage(st, o.rangefinder, ctx=ctx)
    torch.cuda.synchronize()
    dev.append(1e3 * (time.perf_counter() - t0))
a_host = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
a_host.copy_(a)
for i in range(n):
    t0 = time.perf_counter()
    Q.one_pass_qb_host(a_host, o, ctx=ctx)
    host.append(1e3 * (time.perf_counter() - t0))
print("device-resident ms:", " ".join("%.1f" % v for v in dev))
print("host API ms       :", " ".join("%.1f" % v for v in host))
