"""Per-kernel device time of the QB stages (CUPTI via torch.profiler).

usage: python tools/kernel_breakdown.py C2 [method]
Sketches once, then profiles the rangefinder and the core solve separately
and prints, per stage, kernels sorted by total device time.
"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14783_b200 import configs, qlra as Q  # noqa: E402


def table(title, fn, reps=3):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
    rows = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            name = ev.name.replace("qlra_dev::(anonymous namespace)::", "")[:60]
            n, tot = rows.get(name, (0, 0.0))
            rows[name] = (n + 1, tot + ev.device_time_total)
    total = sum(v[1] for v in rows.values()) / reps
    print("== %s: %.1f us device per call" % (title, total))
    for name, (n, tot) in sorted(rows.items(), key=lambda kv: -kv[1][1])[:25]:
        print("  %-62s %5.1f %9.1f" % (name, n / reps, tot / reps))


cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
method = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ctx = Q.Context(0)
a = configs.build_matrix(cfg, ctx=ctx)
o = Q.resolve_defaults(Q.OnePassOptions(r=cfg.s - 5, s=cfg.s, l=cfg.l, rangefinder=method, embedding=cfg.kind))
st = Q.make_sketch(a, o.r, o.s, o.l, o.omega_seed, o.psi_seed, o.embedding, o.density, ctx)
ctx.synchronize()
state = {}


def rangefinder():
    state["rep"] = (Q.pseudo_qr(st.y, o.qr_cfg, ctx) if method == Q.PSEUDO_QR
                    else Q.pseudo_svd(st.y, o.rangefinder_seed, ctx))


def solve():
    Q.qb_solve(st.psi_spec, state["rep"].h, st.w, st.row0, ctx)


table("sketch", lambda: Q.make_sketch(a, o.r, o.s, o.l, o.omega_seed, o.psi_seed, o.embedding, o.density, ctx), 1)
table("rangefinder", rangefinder)
table("solve", solve)
