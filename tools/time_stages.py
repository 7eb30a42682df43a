"""Wall-clock split of one one-pass LRA (sketch / rangefinder / solve)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14783_b200 import configs, qlra as Q  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
method = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ctx = Q.Context(0)
a = configs.build_matrix(cfg, ctx=ctx)
opts = Q.OnePassOptions(r=cfg.s - 5, s=cfg.s, l=cfg.l, rangefinder=method, embedding=cfg.kind)
for it in range(6):
    r = Q.one_pass_qb(a, opts, ctx=ctx, residual=False)
    if it >= 2:
        t = r.times
        print("sketch %.2f ms  rangefinder %.2f ms  solve %.2f ms  steps %d kappa %.3e/%.3e" % (
            1e3 * t["sketch_s"], 1e3 * t["rangefinder_s"], 1e3 * t["solve_s"], r.qb.report.correction_steps_used,
            r.qb.report.kappa_before, r.qb.report.kappa_after))
# the QB stage as one fused call vs rangefinder + solve as two calls
st = r.state
for it in range(4):
    f = Q.qb_stage(st, method, ctx=ctx)
    s = Q.qb_stage(st, method, ctx=ctx, split=True)
    if it >= 1:
        print("qb fused %.2f ms   split: rangefinder %.2f + solve %.2f = %.2f ms" % (
            1e3 * f.rangefinder_s, 1e3 * s.rangefinder_s, 1e3 * s.solve_s, 1e3 * (s.rangefinder_s + s.solve_s)))
