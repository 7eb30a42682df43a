"""pseudo-QR on a config's sketch: fused QB stage, split calls, and the
oracle's kappa/steps (QLRA_DEBUG_PQR=1 prints the device's internals)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14783_b200 import configs, qlra as Q  # noqa: E402

os.environ.setdefault("QLRA_DEBUG_PQR", "1")
cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
ctx = Q.Context(0)
a = configs.build_matrix(cfg, ctx=ctx)
st = Q.make_sketch(a, cfg.s - 5, cfg.s, cfg.l, 1, 2, kind=cfg.kind, ctx=ctx)
for name, fn in [("pseudo_qr", lambda: Q.pseudo_qr(st.y, ctx=ctx)),
                 ("qb fused", lambda: Q.qb_stage(st, ctx=ctx).report),
                 ("qb split", lambda: Q.qb_stage(st, ctx=ctx, split=True).report)]:
    try:
        r = fn()
        print(name, "kappa %.6e -> %.6e steps %d" % (r.kappa_before, r.kappa_after, r.correction_steps_used))
    except Q.Error as e:
        print(name, "ERROR", e)
if len(sys.argv) > 2 and sys.argv[2] == "oracle":
    from oracle import oracle as O
    y = st.y.cpu().numpy()
    ro = O.pseudo_qr(y)
    print("oracle pseudo_qr kappa %.6e -> %.6e steps %d" % (ro["kappa_before"], ro["kappa_after"],
                                                             ro["correction_steps_used"]))
