"""C3 diagnostics: kappa of the device sketch Y and whether the reference's
pseudo-QR (CPU oracle) accepts it."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2404_14783_b200 import configs, qlra as Q  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
ctx = Q.Context(0)
a = configs.build_matrix(cfg, ctx=ctx)
st = Q.make_sketch(a, cfg.s - 5, cfg.s, cfg.l, 1, 2, cfg.kind, ctx=ctx)
y = st.y.cpu().numpy()
sv = Q.singular_values(st.y, ctx)
print("device sigma(Y): max %.4e min %.4e kappa %.4e" % (sv[0], sv[-1], sv[0] / sv[-1]))
print("sigma tail", sv[-25:])
t = time.time()
try:
    r = O.pseudo_qr(y)
    print("oracle pseudo_qr OK", r["kappa_before"], r["kappa_after"], r["correction_steps_used"], time.time() - t)
except O.OracleError as e:
    print("oracle pseudo_qr raised", e.kind, e, time.time() - t)
r0 = O.pseudo_qr(y, max_steps=0)
print("oracle QR-only kappa(H0)", r0["kappa_before"])
try:
    g = Q.pseudo_qr(st.y, Q.PseudoQrConfig(max_correction_steps=0), ctx=ctx)
    print("device QR-only kappa(H0)", g.kappa_before)
except Exception as e:
    print("device QR-only raised", e)
