"""Parity diagnostics: isolates sketch vs rangefinder vs solve deviations
between the device path and the CPU oracle on a config (default C1)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2404_14783_b200 import configs, qlra as Q  # noqa: E402
from tests.helpers import largest_principal_angle  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
cfg = configs.CONFIGS[name]
ctx = Q.Context(0)
a = configs.build_matrix(cfg, ctx=ctx)
ah = a.cpu().numpy()
nt = os.cpu_count() or 1
st = Q.make_sketch(a, cfg.s - 5, cfg.s, cfg.l, 1, 2, cfg.kind, ctx=ctx)
yg, wg = st.y.cpu().numpy(), st.w.cpu().numpy()
yo, wo = O.make_sketch(ah, cfg.s - 5, cfg.s, cfg.l, 1, 2, cfg.kind, nthreads=nt)
print("sketch rel diff y %.2e w %.2e" % (np.linalg.norm(yg - yo) / np.linalg.norm(yo),
                                        np.linalg.norm(wg - wo) / np.linalg.norm(wo)))
for method in (0, 1):
    qg = Q.qb_stage(st, method, ctx=ctx)
    rg, ag = Q.residual_fro(a, qg.h, qg.x, ctx)
    eg = rg / ag
    qo = O.qb_stage(yo, wo, 2, method, kind=cfg.kind, nthreads=nt)
    rs, an = O.residual_sq(ah, qo["h"], qo["x"])
    eo = np.sqrt(rs / an)
    qx = O.qb_stage(yg, wg, 2, method, kind=cfg.kind, nthreads=nt)  # oracle on GPU sketch
    rs2, _ = O.residual_sq(ah, qx["h"], qx["x"])
    ex = np.sqrt(rs2 / an)
    hg = qg.h.cpu().numpy()
    # GPU H, oracle-computed X (solve isolation)
    xo_on_hg = O.solve_quaternion_linear(O.qmat_mul(O.gen_test_matrix(cfg.kind, cfg.l, cfg.m, 2), hg), wg)
    rs3, _ = O.residual_sq(ah, hg, xo_on_hg)
    print(f"method {method}: err gpu {eg:.15e} oracle {eo:.15e} oracle(gpu sketch) {ex:.15e}"
          f" gpuH+oracleX {np.sqrt(rs3/an):.15e}")
    print(f"   ratios-1: gpu/oracle {eg/eo-1:.2e}  oracle(gpuY)/oracle {ex/eo-1:.2e}  gpu/oracle(gpuY) {eg/ex-1:.2e}"
          f"  gpuH+oX/oracle(gpuY) {np.sqrt(rs3/an)/ex-1:.2e}")
    print(f"   angles: H_gpu vs H_oracle {largest_principal_angle(hg, qo['h']):.2e}, "
          f"H_gpu vs Y_gpu {largest_principal_angle(hg, yg):.2e}, H_orc vs Y_orc {largest_principal_angle(qo['h'], yo):.2e}")
    print(f"   kappa gpu {qg.report.kappa_before:.6e}/{qg.report.kappa_after:.6e} steps {qg.report.correction_steps_used}"
          f"  oracle {qo['kappa_before']:.6e}/{qo['kappa_after']:.6e} steps {qo['correction_steps_used']}")

if os.environ.get("DIAG_SAVE"):
    out = os.path.join(os.environ["DIAG_SAVE"], f"diag_{name}.npz")
    q0 = Q.qb_stage(st, 0, ctx=ctx)
    q1 = Q.qb_stage(st, 1, ctx=ctx)
    np.savez(out, a=ah, y=yg, w=wg, h0=q0.h.cpu().numpy(), x0=q0.x.cpu().numpy(),
             h1=q1.h.cpu().numpy(), x1=q1.x.cpu().numpy())
    print("saved", out)
