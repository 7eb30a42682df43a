"""C3 pseudo-SVD parity diagnosis: where does the device / oracle QB-error
difference come from -- the basis H or the core solve?  Cross-combines
device and oracle H with device and oracle solves and prints the QB errors,
orthonormality defects and principal angles."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2404_14783_b200 import configs, qlra as Q  # noqa: E402
from tests.test_gpu_configs import principal_angle_sin  # noqa: E402
from tests.helpers import orthonormality_defect  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
ctx = Q.Context(0)
a = configs.build_matrix(cfg, ctx=ctx)
st = Q.make_sketch(a, cfg.s - 5, cfg.s, cfg.l, 1, 2, cfg.kind, ctx=ctx)
yh, wh = st.y.cpu().numpy(), st.w.cpu().numpy()
dev = lambda x: torch.as_tensor(np.ascontiguousarray(x), device="cuda")  # noqa: E731


def err(h, x):
    r, n = Q.residual_fro(a, h, x, ctx)
    return r / n


t = time.time()
qo = O.qb_stage(yh, wh, 2, 1, kind=cfg.kind, nthreads=os.cpu_count())
print("oracle qb", time.time() - t, flush=True)
ho, xo = dev(qo["h"]), dev(qo["x"])
hd = Q.pseudo_svd(st.y, ctx=ctx).h
xd = Q.qb_solve(st.psi_spec, hd, st.w, 0, ctx)
x_od = Q.qb_solve(st.psi_spec, ho, st.w, 0, ctx)  # oracle H, device solve
psi = O.gen_test_matrix(cfg.kind, cfg.l, cfg.m, 2, nthreads=os.cpu_count())
hdh = hd.cpu().numpy()
x_do = O.solve_quaternion_linear(O.qmat_mul(psi, hdh), wh)  # device H, oracle solve
e_oo, e_dd, e_od, e_do = err(ho, xo), err(hd, xd), err(ho, x_od), err(hd, dev(x_do))
print(f"QB err  oracle H/oracle solve {e_oo:.15e}")
print(f"        device H/device solve {e_dd:.15e}  rel {abs(e_dd / e_oo - 1):.2e}")
print(f"        oracle H/device solve {e_od:.15e}  rel {abs(e_od / e_oo - 1):.2e}")
print(f"        device H/oracle solve {e_do:.15e}  rel {abs(e_do / e_oo - 1):.2e}")
print("orthonormality defect device", orthonormality_defect(hdh), "oracle", orthonormality_defect(qo["h"]))
print("angle", principal_angle_sin(hd, ho))
sv = Q.singular_values(st.y, ctx)
print("kappa(Y)", sv[0] / sv[-1], "sigma tail", sv[-22:])
