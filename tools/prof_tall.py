"""One tall x small quaternion product (C5's Y R^-1 shape: 2097152 x 40 by
40 x 40) through qmat_mul -> the 8-product engine's multi-tile stream."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14783_b200 import qlra as Q  # noqa: E402

m, s = (int(x) for x in (sys.argv[1:3] if len(sys.argv) >= 3 else (2097152, 40)))
ctx = Q.Context(0)
torch.manual_seed(0)
y = torch.randn((4, m, s), dtype=torch.float64, device="cuda")
r = torch.randn((4, s, s), dtype=torch.float64, device="cuda")
for _ in range(3):
    h = Q.qmat_mul(y, r, ctx=ctx)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    h = Q.qmat_mul(y, r, ctx=ctx)
e1.record()
torch.cuda.synchronize()
print("ok %.3f ms per product" % (e0.elapsed_time(e1) / 5), float(h.norm()))
