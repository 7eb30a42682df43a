"""One C2-sized sketch (Omega/Psi generation + both products) for ncu.
A comes from torch.randn so the first two qgemm launches are Y then W."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14783_b200 import qlra as Q  # noqa: E402

m, n, s, l = (int(x) for x in (sys.argv[1:5] if len(sys.argv) >= 5 else (8000, 6000, 100, 200)))
reps = int(sys.argv[5]) if len(sys.argv) >= 6 else 1
ctx = Q.Context(0)
torch.manual_seed(0)
a = torch.randn((4, m, n), dtype=torch.float64, device="cuda")
for _ in range(reps):
    st = Q.make_sketch(a, s - 5, s, l, 1, 2, ctx=ctx)
torch.cuda.synchronize()
print("ok", float(st.y.norm()), float(st.w.norm()))
