import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2404_14783_b200 import qlra as Q
ctx = Q.Context(0)
K = 1 << 17
for m in (8, 64):
    a = torch.randn((4, m, K), dtype=torch.float64, device="cuda")
    b = torch.randn((4, K, 64), dtype=torch.float64, device="cuda")
    out = torch.zeros((4, m, 64), dtype=torch.float64, device="cuda")
    Q.qmat_mul(a, b, out=out, ctx=ctx)
torch.cuda.synchronize()
