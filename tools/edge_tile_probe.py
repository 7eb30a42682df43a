"""How fast does a DMMA tile with few valid 8x8 blocks run?  One 64x64 output
tile (M x 64, M in 8..64) at large K (split over 64 CTAs), timed with CUDA
events: an ideal pipe-bound tile would scale with M / 64."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14783_b200 import qlra as Q  # noqa: E402

ctx = Q.Context(0)
K = 1 << 17
for m in (64, 48, 32, 16, 8):
    a = torch.randn((4, m, K), dtype=torch.float64, device="cuda")
    b = torch.randn((4, K, 64), dtype=torch.float64, device="cuda")
    out = torch.zeros((4, m, 64), dtype=torch.float64, device="cuda")
    for _ in range(3):
        Q.qmat_mul(a, b, out=out, ctx=ctx)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        Q.qmat_mul(a, b, out=out, ctx=ctx)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    tf = 32.0 * m * 64 * K / (ms * 1e-3) / 1e12
    print(f"M={m:3d}  {ms:8.3f} ms   useful {tf:6.2f} TF/s")
