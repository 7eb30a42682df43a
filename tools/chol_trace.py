"""Drive the cluster Cholesky+inverse on a 100x100 HPD quaternion matrix
(solve_quaternion_linear -> CholeskyQR2 of a 140x100 matrix); with the
QLRA_CHC_TRACE build (tools: _ab/libqlra_cuda_trace.so) the kernel prints
per-block-step phase cycles from CTA 0."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14783_b200 import qlra as Q  # noqa: E402

ctx = Q.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
a = torch.randn((4, n + 40, n), dtype=torch.float64, device="cuda")
b = torch.randn((4, n + 40, 2), dtype=torch.float64, device="cuda")
for _ in range(2):
    Q.solve_quaternion_linear(a, b, ctx)
torch.cuda.synchronize()
