"""Time the quaternion Jacobi eigensolver through qsvd on an m x n matrix.
usage: QLRA_JACOBI_COOP=0|1 python tools/jacobi_probe.py 2000 220"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14783_b200 import qlra as Q  # noqa: E402
from oracle import oracle as O  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
ctx = Q.Context(0)
a = torch.as_tensor(O.random_gaussian(m, n, 5), device="cuda")
for _ in range(2):
    Q.qsvd(a, ctx)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    Q.qsvd(a, ctx)
    torch.cuda.synchronize()
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and "jacobi" in e.name:
        print(e.name[:60], "%.3f ms" % ((e.time_range.end - e.time_range.start) / 1000))
