"""One QB stage of a config between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` captures of its kernels.

usage: python tools/prof_qb.py C5 [method]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14783_b200 import configs, qlra as Q  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
method = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ctx = Q.Context(0)
a = configs.build_matrix(cfg, ctx=ctx)
st = Q.make_sketch(a, cfg.s - 5, cfg.s, cfg.l, 1, 2, kind=cfg.kind, ctx=ctx)
for _ in range(2):
    Q.qb_stage(st, method, ctx=ctx)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
Q.qb_stage(st, method, ctx=ctx)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
