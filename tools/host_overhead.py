"""Wall clock vs device time of make_sketch (host-side overhead probe)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14783_b200 import configs, qlra as Q  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
ctx = Q.Context(0)
a = configs.build_matrix(cfg, ctx=ctx)
o = Q.resolve_defaults(Q.OnePassOptions(r=cfg.s - 5, s=cfg.s, l=cfg.l, embedding=cfg.kind))
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = Q.empty_sketch(cfg.m, cfg.n, o.r, o.s, o.l, o.omega_seed, o.psi_seed, o.embedding, o.density)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    Q.sketch_update_rows(st, 0, a, ctx)
    t2 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"alloc {1e3*(t1-t0):.1f} ms  launch-return {1e3*(t2-t1):.1f} ms  wall {1e3*(t3-t1):.1f} ms  "
          f"device {e0.elapsed_time(e1):.1f} ms")
