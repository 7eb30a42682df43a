"""Host-streamed sketch vs a plain pinned copy of the same A (C2 by default)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_14783_b200 import configs, qlra as Q  # noqa: E402

cfg = configs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
ctx = Q.Context(0)
a = configs.build_matrix(cfg, ctx=ctx)
a_host = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
a_host.copy_(a)
o = Q.resolve_defaults(Q.OnePassOptions(r=cfg.s - 5, s=cfg.s, l=cfg.l, embedding=cfg.kind))


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


print("plain H2D copy       %.2f ms" % timed(lambda: a.copy_(a_host, non_blocking=True)))
for br in (0, 128, 512, 1024):
    t = timed(lambda: Q.make_sketch_host(a_host, o.r, o.s, o.l, o.omega_seed, o.psi_seed, o.embedding,
                                         ctx=ctx, block_rows=br))
    print("make_sketch_host br=%4d %.2f ms" % (br, t))
t = timed(lambda: Q.one_pass_qb_host(a_host, o, ctx=ctx))
print("one_pass_qb_host     %.2f ms" % t)

# the same chunked copies without any sketch work (copy-engine cost alone)
rows = 256
dev = torch.empty((4, rows, a.shape[2]), dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()


def chunked():
    with torch.cuda.stream(s):
        for r0 in range(0, a.shape[1], rows):
            rp = min(rows, a.shape[1] - r0)
            for p in range(4):
                dev[p, :rp].copy_(a_host[p, r0:r0 + rp], non_blocking=True)
    s.synchronize()


print("chunked copies only  %.2f ms" % timed(chunked))
