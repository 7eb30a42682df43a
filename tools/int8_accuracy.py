"""Relative Frobenius difference of the sketch from the ordered oracle
sketch, both engines (printed; the tests assert the bars).
usage: python tools/int8_accuracy.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2404_14783_b200 import qlra as Q  # noqa: E402
from tests.helpers import random_gaussian, rel_diff  # noqa: E402

ctx = Q.Context(0)
for (m, n, s, l) in [(2000, 3000, 100, 200), (3000, 2500, 64, 128), (1500, 4000, 120, 240)]:
    a = random_gaussian(m, n, 7 + m)
    y, w = O.make_sketch(a, 4, s, l, 3, 4, nthreads=16)
    row = [f"{m}x{n} s={s} l={l}:"]
    for eng in ("int8", "dmma"):
        ctx.set_sketch_engine(eng)
        st = Q.make_sketch(torch.as_tensor(a, device="cuda"), 4, s, l, 3, 4, ctx=ctx)
        row.append(f"{eng} Y {rel_diff(st.y.cpu().numpy(), y):.2e} W {rel_diff(st.w.cpu().numpy(), w):.2e}")
    ctx.set_sketch_engine("auto")
    print("  ".join(row), flush=True)
