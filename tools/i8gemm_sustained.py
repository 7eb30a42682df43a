"""Sustained behaviour of the tcgen05 int8 GEMM under the power cap: per-rep
times of the C4 W* (or Y) product over ~2 s with nvidia-smi clocks / power
sampled beside it.  python tools/i8gemm_sustained.py [w|y] [reps]"""
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
from paper_2404_14783_b200 import qlra as Q  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "w"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 80
    rpad, npad, spad, lpad, nb = 7856, 27136, 512, 1008, 120
    rpi = (rpad + 127) // 128 * 128
    ctx = Q.Context(0)
    ares = torch.randint(-128, 128, (nb, rpad, npad), dtype=torch.int8, device="cuda")
    if which == "w":
        bop = torch.randint(-128, 128, (nb, lpad, rpi), dtype=torch.int8, device="cuda")
        c = torch.zeros((nb, lpad, npad), dtype=torch.int32, device="cuda")
        args = (1, npad, lpad, rpad, ares.data_ptr(), npad, rpad * npad, bop.data_ptr(), rpi, lpad * rpi, c.data_ptr(),
                npad, npad * lpad, nb, 1)
        ops = 2.0 * nb * rpad * npad * lpad
    else:
        bop = torch.randint(-128, 128, (nb, spad, npad), dtype=torch.int8, device="cuda")
        c = torch.zeros((nb, rpad, spad), dtype=torch.int32, device="cuda")
        args = (0, rpad, spad, npad, ares.data_ptr(), npad, rpad * npad, bop.data_ptr(), npad, spad * npad, c.data_ptr(),
                spad, rpad * spad, nb, 0)
        ops = 2.0 * nb * rpad * npad * spad
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                                "--format=csv,noheader,nounits", "-i", "0"], capture_output=True, text=True)
            samples.append((time.perf_counter(), r.stdout.strip()))
    th = threading.Thread(target=sampler)
    th.start()
    ts = []
    t00 = time.perf_counter()
    for _ in range(reps):
        t0 = time.perf_counter()
        ctx._check(ctx.lib.qlra_i8gemm_batched(ctx.h, *args))
        ctx.synchronize()
        ts.append(time.perf_counter() - t0)
    stop.set()
    th.join()
    k = max(1, reps // 8)
    print("per-rep ms (means of", k, "):", " ".join(f"{sum(ts[i:i + k]) / len(ts[i:i + k]) * 1e3:.2f}" for i in range(0, reps, k)))
    print(f"last quarter: {ops / (sum(ts[-reps // 4:]) / (reps // 4)) / 1e12:.0f} TOPS")
    for t, s in samples[:: max(1, len(samples) // 12)]:
        print(f"  t={t - t00:5.2f}s  {s}")


if __name__ == "__main__":
    main()
