"""Times the tcgen05 int8 GEMM kernel (csrc/i8gemm.cu) on the sketch's two
products at a config's panel shape: CUDA events on the context stream.

    python tools/i8gemm_bench.py [C4|C2] [reps]
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2404_14783_b200 import qlra as Q  # noqa: E402

SHAPES = {  # rpad, npad, spad, lpad, batch
    "C4": (7856, 27136, 512, 1008, 120),
    "C2": (8000, 6000, 112, 208, 120),
    "C3": (20000, 15008, 224, 448, 120),
}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    rpad, npad, spad, lpad, nb = SHAPES[name]
    ctx = Q.Context(0)
    dev = "cuda"
    up = lambda x: (x + 127) // 128 * 128  # noqa: E731  the engine's 128-byte row pitches
    npi, rpi = up(npad), up(rpad)
    ares = torch.randint(-128, 128, (nb, rpad, npi), dtype=torch.int8, device=dev)
    ores = torch.randint(-128, 128, (nb, spad, npi), dtype=torch.int8, device=dev)
    pres = torch.randint(-128, 128, (nb, lpad, rpi), dtype=torch.int8, device=dev)
    cy = torch.zeros((nb, rpad, spad), dtype=torch.int32, device=dev)
    cw = torch.zeros((nb, lpad, npad), dtype=torch.int32, device=dev)
    torch.cuda.synchronize()

    def y():
        ctx._check(ctx.lib.qlra_i8gemm_batched(ctx.h, 0, rpad, spad, npad, ares.data_ptr(), npi, rpad * npi,
                                               ores.data_ptr(), npi, spad * npi, cy.data_ptr(), spad, rpad * spad,
                                               nb, 0))

    def w():
        ctx._check(ctx.lib.qlra_i8gemm_batched(ctx.h, 1, npad, lpad, rpad, ares.data_ptr(), npi, rpad * npi,
                                               pres.data_ptr(), rpi, lpad * rpi, cw.data_ptr(), npad, npad * lpad,
                                               nb, 1))

    import time
    for fn, nm, ops in ((y, "Y  (mode 0)", 2.0 * nb * rpad * npad * spad), (w, "W* (mode 1)", 2.0 * nb * rpad * npad * lpad)):
        fn()
        ctx.synchronize()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ctx.synchronize()
            ts.append(time.perf_counter() - t0)
        t = min(ts)
        print(f"{name} {nm}: {t * 1e3:8.3f} ms  {ops / t / 1e12:8.1f} TOPS (int8)  [{', '.join(f'{x*1e3:.2f}' for x in ts)}]")
    print(ctx.lib.qlra_i8gemm_kernel_name().decode())


if __name__ == "__main__":
    main()
