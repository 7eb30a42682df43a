"""Diagnostic timings of the tcgen05 int8 GEMM: mode / beta / K variations at
C4-like tile counts (python tools/i8gemm_probe.py [ksweep|pairs|ncu]).  The
QLRA_I8_DEBUG settings below (1: no TMA stores, 2: no staging either) were a
temporary kernel knob used for DESIGN 3's epilogue-cost numbers; the shipped
kernel ignores it."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2404_14783_b200 import qlra as Q  # noqa: E402


def timeit(ctx, fn, reps=3):
    fn()
    ctx.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ctx.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def case(ctx, mode, M, N, K, nb, beta, label):
    dev = "cuda"
    if mode == 0:
        a = torch.randint(-128, 128, (nb, M, K), dtype=torch.int8, device=dev)
        lda, ldc = K, N
        c = torch.zeros((nb, M, N), dtype=torch.int32, device=dev)
    else:
        a = torch.randint(-128, 128, (nb, K, M), dtype=torch.int8, device=dev)
        lda, ldc = M, M
        c = torch.zeros((nb, N, M), dtype=torch.int32, device=dev)
    b = torch.randint(-128, 128, (nb, N, K), dtype=torch.int8, device=dev)
    torch.cuda.synchronize()

    def fn():
        ctx._check(ctx.lib.qlra_i8gemm_batched(ctx.h, mode, M, N, K, a.data_ptr(), lda, a.stride(0), b.data_ptr(), K,
                                               b.stride(0), c.data_ptr(), ldc, c.stride(0), nb, beta))
    t = timeit(ctx, fn)
    print(f"{label:44s} mode {mode} M {M:6d} N {N:5d} K {K:6d} nb {nb:3d} beta {beta}: {t*1e3:8.3f} ms "
          f"{2.0*nb*M*N*K/t/1e12:8.1f} TOPS", flush=True)
    del a, b, c
    torch.cuda.empty_cache()


def main():
    ctx = Q.Context(0)
    if len(sys.argv) > 1 and sys.argv[1] == "ncu":
        global timeit
        timeit = lambda ctx, fn, reps=1: (fn(), ctx.synchronize(), 1.0)[2]  # noqa: E731  one launch per case
        case(ctx, 1, 27136, 1008, 7856, 8, 1, "W*")
        case(ctx, 0, 7856, 512, 27136, 8, 0, "Y")
        case(ctx, 1, 27136, 1008, 31424, 2, 1, "W* K x4")
        return
    nb = 30
    if len(sys.argv) > 1 and sys.argv[1] == "pairs":
        import os
        for ctas in ("1", "2"):
            os.environ["QLRA_I8_CTAS"] = ctas
            for dbg in ("2", "0"):
                os.environ["QLRA_I8_DEBUG"] = dbg
                case(ctx, 1, 27136, 1008, 7936, 30, 1, f"W* ctas={ctas} dbg={dbg}")
                case(ctx, 1, 27136, 1024, 7936, 30, 1, f"W* N=1024 ctas={ctas} dbg={dbg}")
                case(ctx, 0, 7856, 512, 27136, 30, 0, f"Y ctas={ctas} dbg={dbg}")
                case(ctx, 1, 8192, 8192, 8192, 4, 0, f"square MN ctas={ctas} dbg={dbg}")
        return
    if len(sys.argv) > 1 and sys.argv[1] == "ksweep":
        import os
        for dbg in ("2", "0"):
            os.environ["QLRA_I8_DEBUG"] = dbg
            for K in (1024, 2048, 4096, 7856, 7936, 16384, 31424):
                case(ctx, 1, 27136, 1008, K, max(2, 30 * 7856 // K // 2), 1, f"dbg={dbg}")
            case(ctx, 1, 27136, 1024, 7936, 15, 1, f"dbg={dbg} N=1024")
            case(ctx, 1, 27136, 512, 7936, 30, 1, f"dbg={dbg} N=512")
            case(ctx, 1, 27136, 256, 7936, 60, 1, f"dbg={dbg} N=256")
        return
    import os
    for dbg in ("1", "2"):
        os.environ["QLRA_I8_DEBUG"] = dbg
        case(ctx, 1, 27136, 1008, 7856, nb, 1, f"W* dbg={dbg} (1: no TMA store, 2: no staging)")
        case(ctx, 0, 27136, 1008, 7856, nb, 1, f"mode 0 same tiles dbg={dbg}")
    os.environ["QLRA_I8_DEBUG"] = "0"
    case(ctx, 1, 27136, 1008, 7856, nb, 1, "W* as shipped")
    case(ctx, 1, 27136, 1008, 7856, nb, 0, "W* beta 0 (no epilogue loads)")
    case(ctx, 1, 27136, 1008, 31424, 8, 1, "W* K x4 (epilogue amortised)")
    case(ctx, 0, 27136, 1008, 7856, nb, 1, "same tiles, K-major A, row-major C")
    case(ctx, 0, 27136, 1008, 7856, nb, 0, "same, beta 0")
    case(ctx, 0, 7856, 512, 27136, nb, 0, "Y as shipped")
    case(ctx, 0, 8192, 8192, 8192, 4, 0, "square 8192")
    case(ctx, 1, 8192, 8192, 8192, 4, 0, "square 8192 MN-major A")


if __name__ == "__main__":
    main()
