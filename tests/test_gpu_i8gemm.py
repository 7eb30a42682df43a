"""The int8 engine's own tcgen05 GEMM kernel (csrc/i8gemm.cu) through the C ABI
(qlra_i8gemm_batched): exact int32 products against an fp64 matmul of the same
int8 operands (exact below 2^53), on full, ragged and clipped tiles, both
operand layouts, beta = 0 / 1; and the sketch computed through it against the
cuBLASLt route (bitwise: integer products do not depend on the kernel)."""
import os

import pytest
import torch

from paper_2404_14783_b200 import qlra as Q

pytestmark = pytest.mark.gpu


def up(x, m):
    return (x + m - 1) // m * m


def run(ctx, mode, M, N, K, batch, beta, pad_m=0, pad_k=0, seed=0):
    """Operands with leading dimensions padded past M / K (the pad holds
    garbage that must not be read into the valid products: TMA clips at the
    extents, not at the leading dimension)."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    dev = "cuda"
    if mode == 0:
        lda = up(K + pad_k, 16)
        a = torch.randint(-128, 128, (batch, M + pad_m, lda), dtype=torch.int8, device=dev, generator=g)
        a_ref = a[:, :M, :K].double()                       # M x K
    else:
        lda = up(M + pad_m, 16)
        a = torch.randint(-128, 128, (batch, K + pad_k, lda), dtype=torch.int8, device=dev, generator=g)
        a_ref = a[:, :K, :M].double().transpose(1, 2)       # M x K
    ldb = up(K + pad_k, 16)
    b = torch.randint(-128, 128, (batch, N, ldb), dtype=torch.int8, device=dev, generator=g)
    ref = a_ref @ b[:, :, :K].double().transpose(1, 2)      # M x N
    if mode == 0:
        ldc = up(N, 4) + 4
        c = torch.randint(-1000, 1000, (batch, M, ldc), dtype=torch.int32, device=dev, generator=g)
        want = c.clone()
        want[:, :, :N] = (ref + (c[:, :, :N].double() if beta else 0)).to(torch.int32)
    else:
        ldc = up(M, 4) + 4
        c = torch.randint(-1000, 1000, (batch, N, ldc), dtype=torch.int32, device=dev, generator=g)
        want = c.clone()
        want[:, :, :M] = (ref.transpose(1, 2) + (c[:, :, :M].double() if beta else 0)).to(torch.int32)
    torch.cuda.synchronize()
    rc = ctx.lib.qlra_i8gemm_batched(ctx.h, mode, M, N, K, a.data_ptr(), lda, a.stride(0), b.data_ptr(), ldb,
                                     b.stride(0), c.data_ptr(), ldc, c.stride(0), batch, beta)
    ctx._check(rc)
    ctx.synchronize()
    assert torch.equal(c, want), (mode, M, N, K, batch, beta, (c != want).sum().item())


@pytest.fixture(scope="module")
def ctx():
    c = Q.Context(0)
    yield c
    c.close()


@pytest.fixture(params=["pairs", "single"])
def ctas(request):
    """Both kernels: CTA pairs (tcgen05.mma.cta_group::2, the default above 128
    rows) and the 1-CTA form forced on the same shapes."""
    old = os.environ.get("QLRA_I8_CTAS")
    os.environ["QLRA_I8_CTAS"] = "2" if request.param == "pairs" else "1"
    yield request.param
    if old is None:
        os.environ.pop("QLRA_I8_CTAS", None)
    else:
        os.environ["QLRA_I8_CTAS"] = old


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("beta", [0, 1])
def test_i8gemm_one_tile(ctx, ctas, mode, beta):
    run(ctx, mode, 128, 256, 128, 1, beta)
    run(ctx, mode, 128, 256, 512, 2, beta, seed=1)


@pytest.mark.parametrize("mode", [0, 1])
def test_i8gemm_ragged_and_clipped(ctx, ctas, mode):
    # M, K off the tile, N a multiple of 16 below / above one tile, padded lds
    run(ctx, mode, 112, 112, 96, 3, 0, pad_m=16, pad_k=32, seed=2)
    run(ctx, mode, 1000, 208, 6000, 2, 1, pad_m=0, pad_k=16, seed=3)
    run(ctx, mode, 400, 1008, 784, 2, 1, pad_m=16, pad_k=0, seed=4)
    run(ctx, mode, 16, 16, 16, 5, 0, seed=5)
    run(ctx, mode, 300, 240, 200, 3, 1, seed=8)   # 240 columns: 120 B rows per CTA of a pair
    run(ctx, mode, 132, 48, 4000, 2, 0, seed=9)   # the pair's second CTA holds four valid rows


@pytest.mark.parametrize("mode", [0, 1])
def test_i8gemm_many_tiles_persistent(ctx, ctas, mode):
    # more tiles than SMs: the persistent loop, ring and TMEM stage phases wrap
    run(ctx, mode, 2048, 512, 1024, 15, 0, seed=6)
    run(ctx, mode, 1536, 272, 2000, 9, 1, seed=7)


def test_i8gemm_extreme_values(ctx):
    """-128 * -128 * K at the int32 accumulation bound of the engine (K < 2^17)."""
    M, N, K = 128, 16, 131056
    a = torch.full((1, M, K), -128, dtype=torch.int8, device="cuda")
    b = torch.full((1, N, K), -128, dtype=torch.int8, device="cuda")
    c = torch.zeros((1, M, N), dtype=torch.int32, device="cuda")
    ctx._check(ctx.lib.qlra_i8gemm_batched(ctx.h, 0, M, N, K, a.data_ptr(), K, M * K, b.data_ptr(), K, N * K,
                                           c.data_ptr(), N, M * N, 1, 0))
    ctx.synchronize()
    assert int(c.min()) == int(c.max()) == 128 * 128 * K


def test_i8gemm_rejects_misaligned(ctx):
    a = torch.zeros(1 << 16, dtype=torch.int8, device="cuda")
    c = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")
    rc = ctx.lib.qlra_i8gemm_batched(ctx.h, 0, 64, 24, 64, a.data_ptr(), 64, 4096, a.data_ptr(), 64, 4096,
                                     c.data_ptr(), 24, 4096, 1, 0)
    assert rc != 0


def test_sketch_through_tcgen05_equals_cublaslt(ctx):
    """The whole int8 sketch (residues -> GEMMs -> CRT) with the tcgen05 kernel
    and with cuBLASLt's: bitwise equal Y and W on a ragged shape."""
    a = torch.randn(4, 3001, 2500, dtype=torch.float64, device="cuda")
    old_e, old_g = os.environ.get("QLRA_SKETCH_ENGINE"), os.environ.get("QLRA_OZ_GEMM")
    try:
        os.environ["QLRA_SKETCH_ENGINE"] = "int8"
        os.environ["QLRA_OZ_GEMM"] = "lt"
        s_lt = Q.make_sketch(a, 90, 100, 200, 1, 2, ctx=ctx)
        os.environ["QLRA_OZ_GEMM"] = "tcgen05"
        s_tc = Q.make_sketch(a, 90, 100, 200, 1, 2, ctx=ctx)
        ctx.synchronize()
    finally:
        for k, v in (("QLRA_SKETCH_ENGINE", old_e), ("QLRA_OZ_GEMM", old_g)):
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert torch.equal(s_lt.y, s_tc.y)
    assert torch.equal(s_lt.w, s_tc.w)
    assert float(s_tc.y.abs().max()) > 0
