"""The int8 tensor-core sketch engine (csrc/ozaki.cu) against the CPU oracle.

The engine computes every real product of the sketch exactly in integers
(Ozaki scheme, CRT over 16 moduli) from a 52-bit fixed-point image of A,
Omega and Psi, and rounds once; the reference's ordered fp64 sketch
(qmatrix.cpp:203-242) rounds every multiply-add.  Bars: 1e-13 relative
Frobenius (the same as the DMMA engine's), observed ~1e-16.  Shapes cover
the epoch logic: several panels, host-streamed chunks with a scale change
(flush), more rows than one int32 accumulation allows (KMAX), all-zero
panels, ragged n and R, and bitwise determinism."""
import contextlib

import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.helpers import random_gaussian, rel_diff

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def host(t):
    return t.detach().cpu().numpy()


@contextlib.contextmanager
def engine(ctx, name):
    ctx.set_sketch_engine(name)
    try:
        yield
    finally:
        ctx.set_sketch_engine("auto")


@pytest.mark.parametrize("m,n,s,l,kind", [(300, 200, 10, 20, 0), (1000, 800, 60, 120, 0),
                                          (777, 1025, 33, 70, 0), (513, 2049, 100, 200, 1),
                                          (64, 16, 1, 1, 0), (2100, 300, 40, 80, 3)])
def test_int8_sketch_vs_oracle(ctx, m, n, s, l, kind):
    from paper_2404_14783_b200 import qlra as Q
    a = random_gaussian(m, n, 500 + m + n)
    with engine(ctx, "int8"):
        st = Q.make_sketch(dev(a), min(s, 3), s, l, 7, 8, kind=kind, density=0.5 if kind == 3 else 1.0, ctx=ctx)
        ks = ctx.launch_count()
    y, w = O.make_sketch(a, min(s, 3), s, l, 7, 8, kind=kind, density=0.5 if kind == 3 else 1.0, nthreads=8)
    assert rel_diff(host(st.y), y) < 1e-13
    assert rel_diff(host(st.w), w) < 1e-13
    assert ks > 0


def test_int8_matches_dmma_engine_and_is_deterministic(ctx):
    from paper_2404_14783_b200 import qlra as Q
    a = dev(random_gaussian(3000, 2500, 5))
    with engine(ctx, "int8"):
        s1 = Q.make_sketch(a, 10, 64, 128, 1, 2, ctx=ctx)
        s2 = Q.make_sketch(a, 10, 64, 128, 1, 2, ctx=ctx)
    with engine(ctx, "dmma"):
        sd = Q.make_sketch(a, 10, 64, 128, 1, 2, ctx=ctx)
    assert torch.equal(s1.y, s2.y) and torch.equal(s1.w, s2.w)
    assert rel_diff(host(s1.y), host(sd.y)) < 1e-14
    assert rel_diff(host(s1.w), host(sd.w)) < 1e-14


def test_int8_exact_on_integer_data(ctx):
    """Integer A, Omega-free check: with A and Psi small integers the fixed-
    point image is exact and the int8 engine's W is the exact product
    (rounded once), so it equals an exactly computed reference bitwise."""
    from paper_2404_14783_b200 import qlra as Q
    rng = np.random.default_rng(3)
    a = rng.integers(-1000, 1000, size=(4, 500, 700)).astype(np.float64)
    with engine(ctx, "int8"):
        st = Q.make_sketch(dev(a), 4, 8, 16, 11, 12, kind=1, ctx=ctx)  # Rademacher: +-1/2 planes
    y, w = O.make_sketch(a, 4, 8, 16, 11, 12, kind=1, nthreads=8)
    # every product is a sum of at most 4 * 700 terms of magnitude <= 1000/2: exact in fp64 too
    assert np.array_equal(host(st.y), y)
    assert np.array_equal(host(st.w), w)


def test_int8_host_stream_chunks_and_scale_flush(ctx):
    """Host-streamed chunks whose max |A| grows by 2^10 from chunk to chunk:
    each growth past the epoch's headroom flushes W's integer products and
    rescales; results still match the oracle."""
    from paper_2404_14783_b200 import qlra as Q
    a = random_gaussian(1200, 2100, 17)
    for c in range(4):
        a[:, 300 * c:300 * (c + 1)] *= 2.0 ** (10 * c)
    ah = torch.from_numpy(a).pin_memory()
    y, w = O.make_sketch(a, 4, 70, 90, 3, 4, nthreads=8)
    with engine(ctx, "int8"):
        for br in (0, 300, 160):
            st = Q.make_sketch_host(ah, 4, 70, 90, 3, 4, ctx=ctx, block_rows=br)
            assert rel_diff(host(st.y), y) < 1e-13
            assert rel_diff(host(st.w), w) < 1e-13
        whole = Q.make_sketch(dev(a), 4, 70, 90, 3, 4, ctx=ctx)
    assert rel_diff(host(whole.y), y) < 1e-13
    assert rel_diff(host(whole.w), w) < 1e-13


def test_int8_zero_rows_and_zero_block(ctx):
    from paper_2404_14783_b200 import qlra as Q
    a = random_gaussian(900, 2050, 19)
    a[:, 300:600] = 0.0
    with engine(ctx, "int8"):
        st = Q.make_sketch(dev(a), 4, 65, 66, 5, 6, ctx=ctx)
        y0, w0 = st.y.clone(), st.w.clone()
        Q.sketch_update(st, torch.zeros_like(dev(a)), ctx)
        assert torch.equal(st.y, y0) and torch.equal(st.w, w0)
    y, w = O.make_sketch(a, 4, 65, 66, 5, 6, nthreads=8)
    assert rel_diff(host(st.y), y) < 1e-13
    assert rel_diff(host(st.w), w) < 1e-13
    assert np.all(host(st.y)[:, 300:600] == 0.0)


@pytest.mark.slow
def test_int8_rows_past_one_int32_accumulation(ctx):
    """More rows than one int32 accumulation allows (2^17): W's integer
    products are recovered and restarted (epochs by row count)."""
    from paper_2404_14783_b200 import qlra as Q
    m, n = 140000, 48
    a = random_gaussian(m, n, 23)
    with engine(ctx, "int8"):
        st = Q.make_sketch(dev(a), 4, 6, 10, 9, 10, ctx=ctx)
    y, w = O.make_sketch(a, 4, 6, 10, 9, 10, nthreads=16)
    assert rel_diff(host(st.y), y) < 1e-13
    assert rel_diff(host(st.w), w) < 1e-13


def test_int8_one_pass_qb_vs_dmma(ctx):
    """The whole one-pass QB on both engines: same correction steps and kappa,
    QB error equal to 1e-10 relative."""
    from paper_2404_14783_b200 import configs, qlra as Q
    cfg = configs.CONFIGS["C1"]
    a = configs.build_matrix(cfg, ctx=ctx)
    opts = Q.OnePassOptions(r=cfg.s - 5, s=cfg.s, l=cfg.l)
    with engine(ctx, "int8"):
        ri = Q.one_pass_qb(a, opts, ctx=ctx)
    with engine(ctx, "dmma"):
        rd = Q.one_pass_qb(a, opts, ctx=ctx)
    assert ri.qb.report.correction_steps_used == rd.qb.report.correction_steps_used
    assert abs(ri.qb_residual / rd.qb_residual - 1) < 1e-10


def test_engine_selection_errors(ctx):
    from paper_2404_14783_b200 import qlra as Q
    with pytest.raises(Q.ParameterError):
        ctx.lib and ctx._check(ctx.lib.qlra_ctx_set_sketch_engine(ctx.h, 7))


@pytest.mark.parametrize("op_a,op_b", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_int8_general_product_vs_oracle(ctx, op_a, op_b):
    """Long-K quaternion products (K >= 4096, M N K >= 1.5e9) take the int8
    engine inside qmat_mul: every op pair, alpha / beta, bitwise repeatable,
    and equal to the DMMA path to ~1e-15."""
    from paper_2404_14783_b200 import qlra as Q
    m, k, n = 600, 5000, 640
    a = random_gaussian(k, m, 41) if op_a else random_gaussian(m, k, 41)
    b = random_gaussian(n, k, 42) if op_b else random_gaussian(k, n, 42)
    c0 = random_gaussian(m, n, 43)
    ref = 0.5 * O.qmat_mul(O.adjoint(a) if op_a else a, O.adjoint(b) if op_b else b) - 2.0 * c0
    outs = []
    for _ in range(2):
        out = dev(c0)
        with engine(ctx, "int8"):
            n0 = ctx.launch_count()
            Q.qmat_mul(dev(a), dev(b), op_a=op_a, op_b=op_b, alpha=0.5, beta=-2.0, out=out, ctx=ctx)
            assert ctx.launch_count() > n0
        outs.append(out)
    assert torch.equal(outs[0], outs[1])
    assert rel_diff(host(outs[0]), ref) < 1e-14
    # the residue GEMMs through cuBLASLt instead of the engine's tcgen05 kernel:
    # exact integer products, so bitwise the same quaternion result
    import os
    old = os.environ.get("QLRA_OZ_GEMM")
    os.environ["QLRA_OZ_GEMM"] = "lt"
    try:
        out_lt = dev(c0)
        with engine(ctx, "int8"):
            Q.qmat_mul(dev(a), dev(b), op_a=op_a, op_b=op_b, alpha=0.5, beta=-2.0, out=out_lt, ctx=ctx)
        ctx.synchronize()
    finally:
        if old is None:
            os.environ.pop("QLRA_OZ_GEMM", None)
        else:
            os.environ["QLRA_OZ_GEMM"] = old
    assert torch.equal(outs[0], out_lt)
    out_d = dev(c0)
    with engine(ctx, "dmma"):
        Q.qmat_mul(dev(a), dev(b), op_a=op_a, op_b=op_b, alpha=0.5, beta=-2.0, out=out_d, ctx=ctx)
    assert rel_diff(host(outs[0]), host(out_d)) < 1e-14


@pytest.mark.parametrize("m,s", [(20000, 300), (140000, 128)])
def test_int8_gram_exactly_hermitian_vs_oracle(ctx, m, s):
    """Grams H^* H of the rangefinders (rangefinders.cpp:68,102) on the int8
    engine: exact integer products give an exactly Hermitian result (real
    diagonal); K past one int32 accumulation (140000 rows) is chunked."""
    from paper_2404_14783_b200 import qlra as Q
    y = random_gaussian(m, s, 44 + m)
    with engine(ctx, "int8"):
        g = host(Q.gram(dev(y), ctx=ctx))
    ref = O.qmat_mul(O.adjoint(y), y)
    assert rel_diff(g, ref) < 1e-14
    gh = O.adjoint(g)
    assert np.array_equal(g, gh)
    assert np.all(g[1:][:, np.arange(s), np.arange(s)] == 0.0)


def test_int8_nonfinite_input_takes_the_fp64_engine(ctx):
    """NaN / inf in A have no fixed-point image: the int8 engine hands the
    block (device-resident) or the chunk (host-streamed) to the FP64 engine,
    so they propagate exactly as the reference's products propagate them."""
    from paper_2404_14783_b200 import qlra as Q
    a = random_gaussian(900, 2100, 29)
    a[1, 500, 7] = np.nan
    a[3, 10, 2000] = np.inf
    with engine(ctx, "dmma"):
        ref = Q.make_sketch(dev(a), 4, 70, 80, 3, 4, ctx=ctx)
    with engine(ctx, "int8"):
        got = Q.make_sketch(dev(a), 4, 70, 80, 3, 4, ctx=ctx)
        ah = torch.from_numpy(a).pin_memory()
        streamed = Q.make_sketch_host(ah, 4, 70, 80, 3, 4, ctx=ctx, block_rows=300)
    for st in (got, streamed):
        for x, r in ((host(st.y), host(ref.y)), (host(st.w), host(ref.w))):
            assert np.array_equal(np.isnan(x), np.isnan(r)) and np.array_equal(np.isinf(x), np.isinf(r))
            fin = np.isfinite(r)
            assert np.abs(x[fin] - r[fin]).max() <= 1e-13 * np.abs(r[fin]).max()


@pytest.mark.parametrize("cfg_name,method", [("C2", 0), ("C2", 1), ("C1", 0)])
def test_fused_one_pass_equals_split_calls(ctx, cfg_name, method):
    """qlra_one_pass_qb (sketch + rangefinder + core solve in one call)
    returns exactly what make_sketch + qb_stage return."""
    from paper_2404_14783_b200 import configs, qlra as Q
    cfg = configs.CONFIGS[cfg_name]
    a = configs.build_matrix(cfg, ctx=ctx)
    st = Q.make_sketch(a, cfg.s - 5, cfg.s, cfg.l, 1, 2, kind=cfg.kind, ctx=ctx)
    qb = Q.qb_stage(st, method, ctx=ctx)
    for _ in range(2):
        st2, qb2 = Q.one_pass_qb_fused(a, cfg.s - 5, cfg.s, cfg.l, 1, 2, kind=cfg.kind, method=method, ctx=ctx)
        assert torch.equal(st2.y, st.y) and torch.equal(st2.w, st.w)
        assert torch.equal(qb2.h, qb.h) and torch.equal(qb2.x, qb.x)
        assert qb2.report.correction_steps_used == qb.report.correction_steps_used
