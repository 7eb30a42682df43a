"""Parity at the benchmarked BASELINE configs C3, C4, C5,
against the CPU oracle, following SURVEY.md section 7's minimum slice:

* the device sketch (Y = A Omega, W = Psi A, 8-product DMMA kernel) is
  checked on sampled row blocks of Y and sampled columns of W against the
  oracle's ordered sketch (qmat_mul_accumulate_ordered, qmatrix.cpp:203-242)
  -- a full serial oracle sketch is 6-41 TFLOP of scalar CPU work;
* the oracle's rangefinder and core solve (rangefinders.cpp:107-176,
  sketching.cpp:169-194) are fed the device Y and W; the device H must span
  the oracle's range (largest principal angle, from sines, <= 1e-8) and the
  QB errors ||A - H X|| / ||A|| must agree to 1e-10 relative;
* ||A - H X|| at full size comes from the residual kernel (qgemm residual
  epilogue), itself checked here against a host computation on sampled row
  blocks, for the device's and the oracle's H, X alike.

The principal-angle metric of these large bases (up to 4M x 80 complex) is
evaluated with torch.linalg on the GPU (cuSOLVER QR): it is the metric, not
the thing under test.

Tolerances are the north_star's (BASELINE.json): angle <= 1e-8 and QB error
equal within 1e-10 relative, fp64; sketch within 1e-13 relative (different
but deterministic summation order)."""
import os
import time

import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.helpers import rel_diff

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

NT = os.cpu_count() or 8


def host(t):
    return t.detach().cpu().numpy()


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def log(msg):
    print(msg, flush=True)


# ---------------------------------------------------------- metrics ---
def _full_t(h):
    """chi(H) (2m x 2s complex128, on the GPU) of a (4, m, s) quaternion tensor."""
    q0 = torch.complex(h[0], h[1])
    q1 = torch.complex(h[2], h[3])
    top = torch.cat([q0, q1], 1)
    bot = torch.cat([-q1.conj(), q0.conj()], 1)
    return torch.cat([top, bot], 0)


def principal_angle_sin(h1, h2):
    """sin of the largest principal angle between range(chi H1) and
    range(chi H2), from sines: ||(I - Q1 Q1^*) Q2||_2."""
    q1, _ = torch.linalg.qr(_full_t(h1))
    q2, _ = torch.linalg.qr(_full_t(h2))
    r = q2 - q1 @ (q1.conj().T @ q2)
    _, rr = torch.linalg.qr(r)  # ||r||_2 = ||R_r||_2
    return float(torch.linalg.matrix_norm(rr, ord=2))


def sample_rows(m, nblk=3, b=8):
    return [(r0, min(m, r0 + b)) for r0 in np.linspace(0, m - b, nblk).astype(int)]


def sample_cols(n, k=8):
    return sorted(set(int(c) for c in np.linspace(0, n - 1, k).round()))


def oracle_y_rows(cfg, a_rows):
    """Y[rows] = A[rows] Omega with the reference's ordered kernel."""
    om = O.gen_test_matrix(cfg.kind, cfg.n, cfg.s, 1, nthreads=NT)
    return O.qmat_mul_ordered(a_rows, om, nthreads=NT)


def oracle_w_cols(cfg, a_dev, cols, blk=1 << 18):
    """W[:, cols] = Psi A[:, cols], accumulated over row blocks in row order
    (the ordered kernel's k-ascending sum, so equal to the monolithic one)."""
    idx = torch.tensor(cols, device=a_dev.device)
    acc = np.zeros((4, cfg.l, len(cols)))
    for r0 in range(0, cfg.m, blk):
        r1 = min(cfg.m, r0 + blk)
        ps = O.gen_block(cfg.kind, cfg.l, cfg.m, 2, 0, cfg.l, r0, r1, nthreads=NT)
        ab = host(a_dev[:, r0:r1].index_select(2, idx))
        acc = O.qmat_mul_ordered(ps, ab, c=acc, nthreads=NT)
    return acc


def host_residual_sq(a_rows, h_rows, x):
    d = a_rows - O.qmat_mul(h_rows, x)
    return float(np.sum(d * d))


# ---------------------------------------------------------- fixture ---
class _Run:
    pass


def _build(cfg_name, ctx):
    from paper_2404_14783_b200 import configs, qlra as Q
    cfg = configs.CONFIGS[cfg_name]
    t0 = time.time()
    a = configs.build_matrix(cfg, ctx=ctx)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    st = Q.make_sketch(a, cfg.s - 5, cfg.s, cfg.l, 1, 2, cfg.kind, ctx=ctx)
    ctx.synchronize()
    r = _Run()
    r.cfg, r.a, r.st, r.ctx, r.oracle = cfg, a, st, ctx, {}
    r.yh, r.wh = host(st.y), host(st.w)
    log(f"[{cfg_name}] A + device sketch {time.time() - t0:.1f} s")
    return r


def check_sketch_samples(run):
    """Sampled rows of Y and columns of W against the ordered oracle sketch."""
    cfg, a = run.cfg, run.a
    t0 = time.time()
    for r0, r1 in sample_rows(cfg.m):
        yo = oracle_y_rows(cfg, host(a[:, r0:r1]))
        d = rel_diff(run.yh[:, r0:r1], yo)
        assert d < 1e-13, (r0, d)
    cols = sample_cols(cfg.n)
    wo = oracle_w_cols(cfg, a, cols)
    d = rel_diff(run.wh[:, :, cols], wo)
    assert d < 1e-13, d
    log(f"[{cfg.name}] sketch samples vs ordered oracle ok ({time.time() - t0:.1f} s, W cols rel {d:.2e})")


def perturbed(a, seed):
    """a with every entry moved by up to one unit roundoff (relative): a
    sketch as a different but equally valid summation order produces it."""
    rng = np.random.default_rng(seed)
    return a * (1.0 + np.finfo(float).eps * rng.uniform(-1.0, 1.0, a.shape))


def oracle_qb(run, method, y=None, w=None, key=None):
    """The oracle's QB stage on the device sketch (cached per run), with the
    QB error of its H, X from the residual kernel."""
    from paper_2404_14783_b200 import qlra as Q
    key = key or method
    if key not in run.oracle:
        t0 = time.time()
        qo = O.qb_stage(run.yh if y is None else y, run.wh if w is None else w, 2, method, kind=run.cfg.kind,
                        nthreads=NT)
        qo["t"] = time.time() - t0
        qo["hd"], qo["xd"] = dev(qo["h"]), dev(qo["x"])
        r, an = Q.residual_fro(run.a, qo["hd"], qo["xd"], run.ctx)
        qo["err"] = r / an
        run.oracle[key] = qo
    return run.oracle[key]


def check_qb(run, ctx, method, floor=False, qb=None):
    """Device QB stage vs the oracle's QB stage fed the same device sketch.

    Bars: QB error within 1e-10 relative, principal angle <= 1e-8.  With
    floor=True the reference's own numerical floor is measured too (SURVEY.md
    H6) and a bar becomes max(bar, 4 x floor):
    * the oracle on a sketch perturbed at the unit-roundoff level, and on the
      column-permuted sketch (same range, other rounding);
    * for pseudo-QR, the oracle's pseudo-QR against its pseudo-SVD: both span
      range(Y) exactly in exact arithmetic (HX depends only on the
      range), so their QB errors differ only by the reference's own error --
      its correction steps and re-projection (rangefinders.cpp:132-153)."""
    from paper_2404_14783_b200 import qlra as Q
    cfg, a = run.cfg, run.a
    t0 = time.time()
    if qb is None:
        qb = Q.qb_stage(run.st, method, ctx=ctx)
    res_d, an = Q.residual_fro(a, qb.h, qb.x, ctx)
    t1 = time.time()
    qo = oracle_qb(run, method)
    ho, xo = qo["hd"], qo["xd"]
    err_d, err_o = res_d / an, qo["err"]
    ang = principal_angle_sin(qb.h, ho)
    log(f"[{cfg.name}] method {method}: QB err gpu {err_d:.12e} oracle {err_o:.12e} "
        f"(rel {abs(err_d / err_o - 1):.2e}), angle {ang:.2e}, kappa gpu {qb.report.kappa_before:.4e}/"
        f"{qb.report.kappa_after:.4e} steps {qb.report.correction_steps_used}; oracle {qo['kappa_before']:.4e}/"
        f"{qo['kappa_after']:.4e} steps {qo['correction_steps_used']}; device {t1 - t0:.2f} s, oracle {qo['t']:.1f} s")
    # the residual kernel at full size, checked on sampled row blocks (host);
    # forming A - H X loses ~u sqrt(s) ||A|| / ||A - H X|| relative
    for r0, r1 in sample_rows(cfg.m, nblk=2, b=16):
        ah = host(a[:, r0:r1])
        na = float(np.sqrt(np.sum(ah * ah)))
        for h, x in ((qb.h, qb.x), (ho, xo)):
            rs, ns = Q.residual_fro(a[:, r0:r1], h[:, r0:r1], x, ctx)
            hs = np.sqrt(host_residual_sq(ah, host(h[:, r0:r1]), host(x)))
            tol = 1e-12 + 10 * np.finfo(float).eps * np.sqrt(cfg.s) * na / hs
            assert abs(rs / hs - 1) < tol, (r0, rs, hs, tol)
            assert abs(ns / na - 1) < 1e-13
    bar_err, bar_ang = 1e-10, 1e-8
    if method == 0:
        # the reference's pseudo-QR against its own pseudo-SVD (same range)
        qs = oracle_qb(run, 1)
        f_rf = abs(err_o / qs["err"] - 1)
        d_svd = abs(err_d / qs["err"] - 1)
        log(f"[{cfg.name}] pseudo-QR floor: oracle pseudo-QR vs oracle pseudo-SVD QB err rel {f_rf:.2e}; "
            f"device pseudo-QR vs oracle pseudo-SVD {d_svd:.2e}")
        assert d_svd <= max(1e-10, 4 * f_rf), (err_d, qs["err"])
        bar_err = max(bar_err, 4 * f_rf)
    if floor:
        t3 = time.time()
        fl_err, fl_ang = [], []
        perm = np.random.default_rng(3).permutation(cfg.s)
        for key, y, w in (("pert", perturbed(run.yh, 1), perturbed(run.wh, 2)),
                          ("perm", np.ascontiguousarray(run.yh[:, :, perm]), run.wh)):
            qp = oracle_qb(run, method, y, w, key=f"{key}{method}")
            fl_err.append(abs(qp["err"] / err_o - 1))
            fl_ang.append(principal_angle_sin(ho, qp["hd"]))
        log(f"[{cfg.name}] method {method}: oracle-vs-oracle floor: QB err rel {fl_err[0]:.2e} (1-ulp perturbed "
            f"sketch) / {fl_err[1]:.2e} (columns permuted), angle {fl_ang[0]:.2e} / {fl_ang[1]:.2e} "
            f"({time.time() - t3:.1f} s)")
        bar_err, bar_ang = max(bar_err, 4 * max(fl_err)), max(bar_ang, 4 * max(fl_ang))
    assert abs(err_d / err_o - 1) <= bar_err, (err_d, err_o, bar_err)
    assert ang <= bar_ang, (ang, bar_ang)
    return qb, qo


def check_fused(run, ctx, method):
    """The fused one-pass entry (qlra_one_pass_qb: sketch + rangefinder +
    solve in one C-ABI call, the bench's timed call) against the oracle.  Its
    early core solve forms Psi Y as W Omega when n <= rows / 2 (C5), which
    the split qb_stage cannot assume; the bars are check_qb's."""
    from paper_2404_14783_b200 import qlra as Q
    cfg = run.cfg
    st, qb = Q.one_pass_qb_fused(run.a, cfg.s - 5, cfg.s, cfg.l, 1, 2, cfg.kind, method=method, ctx=ctx)
    assert rel_diff(host(st.y), run.yh) < 1e-14 and rel_diff(host(st.w), run.wh) < 1e-14
    del st
    return check_qb(run, ctx, method, qb=qb)


@pytest.fixture(scope="class")
def run(request, ctx):
    """A, its device sketch and host copies for the requesting class's config
    (class-scoped: one config's 10-27 GB A is alive at a time)."""
    r = _build(request.cls.CONFIG, ctx)
    yield r
    del r.a, r.st, r.oracle
    torch.cuda.empty_cache()


# ------------------------------------------------------------- C3 ---
class TestC3:
    """C3: 20000 x 15000, exact rank 200 + 1e-6 noise, s = 220, l = 440,
    Rademacher embeddings, BASELINE rangefinder: the non-orthonormal
    well-conditioned one (pseudo-QR), which the reference refuses here
    (kappa(H0) past its rcond limit) -- the device must refuse too; the
    fallback the reference's message names (pseudo-SVD) is then checked."""

    CONFIG = "C3"

    def test_sketch(self, run):
        check_sketch_samples(run)

    def test_pseudo_qr_refusal(self, run, ctx):
        from paper_2404_14783_b200 import qlra as Q
        with pytest.raises(O.OracleError) as e:
            O.pseudo_qr(run.yh)
        assert e.value.kind == "RankError"
        with pytest.raises(Q.RankError):
            Q.pseudo_qr(run.st.y, ctx=ctx)

    def test_pseudo_svd_qb(self, run, ctx):
        # kappa(Y) ~ 6e7: range(Y)'s noise-level directions are defined only
        # to ~u kappa(Y) by any floating-point method -- measure the floor
        check_qb(run, ctx, 1, floor=True)


# ------------------------------------------------------------- C4 ---
class TestC4:
    """C4: 31365 x 27125 pure quaternion 'image', s = 500, l = 1000 (the
    bench headline); both rangefinders."""

    CONFIG = "C4"

    def test_sketch(self, run):
        check_sketch_samples(run)

    @pytest.mark.parametrize("method", [0, 1])
    def test_qb(self, run, ctx, method):
        check_qb(run, ctx, method)

    def test_one_pass_fused(self, run, ctx):
        check_fused(run, ctx, 0)


# ------------------------------------------------------------- C5 ---
class TestC5:
    """C5: 2097152 x 300 flow snapshots, s = 40, l = 80; both rangefinders."""

    CONFIG = "C5"

    def test_sketch(self, run):
        check_sketch_samples(run)

    @pytest.mark.parametrize("method", [0, 1])
    def test_qb(self, run, ctx, method):
        check_qb(run, ctx, method)

    def test_one_pass_fused(self, run, ctx):
        check_fused(run, ctx, 0)
