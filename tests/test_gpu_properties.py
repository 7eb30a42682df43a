"""Property tests of the reference suite on the device path (the remaining
hot-path cases of proj/tests/test_sketching.cpp and test_rangefinders.cpp,
SURVEY.md section 4), complementing the oracle-parity tests in
test_gpu_parity.py.  Quaternion identities are checked in the complex
adjoint chi (a ring homomorphism that also maps pseudo-inverses, with
||chi(A)||_F^2 = 2 ||A||_F^2)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.helpers import (largest_principal_angle, planted_conditioned_matrix, planted_matrix_with_sigma,
                           random_gaussian, rel_diff, to_full)

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def host(t):
    return t.detach().cpu().numpy()


def _q(a):  # quaternion (4, m, n) -> complex adjoint (2m, 2n)
    return to_full(np.asarray(a))


def test_rank1_sketch_inside_planted_column_space(ctx):  # test_sketching.cpp:76-83
    from paper_2404_14783_b200 import qlra as Q
    u = O.orthonormal_range(random_gaussian(12, 1, 34))
    v = random_gaussian(10, 1, 35)
    a = O.qmat_mul(u, O.adjoint(v))
    st = Q.make_sketch(dev(a), 1, 2, 4, 3, 4, ctx=ctx)
    y = host(st.y)
    resid = y - O.qmat_mul(u, O.qmat_mul(O.adjoint(u), y))
    assert np.linalg.norm(resid) < 1e-12 * np.linalg.norm(y)


def test_sketch_energy_fourfold_rule(ctx):  # test_sketching.cpp:85-98
    """E ||A Omega||_F^2 = 4 ||A||_F^2 for one Gaussian quaternion column."""
    from paper_2404_14783_b200 import qlra as Q
    a = random_gaussian(10, 10, 36)
    ad = dev(a)
    acc = 0.0
    for t in range(200):
        st = Q.make_sketch(ad, 1, 1, 2, 1000 + t, 5000, ctx=ctx)
        acc += float((st.y ** 2).sum())
    acc /= 200
    theory = 4.0 * float(np.sum(a ** 2))
    assert abs(acc - theory) < 0.15 * theory


def test_qb_error_dominates_projection_error(ctx):  # test_sketching.cpp:197-208
    from paper_2404_14783_b200 import qlra as Q
    a = planted_matrix_with_sigma(30, [1, 0.9, 0.8, 0.2, 0.1, 0.05, 0.02, 0.01, 0.005, 0.002], 47)
    wide = O.qmat_mul(a, O.adjoint(O.orthonormal_range(random_gaussian(25, 10, 48))))
    st = Q.make_sketch(dev(wide), 3, 5, 10, 49, 50, ctx=ctx)
    qb = Q.qb_stage(st, Q.PSEUDO_QR, ctx=ctx)
    qb_err = np.linalg.norm(wide - O.qmat_mul(host(qb.h), host(qb.x)))
    uy = O.orthonormal_range(host(st.y))
    proj = wide - O.qmat_mul(uy, O.qmat_mul(O.adjoint(uy), wide))
    assert qb_err >= np.linalg.norm(proj) - 1e-10


def test_qb_error_splits_into_projection_and_crosstalk(ctx):  # test_sketching.cpp:225-254
    """||A - HX||^2 = ||(I - QQ*)A||^2 + ||(Psi Q)^+ Psi (I - QQ*) A||^2 with Q
    an orthonormal basis of range(Y) (the one-pass error identity)."""
    from paper_2404_14783_b200 import qlra as Q
    m, n, r, s, l = 24, 20, 3, 5, 10
    a = O.qmat_mul(planted_matrix_with_sigma(m, [1, 0.8, 0.6, 0.1, 0.05, 0.02, 0.01, 0.005, 0.002, 0.001], 53),
                   O.adjoint(O.orthonormal_range(random_gaussian(n, 10, 54))))
    st = Q.make_sketch(dev(a), r, s, l, 55, 56, ctx=ctx)
    psi = host(Q.gen_test_matrix(st.psi_spec, ctx))
    qb = Q.qb_stage(st, Q.PSEUDO_QR, ctx=ctx)
    lhs = np.linalg.norm(a - O.qmat_mul(host(qb.h), host(qb.x))) ** 2
    q = host(Q.pseudo_svd(st.y, ctx=ctx).h)
    A, Qc, P = _q(a), _q(q), _q(psi)
    comp = A - Qc @ (Qc.conj().T @ A)            # (I - QQ*) A
    cross = np.linalg.pinv(P @ Qc) @ (P @ comp)  # (Psi Q)^+ Psi (I - QQ*) A
    rhs = 0.5 * (np.linalg.norm(comp) ** 2 + np.linalg.norm(cross) ** 2)
    assert abs(lhs - rhs) <= 1e-8 * rhs


def test_one_pass_exact_rank_r_recovered(ctx):  # test_sketching.cpp:266-277
    from paper_2404_14783_b200 import qlra as Q
    left = O.orthonormal_range(random_gaussian(30, 4, 57))
    right = O.orthonormal_range(random_gaussian(25, 4, 58))
    ls = left * np.array([2.0 - 0.3 * j for j in range(4)])[None, None, :]
    a = O.qmat_mul(ls, O.adjoint(right))
    res = Q.one_pass_approx(dev(a), Q.OnePassOptions(r=4, rangefinder=Q.PSEUDO_SVD), ctx=ctx)
    assert res.diagnostics["relative_error"] <= 1e-7
    o = Q.resolve_defaults(Q.OnePassOptions(r=4))  # test_sketching.cpp:279-290
    assert (o.s, o.l) == (9, 18)


def test_pseudo_svd_single_column(ctx):  # test_rangefinders.cpp:97-103
    from paper_2404_14783_b200 import qlra as Q
    y = np.zeros((4, 2, 1))
    y[0, 0, 0] = 3.0
    assert rel_diff(host(Q.pseudo_svd(dev(y), ctx=ctx).h), host(Q.pseudo_qr(dev(y), ctx=ctx).h)) < 1e-14
    with pytest.raises(Q.ParameterError):
        Q.pseudo_svd(dev(random_gaussian(3, 3, 58)), ctx=ctx)


def test_correction_contracts_kappa_below_its_square_root(ctx):  # test_rangefinders.cpp:170-188
    from paper_2404_14783_b200 import qlra as Q
    for trial in range(5):
        y = planted_conditioned_matrix(120, 12, 10.0 ** (3 + trial), 70 + trial)
        h = Q.pseudo_qr(dev(y), Q.PseudoQrConfig(max_correction_steps=0), ctx).h
        kappa = Q.condition_number(h, ctx)
        for _ in range(3):
            if kappa <= 10.0:
                break
            h = Q.correction_step(h, Q.estimate_epsilon(h, 3, ctx), ctx)
            nxt = Q.condition_number(h, ctx)
            if kappa > 4.0:
                assert nxt < np.sqrt(kappa) + 1e-9
            kappa = nxt
        assert kappa < 10.0


def test_range_preserved_across_conditioning(ctx):  # test_rangefinders.cpp:190-198
    from paper_2404_14783_b200 import qlra as Q
    for kappa in (1e2, 1e6):
        y = planted_conditioned_matrix(150, 15, kappa, 80)
        assert largest_principal_angle(host(Q.pseudo_qr(dev(y), ctx=ctx).h), y) <= 1e-7
        assert largest_principal_angle(host(Q.pseudo_svd(dev(y), ctx=ctx).h), y) <= 1e-7
    # kappa = 1e12: kappa^2 is past double precision, so this takes the
    # graded route.  The reference's 1e-7 here compares two bases taken from
    # the SAME qsvd of `hard` (range_distance, analysis.cpp:81-88), so it is
    # met only by sharing that computation: the range of a stored kappa=1e12
    # matrix is defined to ~u*kappa (LAPACK's own SVD of a row-permuted copy
    # moves it by 9e-5, as do Householder QR and CGS2).  What is checked is
    # what any backward-stable method delivers: Y fully captured, H
    # orthonormal, the angle at the u*kappa level, kappa(Y) recovered.
    hard = planted_conditioned_matrix(150, 15, 1e12, 81)
    rep = Q.pseudo_svd(dev(hard), ctx=ctx)
    h = host(rep.h)
    H, Y = _q(h), _q(hard)
    assert np.linalg.norm(H.conj().T @ H - np.eye(H.shape[1])) <= 1e-13
    assert np.linalg.norm(Y - H @ (H.conj().T @ Y)) <= 1e-14 * np.linalg.norm(Y)
    assert largest_principal_angle(h, hard) <= 1e-3
    assert abs(rep.kappa_before / 1e12 - 1) < 1e-2


def test_reports_carry_condition_bookkeeping(ctx):  # test_rangefinders.cpp:200-210
    from paper_2404_14783_b200 import qlra as Q
    y = planted_conditioned_matrix(100, 10, 1e5, 82)
    rep = Q.pseudo_qr(dev(y), ctx=ctx)
    assert rep.kappa_before >= rep.kappa_after >= 1.0
    assert rep.method == Q.PSEUDO_QR
    rep2 = Q.pseudo_svd(dev(y), ctx=ctx)
    assert abs(rep2.kappa_before / 1e5 - 1) < 1e-6
    assert rep2.method == Q.PSEUDO_SVD
