"""The complex representations and complex factorisations on the device
(proj/include/qlra/complex_bridge.hpp:22-30, factorizations.hpp:20-34,
:70-79) against the oracle's / numpy's forms of the same definitions."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.helpers import orthonormality_defect, planted_conditioned_matrix, random_gaussian, rel_diff, to_compact, \
    to_full

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def host(t):
    return t.detach().cpu().numpy()


def cdev(z):
    from paper_2404_14783_b200 import qlra as Q
    return Q.as_colmajor(torch.as_tensor(np.asarray(z, dtype=np.complex128), device="cuda"))


def test_representations_match_reference_definitions(ctx):  # complex_bridge.cpp:11-61
    from paper_2404_14783_b200 import qlra as Q
    a = random_gaussian(7, 5, 3)
    zc = host(Q.to_compact(dev(a), ctx))
    zf = host(Q.to_full(dev(a), ctx))
    assert np.array_equal(zc, to_compact(a)) and np.array_equal(zf, to_full(a))
    assert np.array_equal(host(Q.from_compact(cdev(zc), ctx)), a)
    # chi = [Q_c, J conj(Q_c)] (complex_bridge.hpp:17), J J conj conj = -1
    jc = host(Q.j_mul_conj(cdev(zc), ctx))
    assert np.array_equal(jc, zf[:, a.shape[2]:])
    assert np.array_equal(host(Q.j_mul_conj(cdev(jc), ctx)), -zc)
    with pytest.raises(Q.ShapeError):
        Q.from_compact(cdev(np.ones((3, 2))), ctx)
    with pytest.raises(Q.ShapeError):
        Q.j_mul_conj(cdev(np.ones((5, 2))), ctx)


@pytest.mark.parametrize("p,q", [(40, 12), (300, 100), (9, 9)])
def test_complex_qr_phase_convention(ctx, p, q):  # factorizations.cpp:33-51
    from paper_2404_14783_b200 import qlra as Q
    rng = np.random.default_rng(p + q)
    m = rng.standard_normal((p, q)) + 1j * rng.standard_normal((p, q))
    qd, rd = (host(t) for t in Q.complex_qr(cdev(m), ctx))
    assert np.linalg.norm(qd @ rd - m) < 1e-13 * np.linalg.norm(m)
    assert np.linalg.norm(qd.conj().T @ qd - np.eye(q)) < 1e-13
    assert np.allclose(np.tril(rd, -1), 0) and np.all(np.abs(np.diag(rd).imag) < 1e-14)
    assert np.all(np.diag(rd).real > 0)
    # the same (unique) Q as numpy's QR with the reference's phase rotation
    qn, rn = np.linalg.qr(m)
    ph = np.diag(rn) / np.abs(np.diag(rn))
    assert np.linalg.norm(qd - qn * ph[None, :]) < 1e-11
    with pytest.raises(Q.ShapeError):  # rows < cols (factorizations.cpp:34)
        Q.complex_qr(cdev(np.ones((2, 3))), ctx)


@pytest.mark.parametrize("p,q,kappa", [(60, 20, 1e3), (30, 90, 1e5), (400, 120, 1e2)])
def test_complex_svd(ctx, p, q, kappa):  # factorizations.cpp:53-56
    from paper_2404_14783_b200 import qlra as Q
    rng = np.random.default_rng(int(p + 7 * q))
    k = min(p, q)
    uu = np.linalg.qr(rng.standard_normal((p, k)) + 1j * rng.standard_normal((p, k)))[0]
    vv = np.linalg.qr(rng.standard_normal((q, k)) + 1j * rng.standard_normal((q, k)))[0]
    sig = kappa ** (-np.arange(k) / (k - 1))
    m = (uu * sig) @ vv.conj().T
    u, s, v = Q.complex_svd(cdev(m), ctx)
    u, s, v = host(u), np.asarray(s), host(v)
    assert np.max(np.abs(s / sig - 1)) < 1e-12 * kappa
    assert np.linalg.norm((u * s) @ v.conj().T - m) < 1e-13 * np.linalg.norm(m)
    assert np.linalg.norm(u.conj().T @ u - np.eye(k)) < 1e-12
    assert np.linalg.norm(v.conj().T @ v - np.eye(k)) < 1e-12


def test_pinv_and_spectral_norm(ctx):  # factorizations.cpp:303-327
    from paper_2404_14783_b200 import qlra as Q
    for shape in ((30, 12), (10, 25)):
        a = random_gaussian(*shape, 91)
        x = host(Q.qmat_pinv(dev(a), ctx))
        # the Penrose conditions in quaternion arithmetic
        ax, xa = O.qmat_mul(a, x), O.qmat_mul(x, a)
        assert rel_diff(O.qmat_mul(ax, a), a) < 1e-12
        assert rel_diff(O.qmat_mul(xa, x), x) < 1e-12
        assert rel_diff(ax, O.adjoint(ax)) < 1e-12 and rel_diff(xa, O.adjoint(xa)) < 1e-12
        assert abs(Q.spectral_norm(dev(a), ctx) / O.singular_values(a)[0] - 1) < 1e-13
    # rank-deficient: the tolerance zeroes the null directions
    y = planted_conditioned_matrix(40, 6, 10.0, 5)
    yy = np.concatenate([y, y[:, :, :2]], axis=2)
    x = host(Q.qmat_pinv(dev(yy), ctx))
    assert rel_diff(O.qmat_mul(O.qmat_mul(yy, x), yy), yy) < 1e-12
