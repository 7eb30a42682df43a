"""Test helpers mirroring proj/tests/test_helpers.hpp and the planted-matrix
generators of proj/src/synthetic.cpp:78-101 (built on the CPU oracle)."""
import numpy as np

from oracle import oracle as O


def random_gaussian(rows, cols, seed):
    return O.random_gaussian(rows, cols, seed)


def rel_diff(a, b):
    nb = np.sqrt(np.sum(np.asarray(b) ** 2))
    d = np.sqrt(np.sum((np.asarray(a) - np.asarray(b)) ** 2))
    return d / nb if nb > 0 else d


def scalar(w, x=0.0, y=0.0, z=0.0):
    m = np.zeros((4, 1, 1))
    m[:, 0, 0] = [w, x, y, z]
    return m


def diag_real(d):
    n = len(d)
    m = np.zeros((4, n, n))
    m[0][np.arange(n), np.arange(n)] = d
    return m


def identity(n):
    return diag_real([1.0] * n)


def orthonormality_defect(m):
    return O.fro_norm(O.qmat_mul(O.adjoint(m), m) - identity(m.shape[2]))


def planted_matrix_with_sigma(m, sigma, seed):
    s = len(sigma)
    gu = O.gen_test_matrix(O.GAUSSIAN, m, s, O.stream_key(seed, 1))
    gv = O.gen_test_matrix(O.GAUSSIAN, s, s, O.stream_key(seed, 2))
    us = O.orthonormal_range(gu, O.stream_key(seed, 3))
    v = O.orthonormal_range(gv, O.stream_key(seed, 4))
    us = us * np.asarray(sigma, dtype=np.float64)[None, None, :]
    return O.qmat_mul(us, O.adjoint(v))


def planted_conditioned_matrix(m, s, kappa, seed):
    sigma = [kappa ** (-i / (s - 1)) if s > 1 else 1.0 for i in range(s)]
    return planted_matrix_with_sigma(m, sigma, seed)


# ---- complex forms (numpy) for subspace metrics --------------------------
def to_compact(a):
    a = np.asarray(a)
    return np.concatenate([a[0] + 1j * a[1], -a[2] + 1j * a[3]], axis=0)


def to_full(a):
    a = np.asarray(a)
    q0 = a[0] + 1j * a[1]
    q1 = a[2] + 1j * a[3]
    return np.block([[q0, q1], [-np.conj(q1), np.conj(q0)]])


def range_basis(h):
    """Orthonormal complex basis of range(chi_H) (2m x 2s)."""
    u, s, _ = np.linalg.svd(to_full(h), full_matrices=False)
    tol = max(u.shape) * np.finfo(float).eps * (s[0] if s.size else 0.0)
    return u[:, s > tol]


def largest_principal_angle(h1, h2):
    """sin of the largest principal angle between range(chi_H1) and
    range(chi_H2), computed from sines: sigma_max((I - Q1 Q1^*) Q2)."""
    q1, q2 = range_basis(h1), range_basis(h2)
    if q1.shape[1] != q2.shape[1]:
        return 1.0
    r = q2 - q1 @ (q1.conj().T @ q2)
    return float(np.linalg.norm(r, 2))
