"""CPU checks of the 8-product quaternion algebra the sketch engine uses
(paper_2404_14783_b200/csrc/qtile8.cuh).

The combination tables are read out of the kernel header itself, so these
tests pin the constants the device code runs with: the 8 products of plane
combinations, halves folded into products 5..8, must reproduce the Hamilton
product (proj/include/qlra/quaternion.hpp:33-38) for scalars and, since no
product commutes its factors, for quaternion matrices too.  The matrix case
is checked against the oracle's 16-plane product (oracle/oracle.py)."""
import os
import re

import numpy as np

from oracle import oracle as O

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2404_14783_b200", "csrc", "qtile8.cuh")


def _table(fn, var):
    """The 8 '+/- x[i] +/- x[j]' expressions of lcomb / rcomb as coefficient rows."""
    src = open(HDR).read()
    body = src[src.index(f"double {fn}(int i, const double (&{var})[4])"):]
    body = body[:body.index("\n}\n")]
    exprs = re.findall(r"return ([^;]+);", body)
    assert len(exprs) == 8, exprs
    rows = []
    for e in exprs:
        row = np.zeros(4)
        for sign, idx in re.findall(r"([+-]?)\s*" + var + r"\[(\d)\]", e.replace(" ", "")):
            row[int(idx)] += -1.0 if sign == "-" else 1.0
        rows.append(row)
    return np.array(rows)


def _combine(m):
    """qtile8.cuh combine(): the 4 planes from the 8 products, in its order."""
    src = open(HDR).read()
    body = src[src.index("void combine(const double (&m)[8], double (&c)[4])"):]
    body = body[:body.index("\n}\n")]
    env = {"m": m}
    for line in body.splitlines()[1:]:
        line = line.strip().rstrip(";")
        if not line:
            continue
        line = line.replace("const double ", "").replace(", ", "; ")
        for stmt in line.split("; "):
            lhs, rhs = stmt.split(" = ")
            val = eval(rhs, {}, env)  # noqa: S307 -- expressions from our own header
            if lhs.startswith("c["):
                env.setdefault("c", [0.0] * 4)[int(lhs[2])] = val
            else:
                env[lhs] = val
    return env["c"]


def _hamilton(a, b):
    return np.array([a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3],
                     a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2],
                     a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1],
                     a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0]])


def _products(L, R, a, b):
    half = np.array([1, 1, 1, 1, 0.5, 0.5, 0.5, 0.5])
    return [(L[i] @ a) * (R[i] @ b) * half[i] for i in range(8)]


def test_tables_have_pairwise_sums():
    for L in (_table("lcomb", "a"), _table("rcomb", "b")):
        assert np.all(np.sum(np.abs(L), axis=1) == 2)  # one DADD per combination


def test_scalar_identity():
    L, R = _table("lcomb", "a"), _table("rcomb", "b")
    rng = np.random.default_rng(7)
    for _ in range(200):
        a, b = rng.standard_normal(4), rng.standard_normal(4)
        c = _combine(_products(L, R, a, b))
        assert np.allclose(c, _hamilton(a, b), rtol=0, atol=1e-14 * (1 + np.abs(a).sum() * np.abs(b).sum()))


def test_bilinear_tensor_exact():
    """Coefficient-exact: every (a_p, b_q) monomial gets the Hamilton sign."""
    L, R = _table("lcomb", "a"), _table("rcomb", "b")
    for p in range(4):
        for q in range(4):
            a, b = np.eye(4)[p], np.eye(4)[q]
            assert np.array_equal(np.array(_combine(_products(L, R, a, b))), _hamilton(a, b))


def test_matrix_identity_vs_oracle():
    """8 real GEMMs of plane combinations == the quaternion GEMM (order kept)."""
    L, R = _table("lcomb", "a"), _table("rcomb", "b")
    a, b = O.random_gaussian(23, 17, 3), O.random_gaussian(17, 11, 4)  # (4, rows, cols) planes
    half = [1, 1, 1, 1, 0.5, 0.5, 0.5, 0.5]
    m = [np.einsum("p,pij->ij", L[i], a) @ np.einsum("p,pij->ij", R[i], b) * half[i] for i in range(8)]
    c = np.array(_combine(m))
    ref = O.qmat_mul(a, b)
    assert np.max(np.abs(c - ref)) < 1e-12 * np.max(np.abs(ref))
