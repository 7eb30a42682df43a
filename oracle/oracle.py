"""ctypes wrapper over liboracle_qlra.so -- TEST INFRASTRUCTURE ONLY.

The CPU oracle restates the reference qlra hot path (see qlra_oracle.cpp for
the file:line map).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs import this module; the product package
paper_2404_14783_b200 never does.

Quaternion matrices are numpy float64 arrays of shape (4, rows, cols): the
reference's four row-major planes w, x, y, z (proj/include/qlra/qmatrix.hpp:14-19).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle_qlra.so")

GAUSSIAN, RADEMACHER, SPARSE_GAUSSIAN, SPARSE_RADEMACHER = 0, 1, 2, 3
PSEUDO_QR, PSEUDO_SVD = 0, 1
DEFAULT_RANGEFINDER_SEED = 0x9E3779B9  # proj/include/qlra/rangefinders.hpp:29

STATUS_NAMES = {1: "ShapeError", 2: "ParameterError", 3: "SingularMatrixError",
                4: "RankError", 5: "PreconditionError", 6: "IoError", 99: "InternalError"}


class OracleError(RuntimeError):
    def __init__(self, code, msg, cond):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS_NAMES.get(code, str(code))
        self.estimated_condition = cond


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_last_error.argtypes = [C.POINTER(C.c_double)]
        for name in ("orc_mix64", "orc_stream_key", "orc_u64_at"):
            getattr(L, name).restype = C.c_uint64
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_stream_key.argtypes = [C.c_uint64, C.c_uint64, C.c_int]
        L.orc_u64_at.argtypes = [C.c_uint64, C.c_uint64]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _chk(rc):
    if rc != 0:
        cond = C.c_double(0.0)
        msg = lib().orc_last_error(C.byref(cond)).decode()
        raise OracleError(rc, msg, cond.value)


def _q(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    assert a.ndim == 3 and a.shape[0] == 4
    return a


I64, U64, F64, INT = C.c_int64, C.c_uint64, C.c_double, C.c_int


# ------------------------------------------------------------------- RNG ---
def mix64(z):
    return lib().orc_mix64(U64(z))


def stream_key(seed, sub=None):
    return lib().orc_stream_key(U64(seed), U64(sub or 0), INT(sub is not None))


def u64_at(key, c):
    return lib().orc_u64_at(U64(key), U64(c))


def gen_block(kind, rows, cols, seed, r0, r1, c0, c1, density=1.0, nthreads=1):
    out = np.zeros((4, r1 - r0, c1 - c0))
    _chk(lib().orc_gen_block(INT(kind), I64(rows), I64(cols), U64(seed), F64(density), I64(r0),
                             I64(r1), I64(c0), I64(c1), _p(out), INT(nthreads)))
    return out


def gen_test_matrix(kind, rows, cols, seed, density=1.0, nthreads=1):
    return gen_block(kind, rows, cols, seed, 0, rows, 0, cols, density, nthreads)


def random_gaussian(rows, cols, seed):  # proj/tests/test_helpers.hpp:11-13
    return gen_test_matrix(GAUSSIAN, rows, cols, seed)


# ------------------------------------------------------------- products ---
def qmat_mul_ordered(a, b, c=None, nthreads=1):
    a, b = _q(a), _q(b)
    m, k, n = a.shape[1], a.shape[2], b.shape[2]
    c = np.zeros((4, m, n)) if c is None else _q(c).copy()
    _chk(lib().orc_qmat_mul_acc_ordered(I64(m), I64(k), I64(n), _p(a), _p(b), _p(c), INT(nthreads)))
    return c


def qmat_mul(a, b):
    a, b = _q(a), _q(b)
    m, k, n = a.shape[1], a.shape[2], b.shape[2]
    if b.shape[1] != k:
        raise OracleError(1, "qmat_mul: inner dimensions differ", 0.0)
    c = np.zeros((4, m, n))
    _chk(lib().orc_qmat_mul(I64(m), I64(k), I64(n), _p(a), _p(b), _p(c)))
    return c


def adjoint(a):
    a = _q(a)
    r = np.transpose(a, (0, 2, 1)).copy()
    r[1:] *= -1.0
    return r


def fro_norm(a):
    return float(np.sqrt(np.sum(np.asarray(a) ** 2)))


# --------------------------------------------------------------- sketch ---
def validate_sketch_sizes(m, n, r, s, l):
    _chk(lib().orc_validate_sketch_sizes(I64(m), I64(n), I64(r), I64(s), I64(l)))


def sketch_update_rows(y, w, row0, block, omega_seed, psi_seed, kind=GAUSSIAN, density=1.0,
                       nthreads=1):
    """In-place Y[row0:row0+b] += block*Omega, W += Psi[:, rows]*block (sketching.cpp:125-139)."""
    block = _q(block)
    m, s = y.shape[1], y.shape[2]
    l, n = w.shape[1], w.shape[2]
    assert y.flags.c_contiguous and w.flags.c_contiguous
    _chk(lib().orc_sketch_update_rows(I64(m), I64(n), I64(s), I64(l), INT(kind), F64(density),
                                      U64(omega_seed), U64(psi_seed), I64(row0),
                                      I64(block.shape[1]), _p(block), _p(y), _p(w),
                                      INT(nthreads)))


def make_sketch(a, r, s, l, omega_seed, psi_seed, kind=GAUSSIAN, density=1.0, nthreads=1):
    a = _q(a)
    m, n = a.shape[1], a.shape[2]
    validate_sketch_sizes(m, n, r, s, l)
    y = np.zeros((4, m, s))
    w = np.zeros((4, l, n))
    sketch_update_rows(y, w, 0, a, omega_seed, psi_seed, kind, density, nthreads)
    return y, w


# --------------------------------------------------------- linear algebra ---
def condition_number(a):
    a = _q(a)
    k = C.c_double()
    _chk(lib().orc_condition_number(I64(a.shape[1]), I64(a.shape[2]), _p(a), C.byref(k)))
    return k.value


def singular_values(a):
    a = _q(a)
    sv = np.zeros(min(a.shape[1], a.shape[2]))
    _chk(lib().orc_singular_values(I64(a.shape[1]), I64(a.shape[2]), _p(a), _p(sv)))
    return sv


def solve_quaternion_linear(a, b):
    a, b = _q(a), _q(b)
    x = np.zeros((4, a.shape[2], b.shape[2]))
    _chk(lib().orc_solve_quaternion_linear(I64(a.shape[1]), I64(a.shape[2]), I64(b.shape[2]),
                                           _p(a), _p(b), _p(x)))
    return x


def estimate_epsilon(h, power_iters=3):
    h = _q(h)
    e = C.c_double()
    _chk(lib().orc_estimate_epsilon(I64(h.shape[1]), I64(h.shape[2]), _p(h), INT(power_iters),
                                    C.byref(e)))
    return e.value


def correction_step(h, eps):
    h = _q(h)
    out = np.zeros_like(h)
    _chk(lib().orc_correction_step(I64(h.shape[1]), I64(h.shape[2]), _p(h), F64(eps), _p(out)))
    return out


def pseudo_qr(y, max_steps=3, power_iters=3, delta=1.2):
    y = _q(y)
    h = np.zeros_like(y)
    kb, ka, st = C.c_double(), C.c_double(), C.c_int()
    _chk(lib().orc_pseudo_qr(I64(y.shape[1]), I64(y.shape[2]), _p(y), INT(max_steps),
                             INT(power_iters), F64(delta), _p(h), C.byref(kb), C.byref(ka),
                             C.byref(st)))
    return dict(h=h, kappa_before=kb.value, kappa_after=ka.value, correction_steps_used=st.value)


def pseudo_svd(y, seed=DEFAULT_RANGEFINDER_SEED):
    y = _q(y)
    h = np.zeros_like(y)
    kb, ka = C.c_double(), C.c_double()
    _chk(lib().orc_pseudo_svd(I64(y.shape[1]), I64(y.shape[2]), _p(y), U64(seed), _p(h),
                              C.byref(kb), C.byref(ka)))
    return dict(h=h, kappa_before=kb.value, kappa_after=ka.value, correction_steps_used=0)


def orthonormal_range(y, seed=DEFAULT_RANGEFINDER_SEED):
    y = _q(y)
    h = np.zeros_like(y)
    _chk(lib().orc_orthonormal_range(I64(y.shape[1]), I64(y.shape[2]), _p(y), U64(seed), _p(h)))
    return h


def qsvd(a):
    a = _q(a)
    m, n = a.shape[1], a.shape[2]
    k = min(m, n)
    u, v, sig = np.zeros((4, m, k)), np.zeros((4, n, k)), np.zeros(k)
    _chk(lib().orc_qsvd(I64(m), I64(n), _p(a), _p(u), _p(sig), _p(v)))
    return u, sig, v


def qb_stage(y, w, psi_seed, method=PSEUDO_QR, kind=GAUSSIAN, density=1.0, psi=None,
             rf_seed=DEFAULT_RANGEFINDER_SEED, max_steps=3, power_iters=3, delta=1.2,
             nthreads=1):
    """qb_stage / qb_stage_with_psi (proj/src/sketching.cpp:169-194)."""
    y, w = _q(y), _q(w)
    m, s = y.shape[1], y.shape[2]
    l, n = w.shape[1], w.shape[2]
    h = np.zeros((4, m, s))
    x = np.zeros((4, s, n))
    kb, ka, st, trf, tso = C.c_double(), C.c_double(), C.c_int(), C.c_double(), C.c_double()
    psi_p = _p(_q(psi)) if psi is not None else None
    keep = _q(psi) if psi is not None else None
    if keep is not None:
        psi_p = _p(keep)
    _chk(lib().orc_qb_stage(I64(m), I64(n), I64(s), I64(l), _p(y), _p(w), INT(kind), F64(density),
                            U64(psi_seed), psi_p, INT(method), U64(rf_seed), INT(max_steps),
                            INT(power_iters), F64(delta), _p(h), _p(x), C.byref(kb), C.byref(ka),
                            C.byref(st), C.byref(trf), C.byref(tso), INT(nthreads)))
    return dict(h=h, x=x, kappa_before=kb.value, kappa_after=ka.value,
                correction_steps_used=st.value, rangefinder_s=trf.value, solve_s=tso.value)


def residual_sq(a, h, x):
    a, h, x = _q(a), _q(h), _q(x)
    rs, as_ = C.c_double(), C.c_double()
    _chk(lib().orc_residual_sq(I64(a.shape[1]), I64(a.shape[2]), I64(h.shape[2]), _p(a), _p(h),
                               _p(x), C.byref(rs), C.byref(as_)))
    return rs.value, as_.value


def truncate_stage(h, x, r):
    h, x = _q(h), _q(x)
    m, s, n = h.shape[1], h.shape[2], x.shape[2]
    ho, vo, sig = np.zeros((4, m, r)), np.zeros((4, n, r)), np.zeros(r)
    _chk(lib().orc_truncate_stage(I64(m), I64(s), I64(n), _p(h), _p(x), I64(r), _p(ho),
                                  _p(sig), _p(vo)))
    return ho, sig, vo
