"""ctypes binding of libqlra_cuda.so (include/qlra_cuda.h).

Fails loudly: there is no CPU fallback anywhere in the product.  If the
library is missing it is built in-tree (nvcc), and if that fails the import
error propagates.
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

_HERE = os.path.dirname(os.path.abspath(__file__))

I64, U64, F64, INT, VP = C.c_int64, C.c_uint64, C.c_double, C.c_int, C.c_void_p


class Spec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("rows", C.c_int64), ("cols", C.c_int64),
                ("seed", C.c_uint64), ("density", C.c_double)]


class QMat(C.Structure):
    _fields_ = [("p", C.c_void_p * 4), ("rows", C.c_int64), ("cols", C.c_int64), ("ld", C.c_int64)]


class CMat(C.Structure):
    """qlra_cmat_t: column-major complex matrix, interleaved (re, im)."""
    _fields_ = [("data", C.c_void_p), ("rows", C.c_int64), ("cols", C.c_int64), ("ld", C.c_int64)]


class PseudoQrConfig(C.Structure):
    _fields_ = [("max_correction_steps", C.c_int32), ("power_iters_for_epsilon", C.c_int32),
                ("delta_budget", C.c_double)]


class Report(C.Structure):
    _fields_ = [("kappa_before", C.c_double), ("kappa_after", C.c_double),
                ("correction_steps_used", C.c_int32), ("method", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("QLRA_LIB_PATH") or _build.LIB  # override: A/B builds in tools/
    if not os.path.exists(path):
        _build.build()
    L = C.CDLL(path)
    P, PS, PQ, PC = C.POINTER, C.POINTER(Spec), C.POINTER(QMat), C.POINTER(CMat)
    sig = {
        "qlra_ctx_create": ([P(VP), INT, INT, INT, VP], INT),
        "qlra_ctx_destroy": ([VP], INT),
        "qlra_group_create": ([P(VP), INT], INT),
        "qlra_group_destroy": ([VP], INT),
        "qlra_ctx_create_local": ([P(VP), INT, VP, INT], INT),
        "qlra_ctx_set_stream": ([VP, VP], INT),
        "qlra_ctx_synchronize": ([VP], INT),
        "qlra_nccl_unique_id": ([VP], INT),
        "qlra_last_error": ([VP, P(F64)], C.c_char_p),
        "qlra_ctx_launch_count": ([VP], I64),
        "qlra_ctx_kernel_timing": ([VP, INT], INT),
        "qlra_ctx_kernel_stats": ([VP, P(F64), P(I64), P(F64), P(F64)], INT),
        "qlra_ctx_kernel_engines": ([VP, P(INT), P(F64)], INT),
        "qlra_ctx_set_sketch_engine": ([VP, INT], INT),
        "qlra_one_pass_qb": ([VP, PQ, I64, PS, PS, INT, U64, P(PseudoQrConfig), PQ, PQ, PQ, PQ, P(Report)], INT),
        "qlra_measure_int8_peak": ([VP, F64, P(F64)], INT),
        "qlra_i8gemm_batched": ([VP, INT, I64, I64, I64, VP, I64, I64, VP, I64, I64, VP, I64, I64, INT, INT], INT),
        "qlra_i8gemm_kernel_name": ([], C.c_char_p),
        "qlra_int8_engine_name": ([], C.c_char_p),
        "qlra_gen_test_matrix_block": ([VP, PS, I64, I64, PQ], INT),
        "qlra_sketch_update_rows": ([VP, PS, PS, I64, PQ, PQ, PQ], INT),
        "qlra_sketch_update_rows_host": ([VP, PS, PS, I64, PQ, PQ, PQ, I64], INT),
        "qlra_sketch_allreduce": ([VP, PQ], INT),
        "qlra_qmat_mul": ([VP, INT, INT, F64, PQ, PQ, F64, PQ], INT),
        "qlra_gram": ([VP, PQ, PQ], INT),
        "qlra_condition_number": ([VP, PQ, P(F64)], INT),
        "qlra_singular_values": ([VP, PQ, P(F64)], INT),
        "qlra_solve_quaternion_linear": ([VP, PQ, PQ, PQ], INT),
        "qlra_estimate_epsilon": ([VP, PQ, INT, P(F64)], INT),
        "qlra_correction_step": ([VP, PQ, F64, PQ], INT),
        "qlra_pseudo_qr": ([VP, PQ, P(PseudoQrConfig), PQ, P(Report)], INT),
        "qlra_pseudo_svd": ([VP, PQ, U64, PQ, P(Report)], INT),
        "qlra_orthonormal_range": ([VP, PQ, U64, PQ], INT),
        "qlra_qb_stage_with_psi": ([VP, PQ, PQ, PQ, INT, U64, P(PseudoQrConfig), PQ, PQ, P(Report)], INT),
        "qlra_ctx_stream": ([VP], VP),
        "qlra_to_compact": ([VP, PQ, PC], INT),
        "qlra_to_full": ([VP, PQ, PC], INT),
        "qlra_from_compact": ([VP, PC, PQ], INT),
        "qlra_j_mul_conj": ([VP, PC, PC], INT),
        "qlra_complex_qr": ([VP, PC, PC, PC], INT),
        "qlra_complex_svd": ([VP, PC, PC, P(F64), PC], INT),
        "qlra_qmat_pinv": ([VP, PQ, PQ], INT),
        "qlra_spectral_norm": ([VP, PQ, P(F64)], INT),
        "qlra_qb_solve": ([VP, PS, I64, PQ, PQ, PQ], INT),
        "qlra_qb_stage": ([VP, PS, I64, PQ, PQ, INT, U64, P(PseudoQrConfig), PQ, PQ, P(Report)], INT),
        "qlra_one_pass_qb_host": ([VP, PQ, I64, PS, PS, INT, U64, P(PseudoQrConfig), I64, PQ, PQ, P(Report)],
                                  INT),
        "qlra_residual_fro": ([VP, PQ, PQ, PQ, P(F64), P(F64)], INT),
        "qlra_qsvd": ([VP, PQ, PQ, P(F64), PQ], INT),
        "qlra_truncate_stage": ([VP, PQ, PQ, I64, PQ, P(F64), PQ], INT),
        "qlra_approx_residual_fro": ([VP, PQ, PQ, P(F64), PQ, P(F64), P(F64)], INT),
        "qlra_write_qmat": ([VP, C.c_char_p, PQ], INT),
        "qlra_qmat_file_shape": ([C.c_char_p, P(I64), P(I64)], INT),
        "qlra_read_qmat": ([VP, C.c_char_p, PQ], INT),
        "qlra_write_sketch": ([VP, C.c_char_p, PS, PS, I64, I64, I64, PQ, PQ], INT),
        "qlra_sketch_file_header": ([C.c_char_p, PS, PS, P(I64)], INT),
        "qlra_read_sketch": ([VP, C.c_char_p, PQ, PQ], INT),
        "qlra_sketch_file_dims": ([C.c_char_p, P(I64)], INT),
        "qlra_sketch_from_qmat_file": ([VP, C.c_char_p, PS, PS, PQ, PQ, I64], INT),
        "qlra_measure_fp64_peak": ([VP, INT, F64, P(F64)], INT),
        "qlra_sketch_kernel_name": ([], C.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def exported_symbols():
    """Names declared in include/qlra_cuda.h (parsed) -- for the export test."""
    import re
    hdr = os.path.join(os.path.dirname(_HERE), "include", "qlra_cuda.h")
    src = open(hdr).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z0-9_]+\s*\*?\s*(qlra_[a-z0-9_]+)\s*\(", src, re.M)))
