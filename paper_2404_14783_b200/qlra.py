"""Python mirror of the reference `qlra` hot-path API, running on the B200
through the C-ABI (include/qlra_cuda.h).

Names, argument meanings and error behaviour follow the reference headers
proj/include/qlra/{sketching,rangefinders,complex_bridge,factorizations,
qmatrix,errors}.hpp so the parity tests read like the reference's own tests.
A QMatrix here is a CUDA float64 tensor of shape (4, rows, cols): the four
row-major planes w, x, y, z of proj/include/qlra/qmatrix.hpp:14-19.  torch
only provides device memory and streams; every FLOP runs in the library's
sm_100a kernels.

Multi-GPU (one process per GPU): create the Context with
rank/nranks and an NCCL id; data matrices (A, Y, H) are then the rank's row
shard and `row0` is the shard's first global row.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import torch

from . import _lib as L

GAUSSIAN, RADEMACHER, SPARSE_GAUSSIAN, SPARSE_RADEMACHER = 0, 1, 2, 3
KIND_NAMES = {"gaussian": 0, "rademacher": 1, "sparse-gaussian": 2, "sparse-rademacher": 3}
PSEUDO_QR, PSEUDO_SVD = 0, 1
DEFAULT_RANGEFINDER_SEED = 0x9E3779B9  # rangefinders.hpp:29


# ------------------------------------------------------------- errors ---
# proj/include/qlra/errors.hpp:9-43
class Error(RuntimeError):
    pass


class ShapeError(Error):
    pass


class ParameterError(Error):
    pass


class SingularMatrixError(Error):
    """Message format of errors.hpp:23-30: msg + " (estimated condition " +
    std::to_string(cond) + ")" (std::to_string(double) is "%f")."""

    def __init__(self, msg, estimated_condition):
        super().__init__(f"{msg} (estimated condition {estimated_condition:f})")
        self.estimated_condition = estimated_condition


class RankError(Error):
    pass


class PreconditionError(Error):
    pass


class IoError(Error):
    pass


class DeviceError(Error):
    pass


_ERR = {1: ShapeError, 2: ParameterError, 4: RankError, 5: PreconditionError, 6: IoError}


# ------------------------------------------------------------ context ---
class LocalGroup:
    """In-process communicator (qlra_group_t): `nranks` Contexts, one per host
    thread, whose all-reduces the library performs itself in rank order --
    the multi-rank path on ONE GPU (NCCL refuses two ranks per device) or
    across the devices of one process."""

    def __init__(self, nranks: int):
        self.lib = L.lib()
        self.nranks = nranks
        h = C.c_void_p()
        if self.lib.qlra_group_create(C.byref(h), nranks) != 0:
            raise ParameterError("qlra_group_create: nranks must lie in [1, 16]")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            if self.lib.qlra_group_destroy(self.h) != 0:
                raise PreconditionError("qlra_group_destroy: contexts still attached")
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """One per process/device (or per thread of a LocalGroup): stream,
    communicator (NCCL or the in-process group), error state."""

    def __init__(self, device: int = 0, rank: int = 0, nranks: int = 1, nccl_id: bytes | None = None,
                 use_torch_stream: bool = True, local_group: LocalGroup | None = None):
        self.lib = L.lib()
        self.device = device
        self.rank, self.nranks = rank, nranks
        h = C.c_void_p()
        if local_group is not None:
            self.nranks = local_group.nranks
            rc = self.lib.qlra_ctx_create_local(C.byref(h), device, local_group.h, rank)
        else:
            buf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
            rc = self.lib.qlra_ctx_create(C.byref(h), device, rank, nranks, buf)
        if rc != 0:
            raise DeviceError(f"qlra_ctx_create failed ({rc})")
        self.group = local_group
        self.h = h
        if use_torch_stream:
            self.set_stream(torch.cuda.current_stream(device))

    def set_stream(self, stream: torch.cuda.Stream):
        self._check(self.lib.qlra_ctx_set_stream(self.h, C.c_void_p(stream.cuda_stream)))
        self.stream = stream

    def synchronize(self):
        self._check(self.lib.qlra_ctx_synchronize(self.h))

    def launch_count(self) -> int:
        return int(self.lib.qlra_ctx_launch_count(self.h))

    def kernel_timing(self, enable: bool):
        """Start/stop CUDA-event timing of every fused sketch launch."""
        self._check(self.lib.qlra_ctx_kernel_timing(self.h, 1 if enable else 0))

    def kernel_stats(self) -> dict:
        ms, n, fl, by = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
        self._check(self.lib.qlra_ctx_kernel_stats(self.h, C.byref(ms), C.byref(n), C.byref(fl), C.byref(by)))
        eng, ops = C.c_int(), C.c_double()
        self._check(self.lib.qlra_ctx_kernel_engines(self.h, C.byref(eng), C.byref(ops)))
        return dict(ms=ms.value, launches=n.value, flops=fl.value, a_bytes=by.value, engines=eng.value,
                    int8_ops=ops.value)

    SKETCH_ENGINES = {"auto": 0, "dmma": 1, "int8": 2}

    def set_sketch_engine(self, engine: str):
        """Sketch engine: "auto" (int8 tensor cores where faster), "dmma"
        (FP64 tensor cores) or "int8" (exact integer products, Ozaki/CRT)."""
        self._check(self.lib.qlra_ctx_set_sketch_engine(self.h, self.SKETCH_ENGINES[engine]))

    def _check(self, rc: int):
        if rc == 0:
            return
        cond = C.c_double(0.0)
        msg = self.lib.qlra_last_error(self.h, C.byref(cond)).decode()
        if rc == 3:
            raise SingularMatrixError(msg, cond.value)
        raise _ERR.get(rc, DeviceError)(f"[{rc}] {msg}")

    def close(self):
        if getattr(self, "h", None):
            self.lib.qlra_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        if L.lib().qlra_nccl_unique_id(buf) != 0:
            raise DeviceError("ncclGetUniqueId failed")
        return buf.raw


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(torch.cuda.current_device())
    return _default_ctx


def set_default_context(ctx: Context):
    global _default_ctx
    _default_ctx = ctx


def _ctx(ctx):
    return ctx if ctx is not None else default_context()


# ---------------------------------------------------------- QMatrix glue ---
def qzeros(rows, cols, device=None):
    return torch.zeros((4, rows, cols), dtype=torch.float64, device=device or "cuda")


def _qm(t: torch.Tensor, host: bool = False) -> L.QMat:
    if t.dtype != torch.float64 or t.dim() != 3 or t.shape[0] != 4 or t.is_cuda == host:
        where = "CPU (pinned)" if host else "CUDA"
        raise ShapeError(f"QMatrix must be a {where} float64 tensor of shape (4, rows, cols)")
    if t.shape[2] > 1 and t.stride(2) != 1:
        raise ShapeError("QMatrix planes must be row-major (unit column stride)")
    q = L.QMat()
    base = t.data_ptr()
    for p in range(4):
        q.p[p] = base + p * t.stride(0) * 8
    q.rows, q.cols = t.shape[1], t.shape[2]
    q.ld = max(t.stride(1), t.shape[2]) if t.shape[1] > 1 else t.shape[2]
    return q


def identity(n, device=None):
    e = qzeros(n, n, device)
    e[0].fill_diagonal_(1.0)
    return e


def adjoint(a: torch.Tensor) -> torch.Tensor:
    r = a.transpose(1, 2).contiguous()
    r[1:] *= -1.0
    return r


def fro_norm(a: torch.Tensor) -> float:
    return float(torch.sqrt(torch.sum(a * a)))


# ------------------------------------------------------- test matrices ---
@dataclass
class TestMatrixSpec:
    """== TestMatrixSpec (sketching.hpp:22-28)."""
    kind: int = GAUSSIAN
    rows: int = 0
    cols: int = 0
    seed: int = 0
    density: float = 1.0

    def c(self) -> L.Spec:
        return L.Spec(self.kind, self.rows, self.cols, self.seed, self.density)


def gen_block(spec: TestMatrixSpec, r0, r1, c0, c1, ctx=None):
    ctx = _ctx(ctx)
    out = qzeros(r1 - r0, c1 - c0)
    s = spec.c()
    ctx._check(ctx.lib.qlra_gen_test_matrix_block(ctx.h, C.byref(s), r0, c0, C.byref(_qm(out))))
    return out


def gen_test_matrix(spec: TestMatrixSpec, ctx=None):
    return gen_block(spec, 0, spec.rows, 0, spec.cols, ctx)


def gen_test_matrix_rows(spec, r0, r1, ctx=None):
    return gen_block(spec, r0, r1, 0, spec.cols, ctx)


def gen_test_matrix_cols(spec, c0, c1, ctx=None):
    return gen_block(spec, 0, spec.rows, c0, c1, ctx)


# ------------------------------------------------------------- sketch ---
@dataclass
class SketchState:
    """== SketchState (sketching.hpp:38-47); y is the rank's row shard."""
    y: torch.Tensor
    w: torch.Tensor
    omega_spec: TestMatrixSpec
    psi_spec: TestMatrixSpec
    r: int
    s: int
    l: int
    row0: int = 0  # global index of y's first row (multi-GPU shards)

    def data_rows(self):
        return self.psi_spec.cols

    def data_cols(self):
        return self.w.shape[2]


def shard_rows(m: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [r0, r1) of A (and Y, H) owned by `rank` of `world`:
    contiguous, balanced to within one row, ordered by rank."""
    if not (0 <= rank < world):
        raise ParameterError("shard_rows: rank out of range")
    return m * rank // world, m * (rank + 1) // world


def validate_sketch_sizes(m, n, r, s, l):
    if r < 1 or not (r <= s <= l <= min(m, n)):
        raise ParameterError("sketch sizes must satisfy 1 <= r <= s <= l <= min(m,n)")


def empty_sketch(m, n, r, s, l, omega_seed, psi_seed, kind=GAUSSIAN, density=1.0, rows_local=None,
                 row0=0):
    """sketching.cpp:110-123 (rows_local/row0 select this rank's Y shard)."""
    validate_sketch_sizes(m, n, r, s, l)
    if not (0.0 < density <= 1.0):
        raise ParameterError("test matrix: density must lie in (0,1]")
    ml = m if rows_local is None else rows_local
    return SketchState(qzeros(ml, s), qzeros(l, n), TestMatrixSpec(kind, n, s, omega_seed, density),
                       TestMatrixSpec(kind, l, m, psi_seed, density), r, s, l, row0)


def sketch_update_rows(state: SketchState, row0: int, block: torch.Tensor, ctx=None):
    """sketching.cpp:125-139; row0 is the GLOBAL row index of block's first row."""
    ctx = _ctx(ctx)
    lr0 = row0 - state.row0
    if block.shape[2] != state.w.shape[2]:
        raise ShapeError("sketch_update_rows: column count mismatch")
    if lr0 < 0 or lr0 + block.shape[1] > state.y.shape[1]:
        raise ShapeError("sketch_update_rows: row range out of bounds")
    if block.shape[1] == 0:
        return
    yv = state.y[:, lr0:lr0 + block.shape[1], :]
    om, ps = state.omega_spec.c(), state.psi_spec.c()
    ctx._check(ctx.lib.qlra_sketch_update_rows(ctx.h, C.byref(om), C.byref(ps), row0,
                                               C.byref(_qm(block)), C.byref(_qm(yv)),
                                               C.byref(_qm(state.w))))


def sketch_update_rows_host(state: SketchState, row0: int, block_host: torch.Tensor, block_rows: int = 0,
                            ctx=None):
    """sketch_update_rows with the block in host memory (pinned for overlap):
    H2D row panels are streamed and double-buffered against the sketch."""
    ctx = _ctx(ctx)
    lr0 = row0 - state.row0
    if block_host.shape[2] != state.w.shape[2]:
        raise ShapeError("sketch_update_rows: column count mismatch")
    if lr0 < 0 or lr0 + block_host.shape[1] > state.y.shape[1]:
        raise ShapeError("sketch_update_rows: row range out of bounds")
    if block_host.shape[1] == 0:
        return
    yv = state.y[:, lr0:lr0 + block_host.shape[1], :]
    om, ps = state.omega_spec.c(), state.psi_spec.c()
    ctx._check(ctx.lib.qlra_sketch_update_rows_host(ctx.h, C.byref(om), C.byref(ps), row0,
                                                    C.byref(_qm(block_host, host=True)),
                                                    C.byref(_qm(yv)), C.byref(_qm(state.w)), block_rows))


def make_sketch_host(a_host, r, s, l, omega_seed, psi_seed, kind=GAUSSIAN, density=1.0, ctx=None, row0=0,
                     m_global=None, block_rows=0):
    """make_sketch from a host-resident (pinned) A: the public streaming entry."""
    ctx = _ctx(ctx)
    m = a_host.shape[1] if m_global is None else m_global
    st = empty_sketch(m, a_host.shape[2], r, s, l, omega_seed, psi_seed, kind, density,
                      rows_local=a_host.shape[1], row0=row0)
    sketch_update_rows_host(st, row0, a_host, block_rows, ctx)
    if ctx.nranks > 1:
        sketch_allreduce(st, ctx)
    return st


def sketch_allreduce(state: SketchState, ctx=None):
    ctx = _ctx(ctx)
    ctx._check(ctx.lib.qlra_sketch_allreduce(ctx.h, C.byref(_qm(state.w))))


def sketch_update(state: SketchState, delta: torch.Tensor, ctx=None):
    if delta.shape[1] != state.y.shape[1]:
        raise ShapeError("sketch_update: row count mismatch")
    sketch_update_rows(state, state.row0, delta, ctx)


def make_sketch(a, r, s, l, omega_seed, psi_seed, kind=GAUSSIAN, density=1.0, ctx=None, row0=0,
                m_global=None):
    """sketching.cpp:141-154.  With a row-sharded `a`, pass row0 / m_global and
    the W partials are all-reduced across ranks."""
    ctx = _ctx(ctx)
    m = a.shape[1] if m_global is None else m_global
    st = empty_sketch(m, a.shape[2], r, s, l, omega_seed, psi_seed, kind, density,
                      rows_local=a.shape[1], row0=row0)
    sketch_update_rows(st, row0, a, ctx)
    if ctx.nranks > 1:
        sketch_allreduce(st, ctx)
    return st


class MatrixSource:
    """sketching.hpp:67-74: the sketch builder is the only reader."""

    def rows(self) -> int:
        raise NotImplementedError

    def cols(self) -> int:
        raise NotImplementedError

    def read_rows(self, r0: int, r1: int) -> torch.Tensor:
        raise NotImplementedError


def sketch_from_source(source: MatrixSource, r, s, l, omega_seed, psi_seed, kind=GAUSSIAN,
                       density=1.0, block_rows=256, ctx=None):
    """sketching.cpp:156-167."""
    if block_rows < 1:
        raise ParameterError("sketch_from_source: block_rows must be >= 1")
    st = empty_sketch(source.rows(), source.cols(), r, s, l, omega_seed, psi_seed, kind, density)
    for r0 in range(0, source.rows(), block_rows):
        r1 = min(source.rows(), r0 + block_rows)
        sketch_update_rows(st, r0, source.read_rows(r0, r1), ctx)
    return st


# ----------------------------------------------------------- products ---
OP_N, OP_C = 0, 1


def qmat_mul(a, b, op_a=OP_N, op_b=OP_N, alpha=1.0, beta=0.0, out=None, ctx=None):
    """qmat_mul (qmatrix.cpp:165-197) generalised to alpha op(A) op(B) + beta C."""
    ctx = _ctx(ctx)
    m = a.shape[1] if op_a == OP_N else a.shape[2]
    n = b.shape[2] if op_b == OP_N else b.shape[1]
    if out is None:
        out = qzeros(m, n)
    ctx._check(ctx.lib.qlra_qmat_mul(ctx.h, op_a, op_b, alpha, C.byref(_qm(a)), C.byref(_qm(b)), beta,
                                     C.byref(_qm(out))))
    return out


def qmat_mul_ordered(a, b, ctx=None):
    return qmat_mul(a, b, ctx=ctx)


def gram(h, ctx=None):
    ctx = _ctx(ctx)
    g = qzeros(h.shape[2], h.shape[2])
    ctx._check(ctx.lib.qlra_gram(ctx.h, C.byref(_qm(h)), C.byref(_qm(g))))
    return g


# ----------------------------------------------------- complex bridge ---
# The reference's CMatrix (Eigen::MatrixXcd) is column-major: a complex128
# tensor here is passed as its column-major buffer (stride(0) == 1).
def czeros(rows, cols, device=None):
    """A column-major complex128 (rows, cols) CUDA tensor."""
    return torch.zeros((cols, rows), dtype=torch.complex128, device=device or "cuda").t()


def as_colmajor(t: torch.Tensor) -> torch.Tensor:
    return t if (t.dim() == 2 and t.stride(0) == 1) else t.t().contiguous().t()


def _cm(t: torch.Tensor) -> L.CMat:
    if t.dtype != torch.complex128 or t.dim() != 2 or not t.is_cuda:
        raise ShapeError("complex matrix must be a CUDA complex128 tensor (rows, cols)")
    if t.shape[0] > 1 and t.stride(0) != 1:
        raise ShapeError("complex matrix must be column-major (see as_colmajor)")
    return L.CMat(t.data_ptr(), t.shape[0], t.shape[1], max(1, t.stride(1) if t.shape[1] > 1 else t.shape[0]))


def to_compact(a, ctx=None):
    """to_compact (complex_bridge.cpp:11-20): [Q0; -conj(Q1)], 2m x n."""
    ctx = _ctx(ctx)
    out = czeros(2 * a.shape[1], a.shape[2])
    ctx._check(ctx.lib.qlra_to_compact(ctx.h, C.byref(_qm(a)), C.byref(_cm(out))))
    return out


def to_full(a, ctx=None):
    """to_full (complex_bridge.cpp:22-35): chi(A), 2m x 2n."""
    ctx = _ctx(ctx)
    out = czeros(2 * a.shape[1], 2 * a.shape[2])
    ctx._check(ctx.lib.qlra_to_full(ctx.h, C.byref(_qm(a)), C.byref(_cm(out))))
    return out


def from_compact(z, ctx=None):
    """from_compact (complex_bridge.cpp:37-52)."""
    ctx = _ctx(ctx)
    z = as_colmajor(z)
    if z.shape[0] % 2:
        raise ShapeError("from_compact: odd row count")
    out = qzeros(z.shape[0] // 2, z.shape[1])
    ctx._check(ctx.lib.qlra_from_compact(ctx.h, C.byref(_cm(z)), C.byref(_qm(out))))
    return out


def j_mul_conj(u, ctx=None):
    """j_mul_conj (complex_bridge.cpp:54-61): J conj(u)."""
    ctx = _ctx(ctx)
    u = as_colmajor(u)
    out = czeros(u.shape[0], u.shape[1])
    ctx._check(ctx.lib.qlra_j_mul_conj(ctx.h, C.byref(_cm(u)), C.byref(_cm(out))))
    return out


def complex_qr(m, ctx=None):
    """complex_qr (factorizations.cpp:33-51): thin (Q, R), diag(R) real >= 0."""
    ctx = _ctx(ctx)
    m = as_colmajor(m)
    q, r = czeros(m.shape[0], m.shape[1]), czeros(m.shape[1], m.shape[1])
    ctx._check(ctx.lib.qlra_complex_qr(ctx.h, C.byref(_cm(m)), C.byref(_cm(q)), C.byref(_cm(r))))
    return q, r


def complex_svd(m, ctx=None):
    """complex_svd (factorizations.cpp:53-56): compact (U, s, V), s nonincreasing."""
    ctx = _ctx(ctx)
    m = as_colmajor(m)
    k = min(m.shape)
    u, v = czeros(m.shape[0], k), czeros(m.shape[1], k)
    s = (C.c_double * max(1, k))()
    ctx._check(ctx.lib.qlra_complex_svd(ctx.h, C.byref(_cm(m)), C.byref(_cm(u)), s, C.byref(_cm(v))))
    return u, [s[i] for i in range(k)], v


def qmat_pinv(a, ctx=None):
    """qmat_pinv (factorizations.cpp:303-314)."""
    ctx = _ctx(ctx)
    out = qzeros(a.shape[2], a.shape[1])
    ctx._check(ctx.lib.qlra_qmat_pinv(ctx.h, C.byref(_qm(a)), C.byref(_qm(out))))
    return out


def spectral_norm(a, ctx=None):
    """spectral_norm (factorizations.cpp:324-327)."""
    ctx = _ctx(ctx)
    v = C.c_double()
    ctx._check(ctx.lib.qlra_spectral_norm(ctx.h, C.byref(_qm(a)), C.byref(v)))
    return v.value


# -------------------------------------------------------- small dense ---
def condition_number(a, ctx=None):
    ctx = _ctx(ctx)
    k = C.c_double()
    ctx._check(ctx.lib.qlra_condition_number(ctx.h, C.byref(_qm(a)), C.byref(k)))
    return k.value


def singular_values(a, ctx=None):
    ctx = _ctx(ctx)
    k = min(a.shape[1], a.shape[2]) if ctx.nranks == 1 else a.shape[2]
    out = (C.c_double * max(1, k))()
    ctx._check(ctx.lib.qlra_singular_values(ctx.h, C.byref(_qm(a)), out))
    return [out[i] for i in range(k)]


def solve_quaternion_linear(a, b, ctx=None):
    """complex_bridge.cpp:63-90."""
    ctx = _ctx(ctx)
    x = qzeros(a.shape[2], b.shape[2])
    ctx._check(ctx.lib.qlra_solve_quaternion_linear(ctx.h, C.byref(_qm(a)), C.byref(_qm(b)),
                                                    C.byref(_qm(x))))
    return x


# ------------------------------------------------------- rangefinders ---
@dataclass
class PseudoQrConfig:
    """== PseudoQrConfig (rangefinders.hpp:23-27)."""
    max_correction_steps: int = 3
    power_iters_for_epsilon: int = 3
    delta_budget: float = 1.2


@dataclass
class RangefinderReport:
    """== RangefinderReport (rangefinders.hpp:14-21)."""
    h: torch.Tensor
    kappa_before: float = 0.0
    kappa_after: float = 0.0
    correction_steps_used: int = 0
    method: int = PSEUDO_QR


def estimate_epsilon(h, power_iters=3, ctx=None):
    ctx = _ctx(ctx)
    e = C.c_double()
    ctx._check(ctx.lib.qlra_estimate_epsilon(ctx.h, C.byref(_qm(h)), power_iters, C.byref(e)))
    return e.value


def correction_step(h, epsilon, ctx=None):
    ctx = _ctx(ctx)
    out = torch.empty_like(h)
    ctx._check(ctx.lib.qlra_correction_step(ctx.h, C.byref(_qm(h)), epsilon, C.byref(_qm(out))))
    return out


def pseudo_qr(y, cfg: PseudoQrConfig = PseudoQrConfig(), ctx=None) -> RangefinderReport:
    """Algorithm 1 (rangefinders.cpp:107-158)."""
    ctx = _ctx(ctx)
    h = torch.empty_like(y)
    c = L.PseudoQrConfig(cfg.max_correction_steps, cfg.power_iters_for_epsilon, cfg.delta_budget)
    rep = L.Report()
    ctx._check(ctx.lib.qlra_pseudo_qr(ctx.h, C.byref(_qm(y)), C.byref(c), C.byref(_qm(h)), C.byref(rep)))
    return RangefinderReport(h, rep.kappa_before, rep.kappa_after, rep.correction_steps_used, PSEUDO_QR)


def pseudo_svd(y, seed=DEFAULT_RANGEFINDER_SEED, ctx=None) -> RangefinderReport:
    """Algorithm 3 (rangefinders.cpp:166-176): orthonormal H spanning range(Y)."""
    ctx = _ctx(ctx)
    h = torch.empty_like(y)
    rep = L.Report()
    ctx._check(ctx.lib.qlra_pseudo_svd(ctx.h, C.byref(_qm(y)), seed, C.byref(_qm(h)), C.byref(rep)))
    return RangefinderReport(h, rep.kappa_before, rep.kappa_after, 0, PSEUDO_SVD)


def orthonormal_range(y, seed=DEFAULT_RANGEFINDER_SEED, ctx=None):
    """orthonormal_range (rangefinders.cpp:160-164): the pseudo-SVD basis of
    range(Y), rows >= cols."""
    ctx = _ctx(ctx)
    h = torch.empty_like(y)
    ctx._check(ctx.lib.qlra_orthonormal_range(ctx.h, C.byref(_qm(y)), seed, C.byref(_qm(h))))
    return h


# ------------------------------------------------------------ QB stage ---
@dataclass
class QbResult:
    """== QbResult (sketching.hpp:88-94)."""
    h: torch.Tensor
    x: torch.Tensor
    report: RangefinderReport
    rangefinder_s: float = 0.0
    solve_s: float = 0.0


def qb_solve(psi_spec: TestMatrixSpec, h, w, row0=0, ctx=None):
    ctx = _ctx(ctx)
    x = qzeros(h.shape[2], w.shape[2])
    ps = psi_spec.c()
    ctx._check(ctx.lib.qlra_qb_solve(ctx.h, C.byref(ps), row0, C.byref(_qm(h)), C.byref(_qm(w)),
                                     C.byref(_qm(x))))
    return x


def qb_stage(state: SketchState, method=PSEUDO_QR, rangefinder_seed=DEFAULT_RANGEFINDER_SEED,
             qr_cfg: PseudoQrConfig = PseudoQrConfig(), ctx=None, timer: Callable | None = None,
             split: bool = False) -> QbResult:
    """qb_stage (sketching.cpp:169-194): rangefinder on Y, then X = (Psi H) \\ W
    with Psi regenerated from its spec.  Never touches A.  One call
    (qlra_qb_stage: the solve starts inside pseudo-QR) unless `split`, which
    runs the rangefinder and the solve as two calls and times them apart
    (rangefinder_s / solve_s; the fused call reports its total as rangefinder_s)."""
    ctx = _ctx(ctx)
    if method not in (PSEUDO_QR, PSEUDO_SVD):
        raise ParameterError("qb_stage: unknown rangefinder")
    if not split:
        t0 = time.perf_counter()
        h = torch.empty_like(state.y)
        x = qzeros(state.y.shape[2], state.w.shape[2])
        c = L.PseudoQrConfig(qr_cfg.max_correction_steps, qr_cfg.power_iters_for_epsilon, qr_cfg.delta_budget)
        rep = L.Report()
        ps = state.psi_spec.c()
        ctx._check(ctx.lib.qlra_qb_stage(ctx.h, C.byref(ps), state.row0, C.byref(_qm(state.y)),
                                         C.byref(_qm(state.w)), method, rangefinder_seed, C.byref(c),
                                         C.byref(_qm(h)), C.byref(_qm(x)), C.byref(rep)))
        ctx.synchronize()
        steps = rep.correction_steps_used if method == PSEUDO_QR else 0
        rr = RangefinderReport(h, rep.kappa_before, rep.kappa_after, steps, method)
        return QbResult(h, x, rr, time.perf_counter() - t0, 0.0)
    t0 = time.perf_counter()
    rep = pseudo_qr(state.y, qr_cfg, ctx) if method == PSEUDO_QR else pseudo_svd(state.y, rangefinder_seed, ctx)
    t1 = time.perf_counter()
    x = qb_solve(state.psi_spec, rep.h, state.w, state.row0, ctx)
    ctx.synchronize()
    t2 = time.perf_counter()
    return QbResult(rep.h, x, rep, t1 - t0, t2 - t1)


def qb_stage_with_psi(state: SketchState, psi, method=PSEUDO_QR, rangefinder_seed=DEFAULT_RANGEFINDER_SEED,
                      qr_cfg: PseudoQrConfig = PseudoQrConfig(), ctx=None) -> QbResult:
    """qb_stage_with_psi (sketching.cpp:169-188) with an explicit Psi: `psi` is
    the (l x rows) column slice of Psi matching state.y's rows (the whole Psi
    on one rank)."""
    ctx = _ctx(ctx)
    if method not in (PSEUDO_QR, PSEUDO_SVD):
        raise ParameterError("qb_stage: unknown rangefinder")
    t0 = time.perf_counter()
    h = torch.empty_like(state.y)
    x = qzeros(state.y.shape[2], state.w.shape[2])
    c = L.PseudoQrConfig(qr_cfg.max_correction_steps, qr_cfg.power_iters_for_epsilon, qr_cfg.delta_budget)
    rep = L.Report()
    ctx._check(ctx.lib.qlra_qb_stage_with_psi(ctx.h, C.byref(_qm(psi)), C.byref(_qm(state.y)),
                                              C.byref(_qm(state.w)), method, rangefinder_seed, C.byref(c),
                                              C.byref(_qm(h)), C.byref(_qm(x)), C.byref(rep)))
    ctx.synchronize()
    steps = rep.correction_steps_used if method == PSEUDO_QR else 0
    return QbResult(h, x, RangefinderReport(h, rep.kappa_before, rep.kappa_after, steps, method),
                    time.perf_counter() - t0, 0.0)


def residual_fro(a, h, x, ctx=None):
    """(||A - H X||_F, ||A||_F) over row-shards (sketching.cpp:270-271)."""
    ctx = _ctx(ctx)
    r, n = C.c_double(), C.c_double()
    ctx._check(ctx.lib.qlra_residual_fro(ctx.h, C.byref(_qm(a)), C.byref(_qm(h)), C.byref(_qm(x)),
                                         C.byref(r), C.byref(n)))
    return r.value, n.value


@dataclass
class OnePassOptions:
    """== OnePassOptions (sketching.hpp:130-141)."""
    r: int = 0
    s: int = -1
    l: int = -1
    rangefinder: int = PSEUDO_QR
    embedding: int = GAUSSIAN
    density: float = 1.0
    omega_seed: int = 1
    psi_seed: int = 2
    rangefinder_seed: int = DEFAULT_RANGEFINDER_SEED
    qr_cfg: PseudoQrConfig = field(default_factory=PseudoQrConfig)


def resolve_defaults(opts: OnePassOptions) -> OnePassOptions:
    """sketching.cpp:222-227."""
    if opts.r < 1:
        raise ParameterError("one_pass_approx: rank must be >= 1")
    import copy
    o = copy.copy(opts)
    if o.s < 0:
        o.s = o.r + 5
    if o.l < 0:
        o.l = 2 * o.s
    return o


@dataclass
class OnePassQb:
    state: SketchState
    qb: QbResult
    qb_residual: float | None
    a_fro: float | None
    times: dict


def one_pass_qb(a, opts: OnePassOptions, ctx=None, row0=0, m_global=None, residual=True) -> OnePassQb:
    """one_pass_approx (sketching.cpp:250-275) through the QB stage: sketch
    (one read of A), rangefinder, core solve, and (diagnostic, second read)
    the QB residual.  Truncation is reported separately."""
    ctx = _ctx(ctx)
    o = resolve_defaults(opts)
    t0 = time.perf_counter()
    st = make_sketch(a, o.r, o.s, o.l, o.omega_seed, o.psi_seed, o.embedding, o.density, ctx,
                     row0=row0, m_global=m_global)
    ctx.synchronize()
    t1 = time.perf_counter()
    qb = qb_stage(st, o.rangefinder, o.rangefinder_seed, o.qr_cfg, ctx)
    res = an = None
    if residual:
        res, an = residual_fro(a, qb.h, qb.x, ctx)
    return OnePassQb(st, qb, res, an, dict(sketch_s=t1 - t0, rangefinder_s=qb.rangefinder_s,
                                           solve_s=qb.solve_s))


def one_pass_qb_fused(a, r, s, l, omega_seed, psi_seed, kind=GAUSSIAN, density=1.0, method=PSEUDO_QR,
                      rangefinder_seed=DEFAULT_RANGEFINDER_SEED, qr_cfg: PseudoQrConfig = PseudoQrConfig(),
                      ctx=None, row0=0, m_global=None):
    """make_sketch + qb_stage (sketching.cpp:141-154, 169-194) as ONE C-ABI
    call (qlra_one_pass_qb) on a device-resident row shard: returns
    (SketchState, QbResult)."""
    ctx = _ctx(ctx)
    if method not in (PSEUDO_QR, PSEUDO_SVD):
        raise ParameterError("qb_stage: unknown rangefinder")
    m = a.shape[1] if m_global is None else m_global
    st = empty_sketch(m, a.shape[2], r, s, l, omega_seed, psi_seed, kind, density,
                      rows_local=a.shape[1], row0=row0)
    t0 = time.perf_counter()
    h = torch.empty_like(st.y)
    x = qzeros(s, st.w.shape[2])
    c = L.PseudoQrConfig(qr_cfg.max_correction_steps, qr_cfg.power_iters_for_epsilon, qr_cfg.delta_budget)
    rep = L.Report()
    om, ps = st.omega_spec.c(), st.psi_spec.c()
    ctx._check(ctx.lib.qlra_one_pass_qb(ctx.h, C.byref(_qm(a)), row0, C.byref(om), C.byref(ps), method,
                                        rangefinder_seed, C.byref(c), C.byref(_qm(st.y)), C.byref(_qm(st.w)),
                                        C.byref(_qm(h)), C.byref(_qm(x)), C.byref(rep)))
    ctx.synchronize()
    steps = rep.correction_steps_used if method == PSEUDO_QR else 0
    rr = RangefinderReport(h, rep.kappa_before, rep.kappa_after, steps, method)
    return st, QbResult(h, x, rr, time.perf_counter() - t0, 0.0)


def one_pass_qb_host(a_host, opts: OnePassOptions, ctx=None, row0=0, m_global=None, block_rows=0,
                     h_out=None, x_out=None) -> QbResult:
    """one_pass_approx through the QB stage (sketching.cpp:250-263), host in and
    host out: A (pinned) streams through the overlapped H2D + sketch pipeline,
    H comes back while the core solve runs, then X.  One C-ABI call."""
    ctx = _ctx(ctx)
    o = resolve_defaults(opts)
    rows, n = a_host.shape[1], a_host.shape[2]
    m = rows if m_global is None else m_global
    validate_sketch_sizes(m, n, o.r, o.s, o.l)
    om = TestMatrixSpec(o.embedding, n, o.s, o.omega_seed, o.density).c()
    ps = TestMatrixSpec(o.embedding, o.l, m, o.psi_seed, o.density).c()
    h = h_out if h_out is not None else torch.empty((4, rows, o.s), dtype=torch.float64, pin_memory=True)
    x = x_out if x_out is not None else torch.empty((4, o.s, n), dtype=torch.float64, pin_memory=True)
    cfg = L.PseudoQrConfig(o.qr_cfg.max_correction_steps, o.qr_cfg.power_iters_for_epsilon,
                           o.qr_cfg.delta_budget)
    rep = L.Report()
    ctx._check(ctx.lib.qlra_one_pass_qb_host(ctx.h, C.byref(_qm(a_host, True)), row0, C.byref(om),
                                             C.byref(ps), o.rangefinder, o.rangefinder_seed, C.byref(cfg),
                                             block_rows, C.byref(_qm(h, True)), C.byref(_qm(x, True)),
                                             C.byref(rep)))
    r = RangefinderReport(h, rep.kappa_before, rep.kappa_after, rep.correction_steps_used, rep.method)
    return QbResult(h, x, r, 0.0, 0.0)


# --------------------------------------------------------- truncation ---
def qsvd(a, ctx=None):
    """qsvd (factorizations.cpp:166-295): (U, sigma, V) with A = U diag(sigma) V^*."""
    ctx = _ctx(ctx)
    m, n = a.shape[1], a.shape[2]
    k = min(m, n)
    u, v = qzeros(m, k), qzeros(n, k)
    sg = (C.c_double * max(1, k))()
    ctx._check(ctx.lib.qlra_qsvd(ctx.h, C.byref(_qm(a)), C.byref(_qm(u)), sg, C.byref(_qm(v))))
    return u, [sg[i] for i in range(k)], v


@dataclass
class ApproxResult:
    """== ApproxResult (sketching.hpp:118-123)."""
    h: torch.Tensor
    sigma: list
    v: torch.Tensor
    diagnostics: dict = field(default_factory=dict)


def truncate_stage(h, x, r, ctx=None) -> ApproxResult:
    """truncate_stage (sketching.cpp:196-211): QSVD of X, keep r triples, fold U_r into H."""
    ctx = _ctx(ctx)
    ho, v = qzeros(h.shape[1], r), qzeros(x.shape[2], r)
    sg = (C.c_double * max(1, r))()
    ctx._check(ctx.lib.qlra_truncate_stage(ctx.h, C.byref(_qm(h)), C.byref(_qm(x)), r, C.byref(_qm(ho)), sg,
                                           C.byref(_qm(v))))
    return ApproxResult(ho, [sg[i] for i in range(r)], v)


def approx_reconstruct(res: ApproxResult, ctx=None):
    """approx_reconstruct (sketching.cpp:213-218): H diag(sigma) V^*."""
    ctx = _ctx(ctx)
    hs = res.h * torch.tensor(res.sigma, dtype=torch.float64, device=res.h.device)[None, None, :]
    return qmat_mul(hs, res.v, op_b=OP_C, ctx=ctx)


def approx_residual_fro(a, res: ApproxResult, ctx=None):
    """(||A - H S V^*||_F, ||A||_F) -- relative_error's terms (analysis.cpp:75-79)."""
    ctx = _ctx(ctx)
    sg = (C.c_double * max(1, len(res.sigma)))(*res.sigma)
    r, n = C.c_double(), C.c_double()
    ctx._check(ctx.lib.qlra_approx_residual_fro(ctx.h, C.byref(_qm(a)), C.byref(_qm(res.h)), sg,
                                                C.byref(_qm(res.v)), C.byref(r), C.byref(n)))
    return r.value, n.value


def one_pass_approx(a, opts: OnePassOptions, ctx=None) -> ApproxResult:
    """one_pass_approx (sketching.cpp:250-275): sketch -> QB stage -> truncation,
    with the qb_residual / relative_error diagnostics (second read of A)."""
    ctx = _ctx(ctx)
    o = resolve_defaults(opts)
    t0 = time.perf_counter()
    st = make_sketch(a, o.r, o.s, o.l, o.omega_seed, o.psi_seed, o.embedding, o.density, ctx)
    ctx.synchronize()
    t1 = time.perf_counter()
    # the rangefinder and the solve as two calls, timed apart like the
    # reference's StageTimes (sketching.cpp:176-186)
    qb = qb_stage(st, o.rangefinder, o.rangefinder_seed, o.qr_cfg, ctx, split=True)
    t2 = time.perf_counter()
    res = truncate_stage(qb.h, qb.x, o.r, ctx)
    ctx.synchronize()
    t3 = time.perf_counter()
    qres, na = residual_fro(a, qb.h, qb.x, ctx)
    diff, _ = approx_residual_fro(a, res, ctx)
    rel = diff / na if na > 0 else (float("inf") if diff > 0 else 0.0)
    res.diagnostics = dict(kappa_h=qb.report.kappa_after, kappa_before=qb.report.kappa_before,
                           correction_steps=qb.report.correction_steps_used, qb_residual=qres,
                           relative_error=rel,
                           times=dict(sketch_s=t1 - t0, rangefinder_s=qb.rangefinder_s, solve_s=qb.solve_s,
                                      truncate_s=t3 - t2))
    return res


def one_pass_approx_from_sketch(state: SketchState, opts: OnePassOptions, ctx=None) -> ApproxResult:
    """one_pass_approx(const SketchState&, opts) (sketching.cpp:220-246,
    run_pipeline): QB stage + truncation from a sketch; A is never touched, so
    the residual diagnostics are absent."""
    ctx = _ctx(ctx)
    o = resolve_defaults(opts)
    qb = qb_stage(state, o.rangefinder, o.rangefinder_seed, o.qr_cfg, ctx, split=True)
    t0 = time.perf_counter()
    res = truncate_stage(qb.h, qb.x, o.r, ctx)
    ctx.synchronize()
    res.diagnostics = dict(kappa_h=qb.report.kappa_after, kappa_before=qb.report.kappa_before,
                           correction_steps=qb.report.correction_steps_used, qb_residual=None,
                           relative_error=None,
                           times=dict(sketch_s=0.0, rangefinder_s=qb.rangefinder_s, solve_s=qb.solve_s,
                                      truncate_s=time.perf_counter() - t0))
    return res


# ------------------------------------------------------- checkpoint I/O ---
def write_qmat(path, m, ctx=None):
    """write_qmat (io.cpp:77-88): QMAT1 file from a device QMatrix."""
    ctx = _ctx(ctx)
    ctx._check(ctx.lib.qlra_write_qmat(ctx.h, str(path).encode(), C.byref(_qm(m))))


def read_qmat(path, ctx=None):
    """read_qmat (io.cpp:89-114) into a new device QMatrix."""
    ctx = _ctx(ctx)
    r, c = C.c_int64(), C.c_int64()
    rc = L.lib().qlra_qmat_file_shape(str(path).encode(), C.byref(r), C.byref(c))
    if rc != 0:
        raise IoError(f"not a readable QMAT1 file: {path}")
    m = qzeros(r.value, c.value)
    ctx._check(ctx.lib.qlra_read_qmat(ctx.h, str(path).encode(), C.byref(_qm(m))))
    return m


def _spec_from_c(cs) -> TestMatrixSpec:
    return TestMatrixSpec(cs.kind, cs.rows, cs.cols, cs.seed, cs.density)


def write_sketch(path, st: SketchState, ctx=None):
    """write_sketch (io.cpp:116-128): QSKT1 checkpoint of a sketch state."""
    ctx = _ctx(ctx)
    om, ps = st.omega_spec.c(), st.psi_spec.c()
    ctx._check(ctx.lib.qlra_write_sketch(ctx.h, str(path).encode(), C.byref(om), C.byref(ps), st.r, st.s,
                                         st.l, C.byref(_qm(st.y)), C.byref(_qm(st.w))))


def read_sketch(path, ctx=None) -> SketchState:
    """read_sketch (io.cpp:130-145)."""
    ctx = _ctx(ctx)
    om, ps, rsl, dims = L.Spec(), L.Spec(), (C.c_int64 * 3)(), (C.c_int64 * 4)()
    if L.lib().qlra_sketch_file_header(str(path).encode(), C.byref(om), C.byref(ps), rsl) != 0:
        raise IoError(f"not a readable QSKT1 file: {path}")
    # Y and W are sized from their own QMAT1 headers, validated before any
    # allocation (io.cpp:130-145)
    if L.lib().qlra_sketch_file_dims(str(path).encode(), dims) != 0:
        raise IoError("read_sketch: inconsistent dimensions")
    st = SketchState(qzeros(dims[0], dims[1]), qzeros(dims[2], dims[3]), _spec_from_c(om), _spec_from_c(ps),
                     rsl[0], rsl[1], rsl[2])
    ctx._check(ctx.lib.qlra_read_sketch(ctx.h, str(path).encode(), C.byref(_qm(st.y)), C.byref(_qm(st.w))))
    return st


def sketch_from_qmat_file(path, r, s, l, omega_seed, psi_seed, kind=GAUSSIAN, density=1.0, block_rows=256,
                          ctx=None) -> SketchState:
    """sketch_from_source over a QMAT1 file (QmatFileSource, io.cpp:213-239):
    the file is the only reader of A; blocks stream through pinned buffers."""
    ctx = _ctx(ctx)
    rr, cc = C.c_int64(), C.c_int64()
    if L.lib().qlra_qmat_file_shape(str(path).encode(), C.byref(rr), C.byref(cc)) != 0:
        raise IoError(f"not a readable QMAT1 file: {path}")
    if block_rows < 1:
        raise ParameterError("sketch_from_source: block_rows must be >= 1")
    st = empty_sketch(rr.value, cc.value, r, s, l, omega_seed, psi_seed, kind, density)
    om, ps = st.omega_spec.c(), st.psi_spec.c()
    ctx._check(ctx.lib.qlra_sketch_from_qmat_file(ctx.h, str(path).encode(), C.byref(om), C.byref(ps),
                                                  C.byref(_qm(st.y)), C.byref(_qm(st.w)), block_rows))
    return st


def measure_fp64_peak(mode=0, ms=200.0, ctx=None):
    ctx = _ctx(ctx)
    t = C.c_double()
    ctx._check(ctx.lib.qlra_measure_fp64_peak(ctx.h, mode, ms, C.byref(t)))
    return t.value


def sketch_kernel_name():
    return L.lib().qlra_sketch_kernel_name().decode()


def int8_engine_name():
    return L.lib().qlra_int8_engine_name().decode()


def measure_int8_peak(ms=300.0, ctx=None):
    """TOPS of back-to-back int8 8192^3 GEMMs (the int8 engine's roofline
    denominator, measured in the same run)."""
    ctx = _ctx(ctx)
    t = C.c_double()
    ctx._check(ctx.lib.qlra_measure_int8_peak(ctx.h, ms, C.byref(t)))
    return t.value
