/*
 * qlra_cuda.h -- C-ABI of the B200-native one-pass quaternion LRA hot path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no C++/torch types.
 * Each entry point replaces one function of the reference's public C++ API
 * (proj/include/qlra/*.hpp of arXiv 2404.14783's reference `qlra`); the
 * replaced declaration is cited beside every prototype.  The C++ facade in
 * paper_2404_14783_b200/csrc/qlra_gpu.hpp wraps these with the reference's
 * signatures and rethrows the reference's exception types
 * (proj/include/qlra/errors.hpp:9-43).
 *
 * Data model (proj/include/qlra/qmatrix.hpp:14-19): a quaternion matrix is four
 * row-major FP64 planes (w, x, y, z) in DEVICE memory, each with leading
 * dimension `ld` (>= cols).  All calls are asynchronous on the context's
 * stream unless noted ("syncs"); results are run-to-run bitwise deterministic
 * (no floating-point atomics, fixed reduction order).
 *
 * Multi-GPU (one process per GPU): a context created with nranks > 1 owns an
 * NCCL communicator.  Data matrices are row-sharded: each rank passes its
 * local rows of A / Y / H with `row0` = global index of its first row; W, X
 * and all small matrices are replicated.  Reductions over rows (W, Grams,
 * Psi*H, norms) are NCCL all-reduces inside the calls.  The same sharded
 * code also runs over an in-process communicator (qlra_group_t: one context
 * per host thread, any devices of the process, including several ranks on ONE
 * GPU, which NCCL refuses): the library sums the ranks' buffers itself, in
 * rank order.
 */
#ifndef QLRA_CUDA_H
#define QLRA_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: 1..6 mirror the reference exception taxonomy
 * (errors.hpp: ShapeError, ParameterError, SingularMatrixError, RankError,
 * PreconditionError, IoError). */
enum {
  QLRA_OK = 0,
  QLRA_ERR_SHAPE = 1,
  QLRA_ERR_PARAMETER = 2,
  QLRA_ERR_SINGULAR = 3,
  QLRA_ERR_RANK = 4,
  QLRA_ERR_PRECONDITION = 5,
  QLRA_ERR_IO = 6,
  QLRA_ERR_INTERNAL = 99,
  QLRA_ERR_CUDA = 100,
  QLRA_ERR_NCCL = 101
};

/* TestMatrixKind (sketching.hpp:14) */
enum { QLRA_GAUSSIAN = 0, QLRA_RADEMACHER = 1, QLRA_SPARSE_GAUSSIAN = 2, QLRA_SPARSE_RADEMACHER = 3 };
/* RangefinderMethod (rangefinders.hpp:12) */
enum { QLRA_PSEUDO_QR = 0, QLRA_PSEUDO_SVD = 1 };
/* operand transform for qlra_qmat_mul */
enum { QLRA_OP_N = 0, QLRA_OP_C = 1 /* conjugate transpose */ };

typedef struct qlra_ctx qlra_ctx_t;
typedef struct qlra_group qlra_group_t;

/* == TestMatrixSpec (sketching.hpp:22-28) */
typedef struct {
  int32_t kind;
  int64_t rows, cols;
  uint64_t seed;
  double density;
} qlra_spec_t;

/* Device view of a QMatrix (qmatrix.hpp:17-84): planes p[0..3] = w,x,y,z. */
typedef struct {
  double* p[4];
  int64_t rows, cols, ld;
} qlra_qmat_t;

/* Device view of a complex matrix -- the reference's CMatrix
 * (Eigen::MatrixXcd, complex_bridge.hpp:9): column-major, interleaved
 * (re, im) doubles, leading dimension ld >= rows. */
typedef struct {
  double* data;
  int64_t rows, cols, ld;
} qlra_cmat_t;

/* == PseudoQrConfig (rangefinders.hpp:23-27) */
typedef struct {
  int32_t max_correction_steps;    /* default 3 */
  int32_t power_iters_for_epsilon; /* default 3 */
  double delta_budget;             /* default 1.2 */
} qlra_pseudo_qr_config_t;

/* == RangefinderReport minus h (rangefinders.hpp:14-21) */
typedef struct {
  double kappa_before;
  double kappa_after;
  int32_t correction_steps_used;
  int32_t method;
} qlra_rangefinder_report_t;

/* ------------------------------------------------------------ context --- */
/* Creates a context on `device`.  nranks > 1 requires a 128-byte NCCL unique
 * id (from qlra_nccl_unique_id on rank 0, broadcast by the caller). */
int qlra_ctx_create(qlra_ctx_t** ctx, int device, int rank, int nranks,
                    const void* nccl_unique_id);
int qlra_ctx_destroy(qlra_ctx_t* ctx);
/* In-process communicator of `nranks` contexts (no reference counterpart: the
 * reference is single-process).  Each rank's context is created
 * with qlra_ctx_create_local from its own host thread; every collective call
 * must then be made by all ranks, as with NCCL.  Destroy the group after its
 * contexts (QLRA_ERR_PRECONDITION while any is attached). */
int qlra_group_create(qlra_group_t** group, int nranks);
int qlra_group_destroy(qlra_group_t* group);
int qlra_ctx_create_local(qlra_ctx_t** ctx, int device, qlra_group_t* group, int rank);
/* Run all further work on an external cudaStream_t (e.g. torch's current
 * stream); NULL selects the legacy default stream.  The context's own
 * non-blocking stream (created by qlra_ctx_create) is released. */
int qlra_ctx_set_stream(qlra_ctx_t* ctx, void* cuda_stream);
int qlra_ctx_synchronize(qlra_ctx_t* ctx);
/* The cudaStream_t (as void*) all of this context's work is ordered on --
 * callers order their own copies / kernels against the library's with it. */
void* qlra_ctx_stream(const qlra_ctx_t* ctx);
int qlra_nccl_unique_id(void* out_128_bytes);
/* Message of the last failing call on this ctx; for QLRA_ERR_SINGULAR also
 * the condition estimate carried by SingularMatrixError (errors.hpp:23-30). */
const char* qlra_last_error(const qlra_ctx_t* ctx, double* estimated_condition);
/* Number of kernels this ctx has launched (diagnostics / bench evidence). */
int64_t qlra_ctx_launch_count(const qlra_ctx_t* ctx);
/* Start (enable=1, resetting) or stop per-launch CUDA-event timing of the
 * fused sketch kernel, and read it back: total device ms, launches, and the
 * algorithmic flops / bytes of A those launches processed; stats syncs. */
int qlra_ctx_kernel_timing(qlra_ctx_t* ctx, int enable);
int qlra_ctx_kernel_stats(qlra_ctx_t* ctx, double* ms, int64_t* launches, double* flops,
                          double* a_bytes);
/* Which engines the timed brackets covered (bit 1: the FP64 DMMA sketch
 * kernel, bit 2: the int8 engine's batched GEMMs) and the int8 tensor-core
 * ops issued inside them. */
int qlra_ctx_kernel_engines(qlra_ctx_t* ctx, int* engines, double* int8_ops);

/* Sketch engine (no reference counterpart: the reference has one CPU
 * product, qmat_mul_accumulate_ordered, qmatrix.cpp:203-242).
 *   QLRA_SKETCH_AUTO  the int8 engine where it is faster (n >= 2048 and
 *                     s, l >= 64), else DMMA; env QLRA_SKETCH_ENGINE=int8|dmma
 *                     overrides AUTO;
 *   QLRA_SKETCH_DMMA  FP64 tensor cores (8-product quaternion GEMM, every
 *                     multiply-add rounded in fp64);
 *   QLRA_SKETCH_INT8  INT8 tensor cores: the products of a 52-bit fixed-point
 *                     image of A, Omega, Psi computed exactly (Ozaki scheme,
 *                     CRT over 16 moduli), rounded once (needs n < 131056).
 * Both match the ordered reference sketch to ~1e-15 relative. */
#define QLRA_SKETCH_AUTO 0
#define QLRA_SKETCH_DMMA 1
#define QLRA_SKETCH_INT8 2
int qlra_ctx_set_sketch_engine(qlra_ctx_t* ctx, int engine);
/* The int8 engine's roofline denominator: TOPS of back-to-back int8 8192^3
 * GEMMs on this GPU for ~ms milliseconds, and the engine's description. */
int qlra_measure_int8_peak(qlra_ctx_t* ctx, double ms, double* tops);
const char* qlra_int8_engine_name(void);
/* The int8 engine's contraction on its own (csrc/i8gemm.cu: tcgen05.mma
 * kind::i8, TMA-staged, int32 accumulators in TMEM): for b < batch, exact,
 *   mode 0: C[b][m*ldc + n] = (beta ? C : 0) + sum_k A[b][m*lda + k] B[b][n*ldb + k]
 *   mode 1: C[b][n*ldc + m] = (beta ? C : 0) + sum_k A[b][k*lda + m] B[b][n*ldb + k]
 * i.e. the residue images of Y += A Omega (mode 0) and of W^* += A^* Psi^*
 * (mode 1) in sketch_update_rows (sketching.cpp:125-139), both read from the
 * same row-major residue panel.  Device pointers, 16-byte aligned; n, lda,
 * ldb, stride_a, stride_b multiples of 16, ldc and stride_c of 4 (mode 1: m
 * too -- TMA stores whole 16-byte units of C's contiguous extent). */
int qlra_i8gemm_batched(qlra_ctx_t* ctx, int mode, int64_t m, int64_t n, int64_t k, const int8_t* a, int64_t lda,
                        int64_t stride_a, const int8_t* b, int64_t ldb, int64_t stride_b, int32_t* c, int64_t ldc,
                        int64_t stride_c, int batch, int beta);
const char* qlra_i8gemm_kernel_name(void);

/* ---------------------------------------------------------- embeddings --- */
/* gen_block (sketching.cpp:53-71) / gen_test_matrix{,_rows,_cols}
 * (sketching.hpp:30-32): writes entries [r0, r0+out->rows) x [c0, c0+out->cols)
 * of the spec into `out`.  Counter-based: any block is bit-identical in its
 * integer draws to the same block of the full matrix. */
int qlra_gen_test_matrix_block(qlra_ctx_t* ctx, const qlra_spec_t* spec, int64_t r0, int64_t c0,
                               qlra_qmat_t* out);

/* ------------------------------------------------------------- sketch --- */
/* sketch_update_rows (sketching.hpp:65, sketching.cpp:125-139):
 *   y_rows += block * Omega           (y_rows: the block's rows of Y)
 *   w      += Psi[:, row0:row0+b] * block
 * One launch of the fused sketch kernel reads each element of `block` from
 * HBM once.  Omega and the Psi column slice are regenerated on device from
 * their specs (rng.hpp:10-55).  With nranks > 1, `w` accumulates the rank's
 * partial; call qlra_sketch_allreduce once all local rows are in. */
int qlra_sketch_update_rows(qlra_ctx_t* ctx, const qlra_spec_t* omega, const qlra_spec_t* psi,
                            int64_t row0, const qlra_qmat_t* block, qlra_qmat_t* y_rows,
                            qlra_qmat_t* w);
/* Streaming form of qlra_sketch_update_rows (sketch_from_source,
 * sketching.cpp:156-167, with the source in host memory): `host_block` holds
 * HOST plane pointers (pinned memory for full overlap).  Row panels of
 * `block_rows` rows (0 = automatic) are copied H2D on an internal stream,
 * double-buffered against the fused sketch of the previous panel, so the
 * transfer of A overlaps the FP64 work and A is still read exactly once. */
int qlra_sketch_update_rows_host(qlra_ctx_t* ctx, const qlra_spec_t* omega,
                                 const qlra_spec_t* psi, int64_t row0,
                                 const qlra_qmat_t* host_block, qlra_qmat_t* y_rows,
                                 qlra_qmat_t* w, int64_t block_rows);
/* Sum of the per-rank W partials (NCCL all-reduce; no-op for one rank). */
int qlra_sketch_allreduce(qlra_ctx_t* ctx, qlra_qmat_t* w);

/* ------------------------------------------------------------ products --- */
/* qmat_mul (qmatrix.hpp:87, qmatrix.cpp:165-197) generalised:
 *   C = alpha * op(A) op(B) + beta * C,  op = identity or adjoint.
 * Not collective. */
int qlra_qmat_mul(qlra_ctx_t* ctx, int op_a, int op_b, double alpha, const qlra_qmat_t* a,
                  const qlra_qmat_t* b, double beta, qlra_qmat_t* c);
/* H^* H over row-sharded H (all-reduced): the Gram used by estimate_epsilon /
 * correction_step (rangefinders.cpp:68,102).  g is s x s. */
int qlra_gram(qlra_ctx_t* ctx, const qlra_qmat_t* h, qlra_qmat_t* g);

/* --------------------------------------------------- small dense (K4) --- */
/* condition_number (factorizations.hpp:54, factorizations.cpp:330-337) of a
 * row-sharded tall H; syncs. */
int qlra_condition_number(qlra_ctx_t* ctx, const qlra_qmat_t* h, double* kappa);
/* singular_values (factorizations.cpp:316-323) of a row-sharded tall A,
 * nonincreasing, min(rows, cols) values written to host `sv`; syncs. */
int qlra_singular_values(qlra_ctx_t* ctx, const qlra_qmat_t* a, double* sv);
/* solve_quaternion_linear (complex_bridge.hpp:36, complex_bridge.cpp:63-90):
 * square systems solve exactly; overdetermined ones return the least-squares
 * solution.  A, B replicated (not row-sharded).  syncs. */
int qlra_solve_quaternion_linear(qlra_ctx_t* ctx, const qlra_qmat_t* a, const qlra_qmat_t* b,
                                 qlra_qmat_t* x);

/* -------------------------------------------------------- rangefinders --- */
/* estimate_epsilon (rangefinders.hpp:50, rangefinders.cpp:66-97); syncs. */
int qlra_estimate_epsilon(qlra_ctx_t* ctx, const qlra_qmat_t* h, int power_iters, double* eps);
/* correction_step (rangefinders.hpp:46, rangefinders.cpp:99-105); h_out may
 * alias h; syncs. */
int qlra_correction_step(qlra_ctx_t* ctx, const qlra_qmat_t* h, double epsilon,
                         qlra_qmat_t* h_out);
/* pseudo_qr (rangefinders.hpp:40, rangefinders.cpp:107-158): Algorithm 1.
 * y, h: m x s (row-sharded), h may not alias y; syncs. */
int qlra_pseudo_qr(qlra_ctx_t* ctx, const qlra_qmat_t* y, const qlra_pseudo_qr_config_t* cfg,
                   qlra_qmat_t* h, qlra_rangefinder_report_t* report);
/* pseudo_svd (rangefinders.hpp:57, rangefinders.cpp:166-176): Algorithm 3,
 * orthonormal H with range(H) = range(Y); syncs. */
int qlra_pseudo_svd(qlra_ctx_t* ctx, const qlra_qmat_t* y, uint64_t seed, qlra_qmat_t* h,
                    qlra_rangefinder_report_t* report);
/* orthonormal_range (rangefinders.hpp:61, rangefinders.cpp:160-164): the
 * pseudo-SVD basis of range(Y) for rows >= cols (ParameterError otherwise),
 * without the condition bookkeeping.  syncs. */
int qlra_orthonormal_range(qlra_ctx_t* ctx, const qlra_qmat_t* y, uint64_t seed, qlra_qmat_t* h);

/* ------------------------------------------------ complex bridge --- */
/* complex_bridge.hpp:22-30 (complex_bridge.cpp:11-61): Q = Q0 + Q1 j,
 * compact Q_c = [Q0; -conj(Q1)] (2m x n), full chi = [Q0, Q1; -conj(Q1),
 * conj(Q0)] (2m x 2n), from_compact its inverse (odd row count ->
 * QLRA_ERR_SHAPE), j_mul_conj = J conj(u) (a block swap with one sign flip). */
int qlra_to_compact(qlra_ctx_t* ctx, const qlra_qmat_t* a, qlra_cmat_t* out);
int qlra_to_full(qlra_ctx_t* ctx, const qlra_qmat_t* a, qlra_cmat_t* out);
int qlra_from_compact(qlra_ctx_t* ctx, const qlra_cmat_t* z, qlra_qmat_t* out);
int qlra_j_mul_conj(qlra_ctx_t* ctx, const qlra_cmat_t* u, qlra_cmat_t* out);
/* complex_qr (factorizations.hpp:20-26, factorizations.cpp:33-51): thin
 * Q (p x q) and R (q x q) with diag(R) real and nonnegative, p >= q.  Runs
 * as CholeskyQR2 (shifted CholeskyQR3 when needed) in the complex subalgebra
 * of the quaternion kernels; numerically rank-deficient input (which the
 * reference's Householder QR still factors) -> QLRA_ERR_RANK.  syncs. */
int qlra_complex_qr(qlra_ctx_t* ctx, const qlra_cmat_t* m, qlra_cmat_t* q, qlra_cmat_t* r);
/* complex_svd (factorizations.hpp:28-34, factorizations.cpp:53-56): compact
 * SVD M = U diag(s) V^*, k = min(p, q), s nonincreasing (host array), through
 * the device QSVD of M as a quaternion matrix of its complex subalgebra
 * (whose factors stay complex).  syncs. */
int qlra_complex_svd(qlra_ctx_t* ctx, const qlra_cmat_t* m, qlra_cmat_t* u, double* s, qlra_cmat_t* v);
/* qmat_pinv (factorizations.hpp:72, factorizations.cpp:303-314): V S^+ U^*
 * with singular values <= max(m, n) eps sigma_max treated as zero; out is
 * n x m.  spectral_norm (:79, :324-327): sigma_max.  sync. */
int qlra_qmat_pinv(qlra_ctx_t* ctx, const qlra_qmat_t* a, qlra_qmat_t* out);
int qlra_spectral_norm(qlra_ctx_t* ctx, const qlra_qmat_t* a, double* norm);

/* --------------------------------------------------------- core solve --- */
/* The solve half of qb_stage_with_psi (sketching.cpp:184-185):
 *   X = argmin || (Psi H) X - W ||_F,   Psi regenerated from `psi`,
 * with H row-sharded (local rows start at global row `row0`), W and X
 * replicated (l x n and s x n).  Psi H is all-reduced.  syncs. */
int qlra_qb_solve(qlra_ctx_t* ctx, const qlra_spec_t* psi, int64_t row0, const qlra_qmat_t* h,
                  const qlra_qmat_t* w, qlra_qmat_t* x);

/* The whole QB stage, qb_stage_with_psi (sketching.cpp:169-194): the
 * rangefinder on Y (`method`, `rangefinder_seed`, `cfg` as in qlra_pseudo_qr /
 * qlra_pseudo_svd; NULL cfg = defaults) into H, then X as qlra_qb_solve.  With
 * pseudo-QR on one rank the solve starts inside the rangefinder: X = C^{-1} X0
 * where H = Q0 C and X0 = (Psi Q0)^+ W runs on a second stream; results agree
 * with the two separate calls to rounding.  syncs. */
int qlra_qb_stage(qlra_ctx_t* ctx, const qlra_spec_t* psi, int64_t row0, const qlra_qmat_t* y,
                  const qlra_qmat_t* w, int method, uint64_t rangefinder_seed,
                  const qlra_pseudo_qr_config_t* cfg, qlra_qmat_t* h, qlra_qmat_t* x,
                  qlra_rangefinder_report_t* report);
/* qb_stage_with_psi (sketching.hpp:104-107, sketching.cpp:169-188) with an
 * explicitly supplied Psi: `psi` is this rank's column slice
 * Psi(:, row0 : row0 + y->rows) in device memory (l x y->rows); the
 * reference's tests inject structured ones this way (test_sketching.cpp:
 * 170-183).  Rangefinder on Y, P = Psi H (all-reduced), X = P \ W.  syncs. */
int qlra_qb_stage_with_psi(qlra_ctx_t* ctx, const qlra_qmat_t* psi, const qlra_qmat_t* y,
                           const qlra_qmat_t* w, int method, uint64_t rangefinder_seed,
                           const qlra_pseudo_qr_config_t* cfg, qlra_qmat_t* h, qlra_qmat_t* x,
                           qlra_rangefinder_report_t* report);

/* one_pass_approx through the QB stage (sketching.cpp:250-263 -> make_sketch
 * :141-154 + qb_stage :169-194) on a device-resident row shard `a` (global
 * rows row0 ..): y (a->rows x s) and w (l x n) receive the sketch (zeroed
 * here; W all-reduced across ranks), h the rangefinder basis, x the core
 * solve.  Equivalent to qlra_sketch_update_rows + qlra_sketch_allreduce +
 * qlra_qb_stage, in one call. */
int qlra_one_pass_qb(qlra_ctx_t* ctx, const qlra_qmat_t* a, int64_t row0, const qlra_spec_t* omega,
                     const qlra_spec_t* psi, int method, uint64_t rangefinder_seed,
                     const qlra_pseudo_qr_config_t* cfg, qlra_qmat_t* y, qlra_qmat_t* w, qlra_qmat_t* h,
                     qlra_qmat_t* x, qlra_rangefinder_report_t* rep);

/* ------------------------------------------------ host-side one-pass --- */
/* one_pass_approx through the QB stage (sketching.cpp:250-263) for a host
 * resident row shard of A (pinned memory overlaps best): the sketch streams A
 * through the overlapped H2D + fused-sketch pipeline (block_rows as in
 * sketch_from_source, 0 = automatic), W is all-reduced, the rangefinder
 * (`method` = QLRA_PSEUDO_QR / QLRA_PSEUDO_SVD, `rangefinder_seed` for the
 * latter, `cfg` may be NULL) forms H, and H is copied back on a side stream
 * while the core solve computes X.  h_host (rows x s) and x_host (s x n) are
 * host views.  Replaces the QB half of one_pass_approx
 * (proj/include/qlra/sketching.hpp:143, sketching.cpp:250-263).  syncs. */
int qlra_one_pass_qb_host(qlra_ctx_t* ctx, const qlra_qmat_t* a_host, int64_t row0,
                          const qlra_spec_t* omega, const qlra_spec_t* psi, int method,
                          uint64_t rangefinder_seed, const qlra_pseudo_qr_config_t* cfg,
                          int64_t block_rows, qlra_qmat_t* h_host, qlra_qmat_t* x_host,
                          qlra_rangefinder_report_t* report);

/* ------------------------------------------------ truncation (next) --- */
/* qsvd (factorizations.hpp:44, factorizations.cpp:166-295) of a replicated
 * A (m x n): u m x k, v n x k, k = min(m, n); sigma (host, k) nonincreasing;
 * phase convention of factorizations.cpp:273-293.  syncs. */
int qlra_qsvd(qlra_ctx_t* ctx, const qlra_qmat_t* a, qlra_qmat_t* u, double* sigma,
              qlra_qmat_t* v);
/* truncate_stage (sketching.hpp:128, sketching.cpp:196-211): QSVD of X
 * (s x n), keep the leading r triples, h_out = H U_r (H row-sharded),
 * sigma (host, r), v = V_r (n x r).  syncs. */
int qlra_truncate_stage(qlra_ctx_t* ctx, const qlra_qmat_t* h, const qlra_qmat_t* x, int64_t r,
                        qlra_qmat_t* h_out, double* sigma, qlra_qmat_t* v);
/* ||A - H diag(sigma) V^*||_F and ||A||_F: the relative_error diagnostic of
 * one_pass_approx (sketching.cpp:272-273; analysis.cpp:75-79).  syncs. */
int qlra_approx_residual_fro(qlra_ctx_t* ctx, const qlra_qmat_t* a, const qlra_qmat_t* h,
                             const double* sigma, const qlra_qmat_t* v, double* res_fro,
                             double* a_fro);

/* ---------------------------------------------------------- residual --- */
/* ||A - H X||_F and ||A||_F (sketching.cpp:270-271; analysis.cpp:75-79) over
 * row-sharded A and H: a fused GEMM-subtract-square-reduce (second read of A,
 * diagnostic only); syncs. */
int qlra_residual_fro(qlra_ctx_t* ctx, const qlra_qmat_t* a, const qlra_qmat_t* h,
                      const qlra_qmat_t* x, double* res_fro, double* a_fro);

/* ------------------------------------------------ checkpoint I/O (next) --- */
/* QMAT1 / QSKT1 files byte-compatible with the reference (io.hpp:13-33,
 * io.cpp:77-145).  Device matrices are dense-packed on write.  All sync. */
int qlra_write_qmat(qlra_ctx_t* ctx, const char* path, const qlra_qmat_t* m);
int qlra_qmat_file_shape(const char* path, int64_t* rows, int64_t* cols);
int qlra_read_qmat(qlra_ctx_t* ctx, const char* path, qlra_qmat_t* m);
int qlra_write_sketch(qlra_ctx_t* ctx, const char* path, const qlra_spec_t* omega,
                      const qlra_spec_t* psi, int64_t r, int64_t s, int64_t l,
                      const qlra_qmat_t* y, const qlra_qmat_t* w);
/* Shapes of the Y and W embedded in a QSKT1 file (dims = y rows, y cols,
 * w rows, w cols) from their own QMAT1 headers, checked as read_sketch does
 * (io.cpp:130-145: y.cols == s and w.rows == l, else QLRA_ERR_IO) and against
 * the file length; no device work, no context. */
int qlra_sketch_file_dims(const char* path, int64_t* dims);
/* header of a QSKT1 file: both specs and r, s, l (rsl[3]) */
int qlra_sketch_file_header(const char* path, qlra_spec_t* omega, qlra_spec_t* psi, int64_t* rsl);
int qlra_read_sketch(qlra_ctx_t* ctx, const char* path, qlra_qmat_t* y, qlra_qmat_t* w);
/* sketch_from_source over a QMAT1 file (QmatFileSource, io.cpp:213-239):
 * blocks of block_rows rows are read into pinned buffers and sketched with
 * H2D overlap; y (m x s) and w (l x n) accumulate. */
int qlra_sketch_from_qmat_file(qlra_ctx_t* ctx, const char* path, const qlra_spec_t* omega,
                               const qlra_spec_t* psi, qlra_qmat_t* y, qlra_qmat_t* w,
                               int64_t block_rows);

/* ---------------------------------------------------------- diagnostics --- */
/* Measured FP64 throughput of this GPU: mode 0 = DFMA, 1 = DMMA (m8n8k4),
 * 2 = half the warps DMMA and half DFMA (pipe-sharing probe: on B200 it lands
 * between the two, 35.0 TF/s, so the FP64 CUDA-core and tensor paths share one
 * pipe).  Runs ~`ms` milliseconds; syncs. */
int qlra_measure_fp64_peak(qlra_ctx_t* ctx, int mode, double ms, double* tflops);
/* Name of the kernel variant the sketch uses for the given shape. */
const char* qlra_sketch_kernel_name(void);

#ifdef __cplusplus
}
#endif

#endif /* QLRA_CUDA_H */
