// qlra_gpu.hpp -- header-only C++17 facade over the qlra_cuda.h C-ABI with the
// reference API's names, argument meanings and exception types
// (proj/include/qlra/{sketching,rangefinders,complex_bridge,factorizations,
// errors}.hpp).  A reference user switches `qlra::make_sketch(a, ...)` to
// `qlra::gpu::make_sketch(ctx, a, ...)`; see INTEGRATION.md.
//
// Errors are the reference's own types: `qlra::ShapeError`,
// `qlra::RankError`, `qlra::SingularMatrixError` ... (errors.hpp:9-43).  When
// the reference's headers are on the include path, its errors.hpp is used
// as-is; otherwise an identical definition under the same include guard, so a
// translation unit may include either first.  A reference caller's
// `catch (const qlra::RankError&)` therefore catches the GPU path's errors.
// Device failures (CUDA/NCCL) throw qlra::gpu::DeviceError, a qlra::Error.
//
// Matrices live on the device (DeviceQMatrix: four row-major FP64 planes, the
// reference QMatrix layout, qmatrix.hpp:14-19).  HostQView wraps the planes of
// a host matrix (e.g. a reference QMatrix's plane(kW).data() ...) for upload
// or for the streaming sketch; pageable memory is staged through pinned
// buffers by the library, pinned memory is copied directly.
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdint>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "qlra_cuda.h"

#if defined(__has_include)
#if __has_include(<qlra/errors.hpp>)
#include <qlra/errors.hpp>
#endif
#endif

#ifndef QLRA_ERRORS_HPP
#define QLRA_ERRORS_HPP
// Identical to proj/include/qlra/errors.hpp:9-43 (same names, bases,
// members and message format), under the same include guard.
namespace qlra {
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ShapeError : Error {
  using Error::Error;
};
struct ParameterError : Error {
  using Error::Error;
};
struct SingularMatrixError : Error {
  double estimated_condition;
  SingularMatrixError(const std::string& msg, double cond)
      : Error(msg + " (estimated condition " + std::to_string(cond) + ")"), estimated_condition(cond) {}
};
struct RankError : Error {
  using Error::Error;
};
struct PreconditionError : Error {
  using Error::Error;
};
struct IoError : Error {
  using Error::Error;
};
}  // namespace qlra
#endif

namespace qlra {
namespace gpu {

using Index = std::int64_t;

using qlra::Error;
using qlra::IoError;
using qlra::ParameterError;
using qlra::PreconditionError;
using qlra::RankError;
using qlra::ShapeError;
using qlra::SingularMatrixError;
// CUDA / NCCL failures (no reference counterpart)
struct DeviceError : qlra::Error {
  using qlra::Error::Error;
};

enum class TestMatrixKind { kGaussian = QLRA_GAUSSIAN, kRademacher = QLRA_RADEMACHER,
                            kSparseGaussian = QLRA_SPARSE_GAUSSIAN,
                            kSparseRademacher = QLRA_SPARSE_RADEMACHER };
enum class RangefinderMethod { kPseudoQr = QLRA_PSEUDO_QR, kPseudoSvd = QLRA_PSEUDO_SVD };
constexpr std::uint64_t kDefaultRangefinderSeed = 0x9E3779B9;  // rangefinders.hpp:29

// ---------------------------------------------------------------- context ---
class Context {
 public:
  explicit Context(int device = 0, int rank = 0, int nranks = 1, const void* nccl_id = nullptr) {
    if (qlra_ctx_create(&h_, device, rank, nranks, nccl_id) != QLRA_OK)
      throw DeviceError("qlra_ctx_create failed");
  }
  ~Context() { qlra_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  qlra_ctx_t* get() const { return h_; }
  cudaStream_t stream() const { return static_cast<cudaStream_t>(qlra_ctx_stream(h_)); }
  void synchronize() const { check(qlra_ctx_synchronize(h_)); }

  void check(int rc) const {
    if (rc == QLRA_OK) return;
    double cond = 0.0;
    const std::string msg = qlra_last_error(h_, &cond);
    switch (rc) {
      case QLRA_ERR_SHAPE: throw ShapeError(msg);
      case QLRA_ERR_PARAMETER: throw ParameterError(msg);
      case QLRA_ERR_SINGULAR: throw SingularMatrixError(msg, cond);
      case QLRA_ERR_RANK: throw RankError(msg);
      case QLRA_ERR_PRECONDITION: throw PreconditionError(msg);
      case QLRA_ERR_IO: throw IoError(msg);
      default: throw DeviceError(msg);
    }
  }

 private:
  qlra_ctx_t* h_ = nullptr;
};

// ------------------------------------------------------------- matrices ---
struct HostQView {
  const double* p[4];
  Index rows, cols, ld;
};

// A host quaternion matrix: four row-major planes back to back (the
// reference QMatrix's storage, qmatrix.hpp:14-19, in one vector).
struct HostQMatrix {
  Index rows = 0, cols = 0;
  std::vector<double> data;  // 4 * rows * cols
  HostQMatrix() = default;
  HostQMatrix(Index r, Index c) : rows(r), cols(c), data((size_t)(4 * r * c), 0.0) {}
  double* plane(int p) { return data.data() + (size_t)p * rows * cols; }
  const double* plane(int p) const { return data.data() + (size_t)p * rows * cols; }
  HostQView view() const { return HostQView{{plane(0), plane(1), plane(2), plane(3)}, rows, cols, cols}; }
};

// Device matrix.  Allocation, zero-fill, upload and download are ordered
// against the library's work: they complete before returning, and download()
// first waits for all work queued on the device (the library runs on its own
// non-blocking stream, which the legacy default stream does not order).
class DeviceQMatrix {
 public:
  DeviceQMatrix() = default;
  DeviceQMatrix(Index rows, Index cols) : rows_(rows), cols_(cols) {
    const size_t bytes = sizeof(double) * 4 * (size_t)(rows * cols);
    if (bytes) {
      if (cudaMalloc(&base_, bytes) != cudaSuccess) throw DeviceError("cudaMalloc failed");
      if (cudaMemset(base_, 0, bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
        throw DeviceError("cudaMemset failed");
    }
  }
  ~DeviceQMatrix() {
    if (base_) cudaFree(base_);
  }
  DeviceQMatrix(DeviceQMatrix&& o) noexcept { *this = std::move(o); }
  DeviceQMatrix& operator=(DeviceQMatrix&& o) noexcept {
    std::swap(base_, o.base_);
    std::swap(rows_, o.rows_);
    std::swap(cols_, o.cols_);
    return *this;
  }
  DeviceQMatrix(const DeviceQMatrix&) = delete;
  DeviceQMatrix& operator=(const DeviceQMatrix&) = delete;

  static DeviceQMatrix upload(const HostQView& h) {
    DeviceQMatrix d(h.rows, h.cols);
    for (int p = 0; p < 4 && h.rows * h.cols > 0; ++p)
      if (cudaMemcpy2D(d.plane(p), sizeof(double) * d.cols_, h.p[p], sizeof(double) * h.ld,
                       sizeof(double) * h.cols, (size_t)h.rows, cudaMemcpyHostToDevice) != cudaSuccess)
        throw DeviceError("upload failed");
    if (cudaDeviceSynchronize() != cudaSuccess) throw DeviceError("upload failed");
    return d;
  }
  // planes w, x, y, z concatenated, each row-major rows x cols
  std::vector<double> download() const {
    std::vector<double> out(4 * (size_t)(rows_ * cols_));
    if (cudaDeviceSynchronize() != cudaSuccess) throw DeviceError("download: device failure");
    if (!out.empty() &&
        cudaMemcpy(out.data(), base_, out.size() * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
      throw DeviceError("download failed");
    return out;
  }
  HostQMatrix to_host() const {
    HostQMatrix h;
    h.rows = rows_;
    h.cols = cols_;
    h.data = download();
    return h;
  }
  double* plane(int p) const { return base_ + (size_t)p * rows_ * cols_; }
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  qlra_qmat_t view() const {
    qlra_qmat_t v;
    for (int p = 0; p < 4; ++p) v.p[p] = plane(p);
    v.rows = rows_;
    v.cols = cols_;
    v.ld = cols_;
    return v;
  }
  // rows [r0, r0 + nr) as a view
  qlra_qmat_t rows_view(Index r0, Index nr) const {
    qlra_qmat_t v = view();
    for (int p = 0; p < 4; ++p) v.p[p] += r0 * cols_;
    v.rows = nr;
    return v;
  }

 private:
  double* base_ = nullptr;
  Index rows_ = 0, cols_ = 0;
};

inline qlra_qmat_t host_qmat(const HostQView& h) {
  qlra_qmat_t v;
  for (int p = 0; p < 4; ++p) v.p[p] = const_cast<double*>(h.p[p]);
  v.rows = h.rows;
  v.cols = h.cols;
  v.ld = h.ld;
  return v;
}

// C = op(A) op(B) (qmat_mul, qmatrix.cpp:165-197, with the adjoint flags)
inline DeviceQMatrix qmat_mul(Context& ctx, const DeviceQMatrix& a, const DeviceQMatrix& b, bool adj_a = false,
                              bool adj_b = false) {
  DeviceQMatrix c(adj_a ? a.cols() : a.rows(), adj_b ? b.rows() : b.cols());
  qlra_qmat_t av = a.view(), bv = b.view(), cv = c.view();
  ctx.check(qlra_qmat_mul(ctx.get(), adj_a ? QLRA_OP_C : QLRA_OP_N, adj_b ? QLRA_OP_C : QLRA_OP_N, 1.0, &av, &bv,
                          0.0, &cv));
  return c;
}

// ------------------------------------------------------------ sketching ---
struct TestMatrixSpec {  // sketching.hpp:22-28
  TestMatrixKind kind = TestMatrixKind::kGaussian;
  Index rows = 0, cols = 0;
  std::uint64_t seed = 0;
  double density = 1.0;
  qlra_spec_t c() const { return {static_cast<int32_t>(kind), rows, cols, seed, density}; }
};

inline DeviceQMatrix gen_test_matrix(Context& ctx, const TestMatrixSpec& spec) {  // sketching.hpp:30
  DeviceQMatrix out(spec.rows, spec.cols);
  const qlra_spec_t s = spec.c();
  qlra_qmat_t v = out.view();
  ctx.check(qlra_gen_test_matrix_block(ctx.get(), &s, 0, 0, &v));
  return out;
}

struct SketchState {  // sketching.hpp:38-47 (y = this rank's row shard)
  DeviceQMatrix y, w;
  TestMatrixSpec omega_spec, psi_spec;
  Index r = 0, s = 0, l = 0, row0 = 0;
  Index data_rows() const { return psi_spec.cols; }
  Index data_cols() const { return w.cols(); }
};

inline SketchState empty_sketch(Index m, Index n, Index r, Index s, Index l, std::uint64_t omega_seed,
                                std::uint64_t psi_seed,
                                TestMatrixKind kind = TestMatrixKind::kGaussian,
                                double density = 1.0, Index rows_local = -1, Index row0 = 0) {
  if (r < 1 || !(r <= s && s <= l && l <= std::min(m, n)))
    throw ParameterError("sketch sizes must satisfy 1 <= r <= s <= l <= min(m,n)");
  if (!(density > 0.0 && density <= 1.0)) throw ParameterError("test matrix: density must lie in (0,1]");
  SketchState st;
  st.y = DeviceQMatrix(rows_local < 0 ? m : rows_local, s);
  st.w = DeviceQMatrix(l, n);
  st.omega_spec = {kind, n, s, omega_seed, density};
  st.psi_spec = {kind, l, m, psi_seed, density};
  st.r = r;
  st.s = s;
  st.l = l;
  st.row0 = row0;
  return st;
}

// sketch_update_rows (sketching.hpp:63-66): rows [row0, row0 + block.rows())
// of A (or an additive update to them), block on the device.
inline void sketch_update_rows(Context& ctx, SketchState& st, Index row0, const DeviceQMatrix& block) {
  const Index lr0 = row0 - st.row0;
  if (block.cols() != st.w.cols()) throw ShapeError("sketch_update_rows: column count mismatch");
  if (lr0 < 0 || lr0 + block.rows() > st.y.rows()) throw ShapeError("sketch_update_rows: row range out of bounds");
  if (block.rows() == 0) return;
  qlra_qmat_t b = block.view(), y = st.y.rows_view(lr0, block.rows()), w = st.w.view();
  const qlra_spec_t om = st.omega_spec.c(), ps = st.psi_spec.c();
  ctx.check(qlra_sketch_update_rows(ctx.get(), &om, &ps, row0, &b, &y, &w));
}

// The same with the block in host memory (streamed H2D, overlapped).
inline void sketch_update_rows(Context& ctx, SketchState& st, Index row0, const HostQView& block,
                               Index block_rows = 0) {
  const Index lr0 = row0 - st.row0;
  if (block.cols != st.w.cols()) throw ShapeError("sketch_update_rows: column count mismatch");
  if (lr0 < 0 || lr0 + block.rows > st.y.rows()) throw ShapeError("sketch_update_rows: row range out of bounds");
  if (block.rows == 0) return;
  qlra_qmat_t b = host_qmat(block), y = st.y.rows_view(lr0, block.rows), w = st.w.view();
  const qlra_spec_t om = st.omega_spec.c(), ps = st.psi_spec.c();
  ctx.check(qlra_sketch_update_rows_host(ctx.get(), &om, &ps, row0, &b, &y, &w, block_rows));
}

// sketch_update (sketching.hpp:59-60): additive update A <- A + delta
// (full shape of this rank's rows).
inline void sketch_update(Context& ctx, SketchState& st, const DeviceQMatrix& delta) {
  if (delta.rows() != st.y.rows()) throw ShapeError("sketch_update: row count mismatch");
  sketch_update_rows(ctx, st, st.row0, delta);
}

// Sum W over the ranks (multi-GPU row shards; no-op on one rank).
inline void sketch_allreduce(Context& ctx, SketchState& st) {
  qlra_qmat_t w = st.w.view();
  ctx.check(qlra_sketch_allreduce(ctx.get(), &w));
}

// make_sketch (sketching.hpp:54-57); A on device.
inline SketchState make_sketch(Context& ctx, const DeviceQMatrix& a, Index r, Index s, Index l,
                               std::uint64_t omega_seed, std::uint64_t psi_seed,
                               TestMatrixKind kind = TestMatrixKind::kGaussian, double density = 1.0) {
  SketchState st = empty_sketch(a.rows(), a.cols(), r, s, l, omega_seed, psi_seed, kind, density);
  sketch_update_rows(ctx, st, 0, a);
  return st;
}

// make_sketch for a host-resident A (streamed row panels, H2D overlapped with
// the sketch; pinned memory copies directly, pageable memory is staged).
inline SketchState sketch_from_host(Context& ctx, const HostQView& a, Index r, Index s, Index l,
                                    std::uint64_t omega_seed, std::uint64_t psi_seed,
                                    TestMatrixKind kind = TestMatrixKind::kGaussian,
                                    double density = 1.0, Index block_rows = 0) {
  SketchState st = empty_sketch(a.rows, a.cols, r, s, l, omega_seed, psi_seed, kind, density);
  sketch_update_rows(ctx, st, 0, a, block_rows);
  return st;
}

// MatrixSource (sketching.hpp:67-74): the sketch builder is the only reader.
class MatrixSource {
 public:
  virtual ~MatrixSource() = default;
  virtual Index rows() const = 0;
  virtual Index cols() const = 0;
  virtual HostQMatrix read_rows(Index r0, Index r1) const = 0;
};

// sketch_from_source (sketching.hpp:76-79, sketching.cpp:156-167): blocks of
// block_rows rows are read in row order, each folded in once.
inline SketchState sketch_from_source(Context& ctx, const MatrixSource& source, Index r, Index s, Index l,
                                      std::uint64_t omega_seed, std::uint64_t psi_seed,
                                      TestMatrixKind kind = TestMatrixKind::kGaussian, double density = 1.0,
                                      Index block_rows = 256) {
  if (block_rows < 1) throw ParameterError("sketch_from_source: block_rows must be >= 1");
  SketchState st = empty_sketch(source.rows(), source.cols(), r, s, l, omega_seed, psi_seed, kind, density);
  for (Index r0 = 0; r0 < source.rows(); r0 += block_rows) {
    const Index r1 = std::min(source.rows(), r0 + block_rows);
    const HostQMatrix blk = source.read_rows(r0, r1);
    if (blk.rows != r1 - r0 || blk.cols != source.cols())
      throw ShapeError("sketch_from_source: read_rows returned a block of the wrong shape");
    sketch_update_rows(ctx, st, r0, blk.view(), blk.rows);
  }
  return st;
}

// ----------------------------------------------------------- rangefinders ---
struct PseudoQrConfig {  // rangefinders.hpp:23-27
  int max_correction_steps = 3;
  int power_iters_for_epsilon = 3;
  double delta_budget = 1.2;
  qlra_pseudo_qr_config_t c() const { return {max_correction_steps, power_iters_for_epsilon, delta_budget}; }
};

struct RangefinderReport {  // rangefinders.hpp:14-21
  DeviceQMatrix h;
  double kappa_before = 0.0, kappa_after = 0.0;
  int correction_steps_used = 0;
  RangefinderMethod method = RangefinderMethod::kPseudoQr;
};

inline RangefinderReport pseudo_qr(Context& ctx, const DeviceQMatrix& y, const PseudoQrConfig& cfg = {}) {
  RangefinderReport rep;
  rep.h = DeviceQMatrix(y.rows(), y.cols());
  const qlra_pseudo_qr_config_t c = cfg.c();
  qlra_rangefinder_report_t r{};
  qlra_qmat_t yv = y.view(), hv = rep.h.view();
  ctx.check(qlra_pseudo_qr(ctx.get(), &yv, &c, &hv, &r));
  rep.kappa_before = r.kappa_before;
  rep.kappa_after = r.kappa_after;
  rep.correction_steps_used = r.correction_steps_used;
  return rep;
}

inline RangefinderReport pseudo_svd(Context& ctx, const DeviceQMatrix& y,
                                    std::uint64_t seed = kDefaultRangefinderSeed) {
  RangefinderReport rep;
  rep.method = RangefinderMethod::kPseudoSvd;
  rep.h = DeviceQMatrix(y.rows(), y.cols());
  qlra_rangefinder_report_t r{};
  qlra_qmat_t yv = y.view(), hv = rep.h.view();
  ctx.check(qlra_pseudo_svd(ctx.get(), &yv, seed, &hv, &r));
  rep.kappa_before = r.kappa_before;
  rep.kappa_after = r.kappa_after;
  return rep;
}

// orthonormal_range (rangefinders.hpp:61): pseudo-SVD basis, rows >= cols.
inline DeviceQMatrix orthonormal_range(Context& ctx, const DeviceQMatrix& y,
                                       std::uint64_t seed = kDefaultRangefinderSeed) {
  DeviceQMatrix h(y.rows(), y.cols());
  qlra_qmat_t yv = y.view(), hv = h.view();
  ctx.check(qlra_orthonormal_range(ctx.get(), &yv, seed, &hv));
  return h;
}

inline double estimate_epsilon(Context& ctx, const DeviceQMatrix& h, int power_iters = 3) {
  double e = 0.0;
  qlra_qmat_t v = h.view();
  ctx.check(qlra_estimate_epsilon(ctx.get(), &v, power_iters, &e));
  return e;
}

inline DeviceQMatrix correction_step(Context& ctx, const DeviceQMatrix& h, double epsilon) {
  DeviceQMatrix out(h.rows(), h.cols());
  qlra_qmat_t v = h.view(), o = out.view();
  ctx.check(qlra_correction_step(ctx.get(), &v, epsilon, &o));
  return out;
}

inline double condition_number(Context& ctx, const DeviceQMatrix& a) {
  double k = 0.0;
  qlra_qmat_t v = a.view();
  ctx.check(qlra_condition_number(ctx.get(), &v, &k));
  return k;
}

inline DeviceQMatrix solve_quaternion_linear(Context& ctx, const DeviceQMatrix& a,
                                             const DeviceQMatrix& b) {
  DeviceQMatrix x(a.cols(), b.cols());
  qlra_qmat_t av = a.view(), bv = b.view(), xv = x.view();
  ctx.check(qlra_solve_quaternion_linear(ctx.get(), &av, &bv, &xv));
  return x;
}

// --------------------------------------------------------------- QB stage ---
struct StageTimes {  // sketching.hpp:81-86
  double sketch_s = 0.0, rangefinder_s = 0.0, solve_s = 0.0, truncate_s = 0.0;
};

struct QbResult {  // sketching.hpp:88-94
  DeviceQMatrix h, x;
  RangefinderReport report;
  double rangefinder_s = 0.0, solve_s = 0.0;
};

namespace detail {
inline double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
inline void fill_report(RangefinderReport& r, const qlra_rangefinder_report_t& c, RangefinderMethod m) {
  r.kappa_before = c.kappa_before;
  r.kappa_after = c.kappa_after;
  r.correction_steps_used = m == RangefinderMethod::kPseudoQr ? c.correction_steps_used : 0;
  r.method = m;
}
}  // namespace detail

// qb_stage (sketching.hpp:98-101): one call -- with pseudo-QR the core solve
// starts inside the rangefinder; Psi is regenerated from its spec.  The
// stage times: `rangefinder_s` holds the whole stage (the two overlap).
inline QbResult qb_stage(Context& ctx, const SketchState& st, RangefinderMethod method,
                         std::uint64_t rangefinder_seed = kDefaultRangefinderSeed,
                         const PseudoQrConfig& qr_cfg = {}) {
  const auto t0 = std::chrono::steady_clock::now();
  QbResult out;
  out.h = DeviceQMatrix(st.y.rows(), st.y.cols());
  out.x = DeviceQMatrix(st.s, st.w.cols());
  const qlra_spec_t ps = st.psi_spec.c();
  const qlra_pseudo_qr_config_t c = qr_cfg.c();
  qlra_rangefinder_report_t r{};
  qlra_qmat_t yv = st.y.view(), wv = st.w.view(), hv = out.h.view(), xv = out.x.view();
  ctx.check(qlra_qb_stage(ctx.get(), &ps, st.row0, &yv, &wv, (int)method, rangefinder_seed, &c, &hv, &xv, &r));
  ctx.synchronize();
  detail::fill_report(out.report, r, method);
  out.rangefinder_s = detail::seconds_since(t0);
  return out;
}

// The same as two timed calls (rangefinder, then solve), as the reference
// reports its StageTimes (sketching.cpp:176-186).
inline QbResult qb_stage_timed(Context& ctx, const SketchState& st, RangefinderMethod method,
                               std::uint64_t rangefinder_seed = kDefaultRangefinderSeed,
                               const PseudoQrConfig& qr_cfg = {}) {
  QbResult out;
  auto t0 = std::chrono::steady_clock::now();
  out.report = method == RangefinderMethod::kPseudoQr ? pseudo_qr(ctx, st.y, qr_cfg)
                                                      : pseudo_svd(ctx, st.y, rangefinder_seed);
  ctx.synchronize();
  out.rangefinder_s = detail::seconds_since(t0);
  t0 = std::chrono::steady_clock::now();
  out.h = std::move(out.report.h);
  out.x = DeviceQMatrix(st.s, st.w.cols());
  const qlra_spec_t ps = st.psi_spec.c();
  qlra_qmat_t hv = out.h.view(), wv = st.w.view(), xv = out.x.view();
  ctx.check(qlra_qb_solve(ctx.get(), &ps, st.row0, &hv, &wv, &xv));
  ctx.synchronize();
  out.solve_s = detail::seconds_since(t0);
  return out;
}

// qb_stage_with_psi (sketching.hpp:103-107): an explicit Psi (device, the
// l x y.rows() column slice of this rank's rows).
inline QbResult qb_stage_with_psi(Context& ctx, const SketchState& st, const DeviceQMatrix& psi,
                                  RangefinderMethod method,
                                  std::uint64_t rangefinder_seed = kDefaultRangefinderSeed,
                                  const PseudoQrConfig& qr_cfg = {}) {
  const auto t0 = std::chrono::steady_clock::now();
  QbResult out;
  out.h = DeviceQMatrix(st.y.rows(), st.y.cols());
  out.x = DeviceQMatrix(st.y.cols(), st.w.cols());
  const qlra_pseudo_qr_config_t c = qr_cfg.c();
  qlra_rangefinder_report_t r{};
  qlra_qmat_t pv = psi.view(), yv = st.y.view(), wv = st.w.view(), hv = out.h.view(), xv = out.x.view();
  ctx.check(qlra_qb_stage_with_psi(ctx.get(), &pv, &yv, &wv, (int)method, rangefinder_seed, &c, &hv, &xv, &r));
  ctx.synchronize();
  detail::fill_report(out.report, r, method);
  out.rangefinder_s = detail::seconds_since(t0);
  return out;
}

// ||A - H X||_F and ||A||_F (sketching.cpp:270-271)
inline std::pair<double, double> qb_residual(Context& ctx, const DeviceQMatrix& a, const QbResult& qb) {
  double r = 0.0, n = 0.0;
  qlra_qmat_t av = a.view(), hv = qb.h.view(), xv = qb.x.view();
  ctx.check(qlra_residual_fro(ctx.get(), &av, &hv, &xv, &r, &n));
  return {r, n};
}

// ------------------------------------------------------------- truncation ---
struct ApproxDiagnostics {  // sketching.hpp:109-116
  double kappa_h = 0.0;
  double kappa_before = 0.0;
  int correction_steps = 0;
  std::optional<double> qb_residual;
  std::optional<double> relative_error;
  StageTimes times;
};

struct ApproxResult {  // sketching.hpp:118-123
  DeviceQMatrix h;            // m x r
  std::vector<double> sigma;  // length r, nonincreasing
  DeviceQMatrix v;            // n x r
  ApproxDiagnostics diagnostics;
};

// truncate_stage (sketching.hpp:128, sketching.cpp:196-211)
inline ApproxResult truncate_stage(Context& ctx, const DeviceQMatrix& h, const DeviceQMatrix& x, Index r) {
  if (h.cols() != x.rows()) throw ShapeError("truncate_stage: H and X do not conform");
  if (r < 1 || r > x.rows()) throw ParameterError("truncate_stage: need 1 <= r <= s");
  ApproxResult out;
  out.h = DeviceQMatrix(h.rows(), r);
  out.v = DeviceQMatrix(x.cols(), r);
  out.sigma.assign((size_t)r, 0.0);
  qlra_qmat_t hv = h.view(), xv = x.view(), ho = out.h.view(), vo = out.v.view();
  ctx.check(qlra_truncate_stage(ctx.get(), &hv, &xv, r, &ho, out.sigma.data(), &vo));
  return out;
}

// approx_reconstruct (sketching.hpp:125, sketching.cpp:213-218): H S V^*
inline DeviceQMatrix approx_reconstruct(Context& ctx, const ApproxResult& res) {
  const Index r = res.h.cols();
  HostQMatrix d(r, r);
  for (Index j = 0; j < r; ++j) d.plane(0)[j * r + j] = res.sigma[(size_t)j];
  const DeviceQMatrix dd = DeviceQMatrix::upload(d.view());
  const DeviceQMatrix hs = qmat_mul(ctx, res.h, dd);
  return qmat_mul(ctx, hs, res.v, false, true);
}

// ||A - H S V^*||_F and ||A||_F (relative_error's terms, analysis.cpp:75-79)
inline std::pair<double, double> approx_residual(Context& ctx, const DeviceQMatrix& a, const ApproxResult& res) {
  double r = 0.0, n = 0.0;
  qlra_qmat_t av = a.view(), hv = res.h.view(), vv = res.v.view();
  ctx.check(qlra_approx_residual_fro(ctx.get(), &av, &hv, res.sigma.data(), &vv, &r, &n));
  return {r, n};
}

// ---------------------------------------------------------------- one pass ---
struct OnePassOptions {  // sketching.hpp:130-141
  Index r = 0;
  Index s = -1;  // defaults to r + 5
  Index l = -1;  // defaults to 2 s
  RangefinderMethod rangefinder = RangefinderMethod::kPseudoQr;
  TestMatrixKind embedding = TestMatrixKind::kGaussian;
  double density = 1.0;
  std::uint64_t omega_seed = 1;
  std::uint64_t psi_seed = 2;
  std::uint64_t rangefinder_seed = kDefaultRangefinderSeed;
  PseudoQrConfig qr_cfg{};
};

namespace detail {
inline OnePassOptions resolve_defaults(OnePassOptions o) {  // sketching.cpp:222-227
  if (o.r < 1) throw ParameterError("one_pass_approx: rank must be >= 1");
  if (o.s < 0) o.s = o.r + 5;
  if (o.l < 0) o.l = 2 * o.s;
  return o;
}
inline ApproxResult run_pipeline(Context& ctx, const SketchState& st, const OnePassOptions& o) {
  QbResult qb = qb_stage_timed(ctx, st, o.rangefinder, o.rangefinder_seed, o.qr_cfg);
  const auto t0 = std::chrono::steady_clock::now();
  ApproxResult res = truncate_stage(ctx, qb.h, qb.x, o.r);
  ctx.synchronize();
  res.diagnostics.times.truncate_s = seconds_since(t0);
  res.diagnostics.times.rangefinder_s = qb.rangefinder_s;
  res.diagnostics.times.solve_s = qb.solve_s;
  res.diagnostics.kappa_h = qb.report.kappa_after;
  res.diagnostics.kappa_before = qb.report.kappa_before;
  res.diagnostics.correction_steps = qb.report.correction_steps_used;
  return res;
}
}  // namespace detail

// one_pass_approx(const SketchState&, opts) (sketching.hpp:144,
// sketching.cpp:244-248): QB stage + truncation; A is never touched.
inline ApproxResult one_pass_approx(Context& ctx, const SketchState& st, const OnePassOptions& opts) {
  const OnePassOptions o = detail::resolve_defaults(opts);
  if (o.r > st.s) throw ParameterError("one_pass_approx: rank exceeds sketch size s");
  return detail::run_pipeline(ctx, st, o);
}

// one_pass_approx(const QMatrix&, opts) (sketching.hpp:143,
// sketching.cpp:250-275), A on the device: sketch (one read of A), QB stage,
// truncation, and the diagnostics ||A - H X|| and ||A - H S V^*|| / ||A||
// (a second read of A).
inline ApproxResult one_pass_approx(Context& ctx, const DeviceQMatrix& a, const OnePassOptions& opts) {
  const OnePassOptions o = detail::resolve_defaults(opts);
  const auto t0 = std::chrono::steady_clock::now();
  const SketchState st = make_sketch(ctx, a, o.r, o.s, o.l, o.omega_seed, o.psi_seed, o.embedding, o.density);
  ctx.synchronize();
  const double t_sketch = detail::seconds_since(t0);
  QbResult qb = qb_stage_timed(ctx, st, o.rangefinder, o.rangefinder_seed, o.qr_cfg);
  const auto t1 = std::chrono::steady_clock::now();
  ApproxResult res = truncate_stage(ctx, qb.h, qb.x, o.r);
  ctx.synchronize();
  res.diagnostics.times.truncate_s = detail::seconds_since(t1);
  res.diagnostics.times.sketch_s = t_sketch;
  res.diagnostics.times.rangefinder_s = qb.rangefinder_s;
  res.diagnostics.times.solve_s = qb.solve_s;
  res.diagnostics.kappa_h = qb.report.kappa_after;
  res.diagnostics.kappa_before = qb.report.kappa_before;
  res.diagnostics.correction_steps = qb.report.correction_steps_used;
  const auto [qres, na] = qb_residual(ctx, a, qb);
  res.diagnostics.qb_residual = qres;
  const auto [diff, na2] = approx_residual(ctx, a, res);
  (void)na2;
  res.diagnostics.relative_error =
      na > 0.0 ? diff / na : (diff > 0.0 ? std::numeric_limits<double>::infinity() : 0.0);
  return res;
}

// one_pass_approx up to the QB stage (sketching.cpp:250-263) for a host-
// resident A, in one call: the sketch streams A (H2D overlapped), and H and
// X come back into the caller's host buffers (4 planes each; pinned memory
// overlaps best).  Seeds and s, l defaults as OnePassOptions
// (sketching.hpp:130-141, sketching.cpp:222-227: s = r + 5, l = 2 s).
struct HostQb {
  std::vector<double> h, x;  // 4 planes each: h rows x s, x s x n
  Index rows = 0, s = 0, n = 0;
  RangefinderReport report;
};
inline HostQb one_pass_qb_host(Context& ctx, const HostQView& a, Index r, Index s = -1, Index l = -1,
                               RangefinderMethod method = RangefinderMethod::kPseudoQr,
                               std::uint64_t omega_seed = 1, std::uint64_t psi_seed = 2,
                               std::uint64_t rangefinder_seed = kDefaultRangefinderSeed,
                               TestMatrixKind kind = TestMatrixKind::kGaussian, double density = 1.0,
                               const PseudoQrConfig& cfg = {}, Index block_rows = 0) {
  if (s < 0) s = r + 5;
  if (l < 0) l = 2 * s;
  HostQb out;
  out.rows = a.rows;
  out.s = s;
  out.n = a.cols;
  out.h.assign((size_t)(4 * a.rows * s), 0.0);
  out.x.assign((size_t)(4 * s * a.cols), 0.0);
  const qlra_spec_t om{(int32_t)kind, a.cols, s, omega_seed, density};
  const qlra_spec_t ps{(int32_t)kind, l, a.rows, psi_seed, density};
  const qlra_pseudo_qr_config_t c = cfg.c();
  qlra_qmat_t av = host_qmat(a), hv, xv;
  for (int p = 0; p < 4; ++p) {
    hv.p[p] = out.h.data() + (size_t)p * a.rows * s;
    xv.p[p] = out.x.data() + (size_t)p * s * a.cols;
  }
  hv.rows = a.rows; hv.cols = s; hv.ld = s;
  xv.rows = s; xv.cols = a.cols; xv.ld = a.cols;
  qlra_rangefinder_report_t rep{};
  ctx.check(qlra_one_pass_qb_host(ctx.get(), &av, 0, &om, &ps, (int)method, rangefinder_seed, &c, block_rows, &hv,
                                  &xv, &rep));
  detail::fill_report(out.report, rep, method);
  return out;
}

}  // namespace gpu
}  // namespace qlra
