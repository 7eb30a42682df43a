// qlra_gpu.hpp -- header-only C++17 facade over the qlra_cuda.h C-ABI with the
// reference API's names, argument meanings and exception types
// (proj/include/qlra/{sketching,rangefinders,complex_bridge,factorizations,
// errors}.hpp).  A reference user switches `qlra::make_sketch(a, ...)` to
// `qlra::gpu::make_sketch(ctx, a, ...)`; see INTEGRATION.md.
//
// Matrices live on the device (DeviceQMatrix: four row-major FP64 planes, the
// reference QMatrix layout, qmatrix.hpp:14-19).  HostQView wraps the planes of
// a host matrix (e.g. a reference QMatrix's plane(kW).data() ...) for upload
// or for the streaming sketch.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "qlra_cuda.h"

namespace qlra {
namespace gpu {

using Index = std::int64_t;

// ---------------------------------------------------------------- errors ---
// proj/include/qlra/errors.hpp:9-43
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
  SingularMatrixError(const std::string& m, double c) : Error(m), estimated_condition(c) {}
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
struct DeviceError : Error {
  using Error::Error;
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

class DeviceQMatrix {
 public:
  DeviceQMatrix() = default;
  DeviceQMatrix(Index rows, Index cols) : rows_(rows), cols_(cols) {
    const size_t bytes = sizeof(double) * 4 * (size_t)(rows * cols);
    if (bytes) {
      if (cudaMalloc(&base_, bytes) != cudaSuccess) throw DeviceError("cudaMalloc failed");
      cudaMemset(base_, 0, bytes);
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
    for (int p = 0; p < 4; ++p)
      cudaMemcpy2D(d.plane(p), sizeof(double) * d.cols_, h.p[p], sizeof(double) * h.ld,
                   sizeof(double) * h.cols, (size_t)h.rows, cudaMemcpyHostToDevice);
    return d;
  }
  // planes w, x, y, z concatenated, each row-major rows x cols
  std::vector<double> download() const {
    std::vector<double> out(4 * (size_t)(rows_ * cols_));
    if (!out.empty()) cudaMemcpy(out.data(), base_, out.size() * sizeof(double), cudaMemcpyDeviceToHost);
    return out;
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

 private:
  double* base_ = nullptr;
  Index rows_ = 0, cols_ = 0;
};

// ------------------------------------------------------------ sketching ---
struct TestMatrixSpec {  // sketching.hpp:22-28
  TestMatrixKind kind = TestMatrixKind::kGaussian;
  Index rows = 0, cols = 0;
  std::uint64_t seed = 0;
  double density = 1.0;
  qlra_spec_t c() const { return {static_cast<int32_t>(kind), rows, cols, seed, density}; }
};

struct SketchState {  // sketching.hpp:38-47 (y = this rank's row shard)
  DeviceQMatrix y, w;
  TestMatrixSpec omega_spec, psi_spec;
  Index r = 0, s = 0, l = 0, row0 = 0;
};

inline SketchState empty_sketch(Index m, Index n, Index r, Index s, Index l, std::uint64_t omega_seed,
                                std::uint64_t psi_seed,
                                TestMatrixKind kind = TestMatrixKind::kGaussian,
                                double density = 1.0, Index rows_local = -1, Index row0 = 0) {
  if (r < 1 || !(r <= s && s <= l && l <= std::min(m, n)))
    throw ParameterError("sketch sizes must satisfy 1 <= r <= s <= l <= min(m,n)");
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

inline void sketch_update_rows(Context& ctx, SketchState& st, Index row0, const DeviceQMatrix& block) {
  qlra_qmat_t b = block.view(), y = st.y.view(), w = st.w.view();
  const Index lr0 = row0 - st.row0;
  for (int p = 0; p < 4; ++p) y.p[p] += lr0 * y.ld;
  y.rows = block.rows();
  const qlra_spec_t om = st.omega_spec.c(), ps = st.psi_spec.c();
  ctx.check(qlra_sketch_update_rows(ctx.get(), &om, &ps, row0, &b, &y, &w));
}

// make_sketch (sketching.hpp:54-57); A on device.
inline SketchState make_sketch(Context& ctx, const DeviceQMatrix& a, Index r, Index s, Index l,
                               std::uint64_t omega_seed, std::uint64_t psi_seed,
                               TestMatrixKind kind = TestMatrixKind::kGaussian, double density = 1.0) {
  SketchState st = empty_sketch(a.rows(), a.cols(), r, s, l, omega_seed, psi_seed, kind, density);
  sketch_update_rows(ctx, st, 0, a);
  return st;
}

// sketch_from_source (sketching.hpp:76-79) for a host-resident source:
// streamed row panels, H2D overlapped with the sketch.
inline SketchState sketch_from_host(Context& ctx, const HostQView& a, Index r, Index s, Index l,
                                    std::uint64_t omega_seed, std::uint64_t psi_seed,
                                    TestMatrixKind kind = TestMatrixKind::kGaussian,
                                    double density = 1.0, Index block_rows = 0) {
  SketchState st = empty_sketch(a.rows, a.cols, r, s, l, omega_seed, psi_seed, kind, density);
  qlra_qmat_t hb;
  for (int p = 0; p < 4; ++p) hb.p[p] = const_cast<double*>(a.p[p]);
  hb.rows = a.rows;
  hb.cols = a.cols;
  hb.ld = a.ld;
  qlra_qmat_t y = st.y.view(), w = st.w.view();
  const qlra_spec_t om = st.omega_spec.c(), ps = st.psi_spec.c();
  ctx.check(qlra_sketch_update_rows_host(ctx.get(), &om, &ps, 0, &hb, &y, &w, block_rows));
  return st;
}

// ----------------------------------------------------------- rangefinders ---
struct PseudoQrConfig {  // rangefinders.hpp:23-27
  int max_correction_steps = 3;
  int power_iters_for_epsilon = 3;
  double delta_budget = 1.2;
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
  const qlra_pseudo_qr_config_t c{cfg.max_correction_steps, cfg.power_iters_for_epsilon, cfg.delta_budget};
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
struct QbResult {  // sketching.hpp:88-94
  DeviceQMatrix h, x;
  RangefinderReport report;
};

inline QbResult qb_stage(Context& ctx, const SketchState& st, RangefinderMethod method,
                         std::uint64_t rangefinder_seed = kDefaultRangefinderSeed,
                         const PseudoQrConfig& qr_cfg = {}) {
  QbResult out;
  out.report = method == RangefinderMethod::kPseudoQr ? pseudo_qr(ctx, st.y, qr_cfg)
                                                      : pseudo_svd(ctx, st.y, rangefinder_seed);
  out.h = std::move(out.report.h);
  out.x = DeviceQMatrix(st.s, st.w.cols());
  const qlra_spec_t ps = st.psi_spec.c();
  qlra_qmat_t hv = out.h.view(), wv = st.w.view(), xv = out.x.view();
  ctx.check(qlra_qb_solve(ctx.get(), &ps, st.row0, &hv, &wv, &xv));
  return out;
}

// ||A - H X||_F and ||A||_F (sketching.cpp:270-271)
inline std::pair<double, double> qb_residual(Context& ctx, const DeviceQMatrix& a, const QbResult& qb) {
  double r = 0.0, n = 0.0;
  qlra_qmat_t av = a.view(), hv = qb.h.view(), xv = qb.x.view();
  ctx.check(qlra_residual_fro(ctx.get(), &av, &hv, &xv, &r, &n));
  return {r, n};
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
  const qlra_pseudo_qr_config_t c{cfg.max_correction_steps, cfg.power_iters_for_epsilon, cfg.delta_budget};
  qlra_qmat_t av, hv, xv;
  for (int p = 0; p < 4; ++p) {
    av.p[p] = const_cast<double*>(a.p[p]);
    hv.p[p] = out.h.data() + (size_t)p * a.rows * s;
    xv.p[p] = out.x.data() + (size_t)p * s * a.cols;
  }
  av.rows = a.rows; av.cols = a.cols; av.ld = a.ld;
  hv.rows = a.rows; hv.cols = s; hv.ld = s;
  xv.rows = s; xv.cols = a.cols; xv.ld = a.cols;
  qlra_rangefinder_report_t rep{};
  ctx.check(qlra_one_pass_qb_host(ctx.get(), &av, 0, &om, &ps, (int)method, rangefinder_seed, &c, block_rows, &hv,
                                  &xv, &rep));
  out.report.kappa_before = rep.kappa_before;
  out.report.kappa_after = rep.kappa_after;
  out.report.correction_steps_used = rep.correction_steps_used;
  out.report.method = method;
  return out;
}

}  // namespace gpu
}  // namespace qlra
