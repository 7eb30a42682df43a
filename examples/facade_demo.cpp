// facade_demo.cpp -- the reference's one-pass flow (sketching.cpp:141-275:
// sketch, QB stage, truncation, diagnostics) written against
// include/qlra_gpu.hpp, the C++ facade of the B200 C-ABI, the way a caller of
// the reference would write it: the reference's exception types are caught
// (`qlra::RankError`, `qlra::SingularMatrixError`).  Prints one line of
// "key=value" results for the harness (tests/test_cpp_facade.py) and exits
// non-zero if any check fails.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "qlra_gpu.hpp"

using namespace qlra::gpu;

namespace {

// A = G1 * G2 (rank k) + 1e-4 noise, generated on the host as plain planes
HostQMatrix make_matrix(Index m, Index n, Index k, unsigned long long seed) {
  unsigned long long z = seed;
  auto rnd = [&] {
    z = z * 6364136223846793005ull + 1442695040888963407ull;
    return (double)(z >> 11) * 0x1.0p-53 - 0.5;
  };
  HostQMatrix g1(m, k), g2(k, n), a(m, n);
  for (auto& v : g1.data) v = rnd();
  for (auto& v : g2.data) v = rnd();
  // quaternion product, reference table quaternion.hpp:33-38
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < n; ++j) {
      double c[4] = {0, 0, 0, 0};
      for (Index t = 0; t < k; ++t) {
        const double aw = g1.plane(0)[i * k + t], ax = g1.plane(1)[i * k + t], ay = g1.plane(2)[i * k + t],
                     az = g1.plane(3)[i * k + t];
        const double bw = g2.plane(0)[t * n + j], bx = g2.plane(1)[t * n + j], by = g2.plane(2)[t * n + j],
                     bz = g2.plane(3)[t * n + j];
        c[0] += aw * bw - ax * bx - ay * by - az * bz;
        c[1] += aw * bx + ax * bw + ay * bz - az * by;
        c[2] += aw * by - ax * bz + ay * bw + az * bx;
        c[3] += aw * bz + ax * by - ay * bx + az * bw;
      }
      for (int p = 0; p < 4; ++p) a.plane(p)[i * n + j] = c[p] + 1e-4 * rnd();
    }
  return a;
}

// MatrixSource over a host matrix, counting the rows it hands out (the
// reference's CountingSource, test_sketching.cpp:133-146)
class CountingSource : public MatrixSource {
 public:
  explicit CountingSource(const HostQMatrix& a) : a_(a) {}
  Index rows() const override { return a_.rows; }
  Index cols() const override { return a_.cols; }
  HostQMatrix read_rows(Index r0, Index r1) const override {
    rows_read_ += r1 - r0;
    HostQMatrix b(r1 - r0, a_.cols);
    for (int p = 0; p < 4; ++p)
      std::memcpy(b.plane(p), a_.plane(p) + r0 * a_.cols, sizeof(double) * (size_t)((r1 - r0) * a_.cols));
    return b;
  }
  mutable Index rows_read_ = 0;

 private:
  const HostQMatrix& a_;
};

double rel(const std::vector<double>& a, const std::vector<double>& b) {
  double d = 0.0, n = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    d += (a[i] - b[i]) * (a[i] - b[i]);
    n += b[i] * b[i];
  }
  return n > 0 ? std::sqrt(d / n) : std::sqrt(d);
}

}  // namespace

int main() {
  Context ctx(0);
  const Index m = 600, n = 400, k = 12;
  const HostQMatrix a = make_matrix(m, n, k, 12345);
  const DeviceQMatrix ad = DeviceQMatrix::upload(a.view());
  const Index r = 12, s = 17, l = 34;
  bool ok = true;

  // 1. one_pass_approx(const QMatrix&, opts): sketch, QB, truncation, diagnostics
  OnePassOptions opts;
  opts.r = r;
  const ApproxResult res = one_pass_approx(ctx, ad, opts);
  const double rel_err = *res.diagnostics.relative_error;
  ok = ok && rel_err < 1e-2 && res.sigma.size() == (size_t)r && res.diagnostics.times.solve_s > 0.0;
  for (size_t i = 1; i < res.sigma.size(); ++i) ok = ok && res.sigma[i] <= res.sigma[i - 1];

  // 2. the same pipeline step by step: make_sketch, qb_stage, truncate_stage,
  //    approx_reconstruct
  SketchState st = make_sketch(ctx, ad, r, s, l, 1, 2);
  QbResult qb = qb_stage(ctx, st, RangefinderMethod::kPseudoQr);
  const auto [qres, an] = qb_residual(ctx, ad, qb);
  const ApproxResult tr = truncate_stage(ctx, qb.h, qb.x, r);
  const std::vector<double> rec = approx_reconstruct(ctx, tr).download();
  const double rec_err = rel(rec, a.data);
  ok = ok && std::fabs(rec_err - rel_err) <= 1e-8 * rel_err && std::fabs(qres - *res.diagnostics.qb_residual) <=
                                                                     1e-8 * qres;

  // 3. sketch_from_source: the source is read exactly once, row blocks in
  //    order, and matches the in-memory sketch
  CountingSource src(a);
  SketchState st2 = sketch_from_source(ctx, src, r, s, l, 1, 2, TestMatrixKind::kGaussian, 1.0, 64);
  ok = ok && src.rows_read_ == m && rel(st2.y.download(), st.y.download()) < 1e-13 &&
       rel(st2.w.download(), st.w.download()) < 1e-13;
  const ApproxResult res2 = one_pass_approx(ctx, st2, opts);  // from the sketch: A untouched
  ok = ok && !res2.diagnostics.qb_residual && std::fabs(res2.sigma[0] / res.sigma[0] - 1) < 1e-10;

  // 4. sketch_update: additive linearity, A + A sketches to 2 x
  SketchState st3 = make_sketch(ctx, ad, r, s, l, 1, 2);
  sketch_update(ctx, st3, ad);
  {
    const auto y1 = st.y.download(), y2 = st3.y.download();
    std::vector<double> y1x2(y1.size());
    for (size_t i = 0; i < y1.size(); ++i) y1x2[i] = 2.0 * y1[i];
    ok = ok && rel(y2, y1x2) < 1e-13;
  }

  // 5. qb_stage_with_psi with the regenerated Psi equals qb_stage
  TestMatrixSpec ps = st.psi_spec;
  const DeviceQMatrix psi = gen_test_matrix(ctx, ps);
  QbResult qbp = qb_stage_with_psi(ctx, st, psi, RangefinderMethod::kPseudoSvd);
  const auto [pres, pan] = qb_residual(ctx, ad, qbp);
  ok = ok && std::fabs(pres / pan - qres / an) <= 1e-8 * (qres / an);

  // 6. orthonormal_range: H^* H = I
  const DeviceQMatrix hq = orthonormal_range(ctx, st.y);
  const std::vector<double> g = qmat_mul(ctx, hq, hq, true, false).download();
  double defect = 0.0;
  for (Index i = 0; i < s; ++i)
    for (Index j = 0; j < s; ++j) defect += std::pow(g[i * s + j] - (i == j ? 1.0 : 0.0), 2);
  ok = ok && std::sqrt(defect) < 1e-12;

  // 7. host in / host out in one call (pageable std::vector planes: staged)
  HostQb hq_host = one_pass_qb_host(ctx, a.view(), r, s, l, RangefinderMethod::kPseudoQr, 1, 2);
  QbResult qb3;
  qb3.h = DeviceQMatrix::upload(
      HostQView{{&hq_host.h[0], &hq_host.h[m * s], &hq_host.h[2 * m * s], &hq_host.h[3 * m * s]}, m, s, s});
  qb3.x = DeviceQMatrix::upload(
      HostQView{{&hq_host.x[0], &hq_host.x[s * n], &hq_host.x[2 * s * n], &hq_host.x[3 * s * n]}, s, n, n});
  const auto [res3, an3] = qb_residual(ctx, ad, qb3);
  ok = ok && std::fabs(res3 / an3 - qres / an) <= 1e-8 * (qres / an);

  // 8. the reference's exception types reach a reference-style catch
  bool rank_caught = false, singular_caught = false, shape_caught = false;
  try {
    DeviceQMatrix zero(40, 6);
    pseudo_qr(ctx, zero);
  } catch (const qlra::RankError& e) {
    rank_caught = std::strstr(e.what(), "use pseudo_svd") != nullptr;
  }
  try {
    DeviceQMatrix zero(3, 3), rhs(3, 1);
    solve_quaternion_linear(ctx, zero, rhs);
  } catch (const qlra::SingularMatrixError& e) {
    singular_caught = e.estimated_condition > 1e14 && std::strstr(e.what(), "(estimated condition ") != nullptr;
  }
  try {
    truncate_stage(ctx, qb.h, qb.x, s + 1);
  } catch (const qlra::ParameterError&) {
    shape_caught = true;
  } catch (const qlra::Error&) {
  }
  ok = ok && rank_caught && singular_caught && shape_caught;

  std::printf("rel_error=%.3e qb_error=%.3e rec_error=%.3e kappa=%.4f sigma1=%.6e rows_read=%lld "
              "rank_caught=%d singular_caught=%d ok=%d\n",
              rel_err, qres / an, rec_err, res.diagnostics.kappa_h, res.sigma[0], (long long)src.rows_read_,
              (int)rank_caught, (int)singular_caught, (int)ok);
  return ok ? 0 : 1;
}
