// facade_demo.cpp -- the reference's one-pass flow (sketching.cpp:250-275,
// through the QB stage) written against include/qlra_gpu.hpp, the C++ facade
// of the B200 C-ABI.  Prints "rel_error=<..> kappa=<..>" for the harness.
#include <cmath>
#include <cstdio>
#include <vector>

#include "qlra_gpu.hpp"

int main() {
  using namespace qlra::gpu;
  Context ctx(0);
  // A = G1 * G2 (rank 12) + 1e-4 noise (kappa(Y) ~ 1e4, inside pseudo-QR's
  // kappa < 1e8 domain), generated on the host as plain planes
  const Index m = 600, n = 400, k = 12;
  std::vector<double> g1(4 * m * k), g2(4 * k * n), a(4 * m * n);
  unsigned long long z = 12345;
  auto rnd = [&] { z = z * 6364136223846793005ull + 1442695040888963407ull; return (double)(z >> 11) * 0x1.0p-53 - 0.5; };
  for (auto& v : g1) v = rnd();
  for (auto& v : g2) v = rnd();
  // quaternion product into a (planes w,x,y,z), reference table quaternion.hpp:33-38
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < n; ++j) {
      double c[4] = {0, 0, 0, 0};
      for (Index t = 0; t < k; ++t) {
        const double* p = &g1[0];
        const double aw = p[0 * m * k + i * k + t], ax = p[1 * m * k + i * k + t],
                     ay = p[2 * m * k + i * k + t], az = p[3 * m * k + i * k + t];
        const double* q = &g2[0];
        const double bw = q[0 * k * n + t * n + j], bx = q[1 * k * n + t * n + j],
                     by = q[2 * k * n + t * n + j], bz = q[3 * k * n + t * n + j];
        c[0] += aw * bw - ax * bx - ay * by - az * bz;
        c[1] += aw * bx + ax * bw + ay * bz - az * by;
        c[2] += aw * by - ax * bz + ay * bw + az * bx;
        c[3] += aw * bz + ax * by - ay * bx + az * bw;
      }
      for (int p = 0; p < 4; ++p) a[p * m * n + i * n + j] = c[p] + 1e-4 * rnd();
    }
  HostQView ah{{&a[0], &a[m * n], &a[2 * m * n], &a[3 * m * n]}, m, n, n};
  DeviceQMatrix ad = DeviceQMatrix::upload(ah);
  const Index r = 12, s = 17, l = 34;
  SketchState st = make_sketch(ctx, ad, r, s, l, 1, 2);
  SketchState st2 = sketch_from_host(ctx, ah, r, s, l, 1, 2);  // streaming form
  QbResult qb = qb_stage(ctx, st, RangefinderMethod::kPseudoQr);
  QbResult qb2 = qb_stage(ctx, st2, RangefinderMethod::kPseudoSvd);
  auto [res, an] = qb_residual(ctx, ad, qb);
  auto [res2, an2] = qb_residual(ctx, ad, qb2);
  // host in / host out in one call: same seeds as make_sketch above
  HostQb hq = one_pass_qb_host(ctx, ah, r, s, l, RangefinderMethod::kPseudoQr, 1, 2);
  QbResult qb3;
  qb3.h = DeviceQMatrix::upload(HostQView{{&hq.h[0], &hq.h[m * s], &hq.h[2 * m * s], &hq.h[3 * m * s]}, m, s, s});
  qb3.x = DeviceQMatrix::upload(HostQView{{&hq.x[0], &hq.x[s * n], &hq.x[2 * s * n], &hq.x[3 * s * n]}, s, n, n});
  auto [res3, an3] = qb_residual(ctx, ad, qb3);
  bool threw = false;
  try {
    DeviceQMatrix zero(3, 3), rhs(3, 1);
    solve_quaternion_linear(ctx, zero, rhs);
  } catch (const SingularMatrixError& e) {
    threw = e.estimated_condition > 1e14;
  }
  std::printf("rel_error=%.3e rel_error_svd=%.3e rel_error_host=%.3e kappa=%.4f singular_threw=%d\n", res / an,
              res2 / an2, res3 / an3, qb.report.kappa_after, (int)threw);
  const bool host_ok = std::fabs(res3 / an3 - res / an) <= 1e-8 * (res / an);
  return (res / an < 1e-2 && res2 / an2 < 1e-2 && threw && host_ok) ? 0 : 1;
}
