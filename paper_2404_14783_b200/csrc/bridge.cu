// bridge.cu -- the complex representations of quaternion matrices on the
// device (proj/src/complex_bridge.cpp:11-61, proj/include/qlra/
// complex_bridge.hpp:11-30).  Writing Q = Q0 + Q1 j with Q0 = w + x i and
// Q1 = y + z i:
//
//   compact  Q_c = [Q0; -conj(Q1)]                 (2m x n)
//   full     chi = [Q0, Q1; -conj(Q1), conj(Q0)]   (2m x 2n)
//
// Complex matrices at the boundary (qlra_cmat_t) are column-major with
// interleaved (re, im) doubles and a leading dimension -- the layout of the
// reference's CMatrix (Eigen::MatrixXcd) -- so a caller's Eigen buffer maps
// onto them without repacking.  Elementwise kernels: HBM-bound, one pass.
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.cuh"

namespace qlra_dev {

namespace {

__device__ __forceinline__ double2 cget(const CView& c, int64_t i, int64_t j) {
  return reinterpret_cast<const double2*>(c.data)[i + j * c.ld];
}
__device__ __forceinline__ void cput(const CView& c, int64_t i, int64_t j, double2 v) {
  reinterpret_cast<double2*>(c.data)[i + j * c.ld] = v;
}

// to_compact (complex_bridge.cpp:11-20) and to_full (:22-35): one thread per
// quaternion entry
__global__ void k_to_complex(QView q, CView out, int full) {
  const int64_t m = q.rows, n = q.cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / m, i = e % m;  // i fastest: coalesced column-major writes
    const int64_t o = i * q.ld + j;
    const double w = q.p[0][o], x = q.p[1][o], y = q.p[2][o], z = q.p[3][o];
    cput(out, i, j, double2{w, x});
    cput(out, m + i, j, double2{-y, z});  // -conj(Q1) = -y + z i
    if (full) {
      cput(out, i, n + j, double2{y, z});       // Q1
      cput(out, m + i, n + j, double2{w, -x});  // conj(Q0)
    }
  }
}

// from_compact (complex_bridge.cpp:37-52): Q0 = z0, Q1 = -conj(z1)
__global__ void k_from_compact(CView z, QView out) {
  const int64_t m = out.rows, n = out.cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / m, i = e % m;
    const double2 z0 = cget(z, i, j), z1 = cget(z, m + i, j);
    const int64_t o = i * out.ld + j;
    out.p[0][o] = z0.x;
    out.p[1][o] = z0.y;
    out.p[2][o] = -z1.x;
    out.p[3][o] = z1.y;
  }
}

// j_mul_conj (complex_bridge.cpp:54-61): [top; bottom] -> [-conj(bottom); conj(top)]
__global__ void k_j_mul_conj(CView u, CView out) {
  const int64_t m = u.rows / 2, k = u.cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * k;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / m, i = e % m;
    const double2 t = cget(u, i, j), b = cget(u, m + i, j);
    cput(out, i, j, double2{-b.x, b.y});
    cput(out, m + i, j, double2{t.x, -t.y});
  }
}

// complex matrix <-> quaternion matrix of its complex subalgebra (w + x i,
// y = z = 0): the complex factorisations run on the quaternion kernels
__global__ void k_cmat_to_quat(CView c, QView out) {
  const int64_t m = out.rows, n = out.cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / m, i = e % m;
    const double2 v = cget(c, i, j);
    const int64_t o = i * out.ld + j;
    out.p[0][o] = v.x;
    out.p[1][o] = v.y;
    out.p[2][o] = 0.0;
    out.p[3][o] = 0.0;
  }
}
__global__ void k_quat_to_cmat(QView q, CView out) {
  const int64_t m = q.rows, n = q.cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / m, i = e % m;
    const int64_t o = i * q.ld + j;
    cput(out, i, j, double2{q.p[0][o], q.p[1][o]});
  }
}

unsigned grid_of(int64_t total) {
  int64_t b = (total + 255) / 256;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

}  // namespace

void to_complex(Ctx& ctx, const QView& q, const CView& out, bool full) {
  if (q.rows * q.cols == 0) return;
  k_to_complex<<<grid_of(q.rows * q.cols), 256, 0, ctx.stream>>>(q, out, full ? 1 : 0);
  QLRA_LAUNCH_CHECK();
  count_launch();
}
void from_compact(Ctx& ctx, const CView& z, const QView& out) {
  if (out.rows * out.cols == 0) return;
  k_from_compact<<<grid_of(out.rows * out.cols), 256, 0, ctx.stream>>>(z, out);
  QLRA_LAUNCH_CHECK();
  count_launch();
}
void j_mul_conj(Ctx& ctx, const CView& u, const CView& out) {
  if (u.rows * u.cols == 0) return;
  k_j_mul_conj<<<grid_of(u.rows / 2 * u.cols), 256, 0, ctx.stream>>>(u, out);
  QLRA_LAUNCH_CHECK();
  count_launch();
}
void cmat_to_quat(Ctx& ctx, const CView& c, const QView& out) {
  if (out.rows * out.cols == 0) return;
  k_cmat_to_quat<<<grid_of(out.rows * out.cols), 256, 0, ctx.stream>>>(c, out);
  QLRA_LAUNCH_CHECK();
  count_launch();
}
void quat_to_cmat(Ctx& ctx, const QView& q, const CView& out) {
  if (q.rows * q.cols == 0) return;
  k_quat_to_cmat<<<grid_of(q.rows * q.cols), 256, 0, ctx.stream>>>(q, out);
  QLRA_LAUNCH_CHECK();
  count_launch();
}

}  // namespace qlra_dev
