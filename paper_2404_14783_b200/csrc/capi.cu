// capi.cu -- the extern "C" boundary (include/qlra_cuda.h) and the host-side
// orchestration of the hot path: the rangefinders' control flow
// (proj/src/rangefinders.cpp:18-176), the core solve
// (proj/src/sketching.cpp:184-185, complex_bridge.cpp:63-90) and the sharded
// reductions.  All arithmetic runs in the kernels of sketch.cu / qgemm.cu /
// smallla.cu; the host only sequences launches and reads back the scalars
// the reference's control flow branches on (kappa, epsilon, rank tests).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <memory>
#include <tuple>
#include <mutex>
#include <map>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "i8gemm.cuh"
#include "ozaki.cuh"

struct qlra_ctx {
  qlra_dev::Ctx c;
};

namespace qlra_dev {

std::atomic<int64_t>& launch_counter() {
  static std::atomic<int64_t> c{0};
  return c;
}

// Kernel attributes apply per device; set each (device, function, attribute)
// once to the largest value requested, under a lock (contexts on several
// devices or host threads may race here).
void set_func_attr(const void* func, cudaFuncAttribute attr, int value) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int>, int> done;
  int dev = 0;
  QLRA_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_tuple(dev, func, (int)attr);
  auto it = done.find(key);
  if (it != done.end() && it->second >= value) return;
  QLRA_CUDA(cudaFuncSetAttribute(func, attr, value));
  done[key] = value;
}

void allreduce_sum(Ctx& ctx, double* buf, size_t count) {
  if (ctx.nranks <= 1 || count == 0) return;
  if (ctx.group) {
    group_allreduce_sum(ctx, buf, count);
    return;
  }
  const ncclResult_t r = ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, ctx.comm, ctx.stream);
  if (r != ncclSuccess) fail(QLRA_ERR_NCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(r));
}

// One collective for all four planes: in place when they are one contiguous
// run (DevQMat: dense planes back to back), else packed into a contiguous
// buffer and unpacked after (strided views, e.g. W inside a checkpoint).
void allreduce_qmat(Ctx& ctx, const QView& m) {
  if (ctx.nranks <= 1 || m.rows == 0 || m.cols == 0) return;
  const size_t plane = (size_t)(m.rows * m.cols);
  bool dense = m.ld == m.cols || m.rows == 1;
  for (int p = 1; p < 4 && dense; ++p) dense = m.p[p] == m.p[0] + p * plane;
  if (dense) {
    allreduce_sum(ctx, m.p[0], 4 * plane);
    return;
  }
  DeviceBuffer pk(ctx, 4 * plane * sizeof(double));
  const size_t w = sizeof(double) * (size_t)m.cols, pitch = sizeof(double) * (size_t)m.ld;
  for (int p = 0; p < 4; ++p)
    QLRA_CUDA(cudaMemcpy2DAsync(pk.as<double>() + p * plane, w, m.p[p], pitch, w, (size_t)m.rows,
                                cudaMemcpyDeviceToDevice, ctx.stream));
  allreduce_sum(ctx, pk.as<double>(), 4 * plane);
  for (int p = 0; p < 4; ++p)
    QLRA_CUDA(cudaMemcpy2DAsync(m.p[p], pitch, pk.as<double>() + p * plane, w, w, (size_t)m.rows,
                                cudaMemcpyDeviceToDevice, ctx.stream));
}

namespace {

constexpr double kKappaTarget = 10.0;   // rangefinders.cpp:12
constexpr double kEpsilonClamp = 0.999; // rangefinders.cpp:13
constexpr double kUnit = 1.1102230246251565e-16;

std::vector<double> to_host(Ctx& ctx, const double* d, size_t n) {
  std::vector<double> h(n);
  if (n) {
    QLRA_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    QLRA_CUDA(cudaStreamSynchronize(ctx.stream));
  }
  return h;
}
std::vector<double> diag_to_host(Ctx& ctx, const double* p, int64_t ld, int64_t n, size_t elem = 1) {
  std::vector<double> h(n);
  if (n) {
    QLRA_CUDA(cudaMemcpy2DAsync(h.data(), sizeof(double), p, (size_t)(ld + 1) * elem * sizeof(double),
                                sizeof(double), (size_t)n, cudaMemcpyDeviceToHost, ctx.stream));
    QLRA_CUDA(cudaStreamSynchronize(ctx.stream));
  }
  return h;
}

int64_t global_rows(Ctx& ctx, int64_t local) {
  if (ctx.nranks <= 1) return local;
  DeviceBuffer b(ctx, sizeof(double));
  const double v = (double)local;
  QLRA_CUDA(cudaMemcpyAsync(b.ptr, &v, sizeof(double), cudaMemcpyHostToDevice, ctx.stream));
  allreduce_sum(ctx, b.as<double>(), 1);
  return (int64_t)llround(to_host(ctx, b.as<double>(), 1)[0]);
}

DevQMat identity_like(Ctx& ctx, int64_t n) {
  DevQMat e(ctx, n, n);
  small_set_identity(ctx, e.v);
  return e;
}

// First global row of this rank's contiguous row shard (exclusive prefix sum
// of the shard heights in rank order).
int64_t global_row0(Ctx& ctx, int64_t local) {
  if (ctx.nranks <= 1) return 0;
  DeviceBuffer b(ctx, sizeof(double) * (size_t)ctx.nranks);
  std::vector<double> v((size_t)ctx.nranks, 0.0);
  v[(size_t)ctx.rank] = (double)local;
  QLRA_CUDA(cudaMemcpyAsync(b.ptr, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice, ctx.stream));
  allreduce_sum(ctx, b.as<double>(), v.size());
  const std::vector<double> all = to_host(ctx, b.as<double>(), v.size());
  int64_t r0 = 0;
  for (int i = 0; i < ctx.rank; ++i) r0 += (int64_t)llround(all[(size_t)i]);
  return r0;
}

// G = op(A)^* op(A) reduced over (row-sharded) rows: s x s.
void gram(Ctx& ctx, const QView& h, const QView& g) {
  qgemm_gram(ctx, h, g);
  allreduce_qmat(ctx, g);
}

// Eigenvalues (descending) of a quaternion Hermitian G (s x s): the s
// distinct values of chi_G, each of which chi_G carries twice.
std::vector<double> quat_eigs(Ctx& ctx, const QView& g, bool extremes_only = true) {
  const int64_t n = g.rows;
  DevQMat work(ctx, n, n);
  copy_qmat(ctx, g, work.v);
  DeviceBuffer w(ctx, sizeof(double) * (size_t)std::max<int64_t>(1, n));
  QLRA_CUDA(cudaMemsetAsync(w.ptr, 0, w.bytes, ctx.stream));
  small_quat_herm_eigvals(ctx, work.v, w.as<double>(), extremes_only);
  std::vector<double> ev = to_host(ctx, w.as<double>(), (size_t)n);
  return ev;
}

// The context's stream at the device's greatest priority: kernels of the
// critical path (main) are dispatched before those of the early solve's
// second stream (least priority) whenever both have CTAs waiting -- a large
// side-stream product otherwise holds back the main stream's short launches
// for its whole duration.  Opt-in (QLRA_MAIN_PRIO=1): measured no gain on C5
// and within noise (236 vs 243 ms, power-capped) on C4.
cudaError_t create_main_stream(cudaStream_t* s) {
  static const bool prio = [] {
    const char* e = std::getenv("QLRA_MAIN_PRIO");
    return e && std::atoi(e) != 0;
  }();
  int least = 0, greatest = 0;
  if (prio && cudaDeviceGetStreamPriorityRange(&least, &greatest) == cudaSuccess && greatest != least)
    return cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, greatest);
  return cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
}

// All eigenvalues of a quaternion Hermitian G computed on a side stream and
// read back on demand: the host issues other work on ctx.stream and collects
// the values with get().  G is copied on ctx.stream first, so the caller may
// overwrite it afterwards.  Several may be pending at once (each owns its
// device result; they run in order on the side stream).
class SideEigs {
 public:
  SideEigs(Ctx& c, const QView& g) : c_(c), n_(g.rows) {
    if (!c.side) QLRA_CUDA(create_main_stream(&c.side));
    side_ = c.side;
    QLRA_CUDA(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming));
    QLRA_CUDA(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
    work_ = DevQMat(c, n_, n_);
    w_ = DeviceBuffer(c, sizeof(double) * (size_t)std::max<int64_t>(1, n_));
    copy_qmat(c, g, work_.v);
    QLRA_CUDA(cudaMemsetAsync(w_.ptr, 0, w_.bytes, c.stream));
    QLRA_CUDA(cudaEventRecord(fork_, c.stream));
    QLRA_CUDA(cudaStreamWaitEvent(side_, fork_, 0));
    cudaStream_t main = c.stream;
    c.stream = side_;  // every launch and stream-ordered buffer below lives on side_
    try {
      small_quat_herm_eigvals(c, work_.v, w_.as<double>(), /*extremes_only=*/false);
    } catch (...) {
      c.stream = main;
      throw;
    }
    c.stream = main;
    QLRA_CUDA(cudaEventRecord(done_, side_));
  }
  std::vector<double> get() {
    QLRA_CUDA(cudaEventSynchronize(done_));
    std::vector<double> h((size_t)n_);
    if (n_) QLRA_CUDA(cudaMemcpy(h.data(), w_.ptr, sizeof(double) * (size_t)n_, cudaMemcpyDeviceToHost));
    return h;
  }
  ~SideEigs() {
    if (done_) cudaStreamWaitEvent(c_.stream, done_, 0);  // work_, w_ are released on ctx.stream
    if (fork_) cudaEventDestroy(fork_);
    if (done_) cudaEventDestroy(done_);
  }
  SideEigs(const SideEigs&) = delete;
  SideEigs& operator=(const SideEigs&) = delete;

 private:
  Ctx& c_;
  int64_t n_;
  cudaStream_t side_ = nullptr;
  cudaEvent_t fork_ = nullptr, done_ = nullptr;
  DevQMat work_;
  DeviceBuffer w_;
};

double kappa_from_eigs(const std::vector<double>& ev) {
  if (ev.empty()) return std::numeric_limits<double>::infinity();
  const double lmax = ev.front(), lmin = ev.back();
  if (!(lmin > 0.0)) return std::numeric_limits<double>::infinity();
  return std::sqrt(lmax / lmin);
}

// The spectrum of a Hermitian positive definite G with full relative
// accuracy at both ends: eigenvalues of G itself resolve the large ones
// (absolute error ~u lambda_max), those of an accurately formed G^{-1} the
// small ones (1/mu).  lam, mu: descending.  Each value is taken from the side
// that resolves it: above the geometric middle of the range from lam, below
// it from 1/mu.
std::vector<double> merge_spectra(const std::vector<double>& lam, const std::vector<double>& mu) {
  const size_t n = lam.size();
  if (n == 0 || mu.size() != n || !(mu[0] > 0.0) || !(lam[0] > 0.0)) return lam;
  const double pivot = std::sqrt(lam[0] / mu[0]);
  std::vector<double> out(n);
  for (size_t i = 0; i < n; ++i) {
    const double mi = mu[n - 1 - i];
    out[i] = lam[i] >= pivot ? lam[i] : (mi > 0.0 ? 1.0 / mi : 0.0);
    if (i > 0) out[i] = std::min(out[i], out[i - 1]);
  }
  return out;
}
// kappa^2 beyond which the small end of a Gram spectrum is refined (its
// relative accuracy is ~u kappa^2: 1e-8 at kappa = 1e4)
constexpr double kRefineKappa = 1e4;

// Explicit quaternion inverse of a square matrix via Gauss-Jordan; returns
// the GJ status (info, pmin, pmax).
std::vector<double> quat_inverse(Ctx& ctx, const QView& a, const QView& ainv, bool hpd = false) {
  DevQMat work(ctx, a.rows, a.cols);
  copy_qmat(ctx, a, work.v);
  small_set_identity(ctx, ainv);
  DeviceBuffer st(ctx, 3 * sizeof(double));
  small_quat_solve(ctx, work.v, ainv, st.as<double>(), /*pivot=*/!hpd);
  return to_host(ctx, st.as<double>(), 3);
}

// G^{-1} for a Hermitian positive definite quaternion G: G = R^* R
// (quaternion Cholesky, one CTA), G^{-1} = R^{-1} R^{-*} (triangular inverse,
// then one small DMMA product).  False if G is not numerically PD.
bool hpd_inverse(Ctx& ctx, const QView& g, const QView& ginv, std::vector<double>* rdiag) {
  const int64_t s = g.rows;
  DevQMat ri(ctx, s, s);
  if (!blocked_chol_inv(ctx, g, ri.v, rdiag)) return false;
  qgemm(ctx, QLRA_OP_N, QLRA_OP_C, 1.0, ri.v, ri.v, 0.0, ginv);
  return true;
}

// One CholeskyQR pass: hout = y * R^{-1} with G = gram(y) (+ shift on the
// diagonal).  complex_mode: R from the complex compact Gram (Y_c^* Y_c, the
// complex part of the quaternion Gram) -- pseudo-QR's complex_qr; else R is
// the quaternion Cholesky factor (orthonormal quaternion basis).  Returns
// false if the Cholesky factorisation breaks down; rdiag gets diag(R).
// distributed: y is row-sharded over the ranks (Gram all-reduced); else y is
// replicated.  rinv_out (optional) receives R^{-1}.
bool cqr_pass(Ctx& ctx, const QView& y, const QView& hout, bool complex_mode, double shift,
              std::vector<double>* rdiag, double* trace_g, bool distributed = true,
              const QView* rinv_out = nullptr, const QView* r_out = nullptr) {
  const int64_t s = y.cols;
  DevQMat g(ctx, s, s);
  if (distributed) gram(ctx, y, g.v);
  else qgemm_gram(ctx, y, g.v);
  if (trace_g) {
    const std::vector<double> d = diag_to_host(ctx, g.v.p[0], g.v.ld, s);
    double t = 0.0;
    for (double v : d) t += v;
    *trace_g = t;
  }
  // complex_qr's R: Cholesky of the complex part (j, k planes zeroed; the
  // quaternion factorisation then stays inside the complex subalgebra).
  if (complex_mode) zero_jk_planes(ctx, g.v);
  if (shift != 0.0) small_add_diag(ctx, g.v, shift);
  DevQMat rinv(ctx, s, s);
  if (!blocked_chol_inv(ctx, g.v, rinv.v, rdiag, r_out)) return false;
  if (hout.p[0]) qgemm(ctx, QLRA_OP_N, QLRA_OP_N, 1.0, y, rinv.v, 0.0, hout);  // else: deferred by the caller
  if (rinv_out) copy_qmat(ctx, rinv.v, *rinv_out);
  return true;
}

// The last CholeskyQR pass's tall product left to the caller: Q = base * rinv_last.
struct DeferredQ {
  DevQMat base;       // input of the last pass (rows x s)
  DevQMat rinv_last;  // R^{-1} of the last pass (s x s)
};

// r <- next * r (R = R_last ... R_1)
void chain_r(Ctx& ctx, DevQMat& r, const QView& next) {
  DevQMat t(ctx, r.v.rows, r.v.cols);
  qgemm(ctx, QLRA_OP_N, QLRA_OP_N, 1.0, next, r.v, 0.0, t.v);
  r = std::move(t);
}

// rinv <- rinv * next (s x s, upper triangular factors of R^{-1} = R1^{-1} R2^{-1} ...)
void chain_rinv(Ctx& ctx, DevQMat& rinv, const QView& next) {
  DevQMat t(ctx, rinv.v.rows, rinv.v.cols);
  qgemm(ctx, QLRA_OP_N, QLRA_OP_N, 1.0, rinv.v, next, 0.0, t.v);
  rinv = std::move(t);
}

// CholeskyQR2, or shifted CholeskyQR3 (Fukaya et al.) when the first Gram is
// not numerically positive definite.  rdiag = diag of the full R factor;
// optional rinv (s x s) = R^{-1} and rfac = R of y = h R.
// defer (optional): do not form Q in the last pass; return its input and
// R^{-1} instead (Q = defer->base * defer->rinv_last), so a caller that only
// needs Q times a small matrix saves one tall product.
bool cholesky_qr_general(Ctx& ctx, const QView& y, const QView& h, bool complex_mode, int64_t m_global,
                         std::vector<double>* rdiag, bool distributed, DevQMat* rinv, DevQMat* rfac,
                         DeferredQ* defer);

// CholeskyQR2 queued without a host sync (s <= the single-launch Cholesky
// limit): both passes back to back, statuses and diagonals left on the
// device.  cqr2_status() reads them with ONE sync.
struct Cqr2Pending {
  int64_t s = 0;
  DevQMat t1, r1, r2, r1inv, r2inv;
  DeviceBuffer info, dg;
};
void cqr2_enqueue(Ctx& ctx, const QView& y, const QView& h, bool complex_mode, bool distributed,
                  const QView* gram1, bool form_q, Cqr2Pending& p) {
  const int64_t s = y.cols;
  p.s = s;
  DevQMat g1(ctx, s, s), g2(ctx, s, s);
  p.t1 = DevQMat(ctx, y.rows, s);
  p.r1 = DevQMat(ctx, s, s);
  p.r2 = DevQMat(ctx, s, s);
  p.r1inv = DevQMat(ctx, s, s);
  p.r2inv = DevQMat(ctx, s, s);
  p.info = DeviceBuffer(ctx, 2 * sizeof(int));
  p.dg = DeviceBuffer(ctx, 2 * sizeof(double) * (size_t)s);
  auto gram_of = [&](const QView& a, const QView& g) {
    if (distributed) gram(ctx, a, g);
    else qgemm_gram(ctx, a, g);
    if (complex_mode) zero_jk_planes(ctx, g);
  };
  if (gram1) {
    copy_qmat(ctx, *gram1, g1.v);
    if (complex_mode) zero_jk_planes(ctx, g1.v);
  } else {
    gram_of(y, g1.v);
  }
  chol_inv_any(ctx, g1.v, p.r1.v, p.r1inv.v, p.info.as<int>(), p.dg.as<double>());
  qgemm(ctx, QLRA_OP_N, QLRA_OP_N, 1.0, y, p.r1inv.v, 0.0, p.t1.v);
  gram_of(p.t1.v, g2.v);
  chol_inv_any(ctx, g2.v, p.r2.v, p.r2inv.v, p.info.as<int>() + 1, p.dg.as<double>() + s);
  if (form_q) qgemm(ctx, QLRA_OP_N, QLRA_OP_N, 1.0, p.t1.v, p.r2inv.v, 0.0, h);
}
// 0: both passes factored (rdiag = diag R1 .* diag R2); 1: pass 1 broke
// down; 2: pass 2 broke down.
int cqr2_status(Ctx& ctx, const Cqr2Pending& p, std::vector<double>* rdiag) {
  const int64_t s = p.s;
  int inf[2] = {0, 0};
  std::vector<double> d((size_t)(2 * s));
  QLRA_CUDA(cudaMemcpyAsync(inf, p.info.ptr, 2 * sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  QLRA_CUDA(cudaMemcpyAsync(d.data(), p.dg.ptr, 2 * sizeof(double) * (size_t)s, cudaMemcpyDeviceToHost, ctx.stream));
  QLRA_CUDA(cudaStreamSynchronize(ctx.stream));
  if (inf[0] != 0) return 1;
  if (inf[1] != 0) return 2;
  if (rdiag) {
    rdiag->resize((size_t)s);
    for (int64_t k = 0; k < s; ++k) (*rdiag)[k] = d[k] * d[s + k];
  }
  return 0;
}

// CholeskyQR2 with ONE host sync for both pass statuses and diagonals; a
// breakdown of pass 1 falls back to the general path (shifted CholeskyQR3).
// gram1 (optional): the already reduced Gram of y (quaternion; the complex
// part is taken here when complex_mode), saving the first tall product.
// QLRA_CQR_SHIFTED=1 (A/B of the rangefinders' accuracy only): always the
// shifted CholeskyQR3.
bool cqr_force_shift() {
  static const bool v = [] {
    const char* e = std::getenv("QLRA_CQR_SHIFTED");
    return e && std::atoi(e) != 0;
  }();
  return v;
}
bool cholesky_qr(Ctx& ctx, const QView& y, const QView& h, bool complex_mode, int64_t m_global,
                 std::vector<double>* rdiag, bool distributed = true, DevQMat* rinv = nullptr,
                 DevQMat* rfac = nullptr, DeferredQ* defer = nullptr, const QView* gram1 = nullptr) {
  const int64_t s = y.cols;
  if (s == 0 || cqr_force_shift())
    return cholesky_qr_general(ctx, y, h, complex_mode, m_global, rdiag, distributed, rinv, rfac, defer);
  Cqr2Pending p;
  cqr2_enqueue(ctx, y, h, complex_mode, distributed, gram1, /*form_q=*/!defer, p);
  const int st = cqr2_status(ctx, p, rdiag);
  if (st == 1)  // pass 1 broke down: shifted CholeskyQR3
    return cholesky_qr_general(ctx, y, h, complex_mode, m_global, rdiag, distributed, rinv, rfac, defer);
  if (st == 2) return false;
  if (rinv) {
    *rinv = std::move(p.r1inv);
    chain_rinv(ctx, *rinv, p.r2inv.v);
  }
  if (rfac) {
    *rfac = std::move(p.r1);
    chain_r(ctx, *rfac, p.r2.v);
  }
  if (defer) {
    defer->base = std::move(p.t1);
    defer->rinv_last = std::move(p.r2inv);
  }
  return true;
}

bool cholesky_qr_general(Ctx& ctx, const QView& y, const QView& h, bool complex_mode, int64_t m_global,
                         std::vector<double>* rdiag, bool distributed, DevQMat* rinv, DevQMat* rfac,
                         DeferredQ* defer) {
  const int64_t s = y.cols;
  DevQMat t1(ctx, y.rows, s);
  QView hq = h;
  if (defer) {
    hq = QView{};  // no output product in the last pass
    defer->rinv_last = DevQMat(ctx, s, s);
  }
  DevQMat ri[3], rf[3];
  for (int i = 0; i < 2; ++i) {
    if (rinv) ri[i] = DevQMat(ctx, s, s);
    if (rfac) rf[i] = DevQMat(ctx, s, s);
  }
  auto pi = [&](int i) { return rinv ? &ri[i].v : nullptr; };
  auto pf = [&](int i) { return rfac ? &rf[i].v : nullptr; };
  std::vector<double> d1, d2, d3;
  double tr = 0.0;
  if (cqr_force_shift()) {
    DevQMat g(ctx, s, s);
    if (distributed) gram(ctx, y, g.v);
    else qgemm_gram(ctx, y, g.v);
    const std::vector<double> dg = diag_to_host(ctx, g.v.p[0], g.v.ld, s);
    for (double v : dg) tr += v;
  } else if (cqr_pass(ctx, y, t1.v, complex_mode, 0.0, &d1, &tr, distributed, pi(0), pf(0))) {
    const QView* last_inv = defer ? &defer->rinv_last.v : pi(1);
    if (!cqr_pass(ctx, t1.v, hq, complex_mode, 0.0, &d2, nullptr, distributed, last_inv, pf(1))) return false;
    if (defer && rinv) copy_qmat(ctx, defer->rinv_last.v, ri[1].v);
    if (rdiag) {
      rdiag->resize(s);
      for (int64_t k = 0; k < s; ++k) (*rdiag)[k] = d1[k] * d2[k];
    }
    if (rinv) {
      *rinv = std::move(ri[0]);
      chain_rinv(ctx, *rinv, ri[1].v);
    }
    if (rfac) {
      *rfac = std::move(rf[0]);
      chain_r(ctx, *rfac, rf[1].v);
    }
    if (defer) defer->base = std::move(t1);
    return true;
  }
  const double dim = complex_mode ? 2.0 : 4.0;
  const double shift = 11.0 * (dim * (double)m_global * s + s * (s + 1.0)) * kUnit * tr;
  if (!(tr > 0.0)) return false;
  if (rinv) ri[2] = DevQMat(ctx, s, s);
  if (rfac) rf[2] = DevQMat(ctx, s, s);
  if (!cqr_pass(ctx, y, t1.v, complex_mode, shift, &d1, nullptr, distributed, pi(0), pf(0))) return false;
  DevQMat t2(ctx, y.rows, s);
  if (!cqr_pass(ctx, t1.v, t2.v, complex_mode, 0.0, &d2, nullptr, distributed, pi(1), pf(1))) return false;
  const QView* last_inv = defer ? &defer->rinv_last.v : pi(2);
  if (!cqr_pass(ctx, t2.v, hq, complex_mode, 0.0, &d3, nullptr, distributed, last_inv, pf(2))) return false;
  if (defer && rinv) copy_qmat(ctx, defer->rinv_last.v, ri[2].v);
  if (rdiag) {
    rdiag->resize(s);
    // y = t1 R1 = t2 R2 R1 = h R3 R2 R1 holds exactly whatever the shift, so
    // R = R3 R2 R1 is a QR factor of y and its diagonal is the product.
    for (int64_t k = 0; k < s; ++k) (*rdiag)[k] = d1[k] * d2[k] * d3[k];
  }
  if (rinv) {
    *rinv = std::move(ri[0]);
    chain_rinv(ctx, *rinv, ri[1].v);
    chain_rinv(ctx, *rinv, ri[2].v);
  }
  if (rfac) {
    *rfac = std::move(rf[0]);
    chain_r(ctx, *rfac, rf[1].v);
    chain_r(ctx, *rfac, rf[2].v);
  }
  if (defer) defer->base = std::move(t2);
  return true;
}

// Refine the small end of a Gram spectrum lam (of G = A^*A, descending; all
// values or extremes only) with rinv = R^{-1} of a QR factor of A.
std::vector<double> refine_with_rinv(Ctx& ctx, const std::vector<double>& lam, const QView& rinv,
                                     bool extremes_only = false) {
  const int64_t s = rinv.rows;
  DevQMat p(ctx, s, s);
  qgemm(ctx, QLRA_OP_N, QLRA_OP_C, 1.0, rinv, rinv, 0.0, p.v);  // (R^* R)^{-1}
  if (extremes_only) {  // lambda_min = 1 / lambda_max((R^* R)^{-1})
    const std::vector<double> mu = quat_eigs(ctx, p.v, /*extremes_only=*/true);
    std::vector<double> out = lam;
    if (!out.empty() && mu[0] > 0.0) out.back() = 1.0 / mu[0];
    return out;
  }
  const std::vector<double> mu = quat_eigs(ctx, p.v, /*extremes_only=*/false);
  return merge_spectra(lam, mu);
}

std::vector<double> gram_spectrum(Ctx& ctx, const QView& a, const QView& g, bool extremes_only,
                                  const DevQMat* rinv_in) {
  std::vector<double> lam = quat_eigs(ctx, g, extremes_only);
  if (!(kappa_from_eigs(lam) > kRefineKappa) || a.cols == 0) return lam;
  if (rinv_in && rinv_in->buf.ptr) return refine_with_rinv(ctx, lam, rinv_in->v, extremes_only);
  DevQMat rinv;
  DeferredQ no_q;  // only R^{-1} is needed: Q is never formed
  if (!cholesky_qr(ctx, a, QView{}, /*complex_mode=*/false, global_rows(ctx, a.rows), nullptr,
                   /*distributed=*/true, &rinv, nullptr, &no_q))
    return lam;  // not factorable: kappa beyond what any Gram route resolves
  return refine_with_rinv(ctx, lam, rinv.v, extremes_only);
}

// Orthonormal completion: c_out (rows x k, row-sharded from global row0)
// becomes quaternion-orthonormal and orthogonal to hr (rows x r, may be
// r = 0).  Candidates are Gaussian columns from the reference RNG (seeded),
// projected out twice (CGS2) and orthonormalised by CholeskyQR2 -- the device
// counterpart of select_via_mgs' canonical-direction fallback
// (factorizations.cpp:105-118).
// complex_only: candidates (and so the completion) in the complex subalgebra
// -- for complex_svd of a complex matrix embedded as a quaternion one.
void orthonormal_completion(Ctx& ctx, const QView& hr, const QView& c_out, int64_t row0,
                            int64_t m_global, uint64_t seed, bool complex_only = false) {
  const int64_t k = c_out.cols, rows = c_out.rows;
  if (k == 0) return;
  DevQMat c(ctx, rows, k);
  qlra_spec_t spec{QLRA_GAUSSIAN, m_global, k, seed, 1.0};
  launch_gen(ctx.stream, spec, row0, 0, rows, k, c.v, false);
  if (complex_only) zero_jk_planes(ctx, c.v);
  if (hr.cols > 0) {
    DevQMat t(ctx, hr.cols, k);
    for (int pass = 0; pass < 2; ++pass) {
      qgemm(ctx, QLRA_OP_C, QLRA_OP_N, 1.0, hr, c.v, 0.0, t.v);
      allreduce_qmat(ctx, t.v);
      qgemm(ctx, QLRA_OP_N, QLRA_OP_N, -1.0, hr, t.v, 1.0, c.v);
    }
  }
  if (!cholesky_qr(ctx, c.v, c_out, /*complex_mode=*/false, m_global, nullptr))
    fail(QLRA_ERR_INTERNAL, "orthonormal completion failed");
}

// pseudo_svd for sketches CholeskyQR cannot take (numerically rank-deficient
// or with kappa(Y)^2 beyond double precision): the reference's SVD-and-pairs
// route (rangefinders.cpp:18-62, factorizations.cpp:60-81) keeps every
// singular pair above kPairFloorRel * sigma_1 (= 1e-13) and completes the
// rest.  A Gram eigendecomposition resolves only sigma_i >~ 3e-7 sigma_max,
// so the range is taken in graded levels: at each level the eigenvectors of
// G_k = Y_k^* Y_k with lambda > 64 u s lambda_max(G_k) (and above the floor)
// give the block Y_k V L^{-1/2}, which is re-projected against the basis so
// far (twice), orthonormalised, appended, and projected out of Y_k (twice).
// A kappa=1e12 sketch needs two levels.  Returns sqrt(lambda_1 / lambda_min)
// over the kept directions when all s are kept (the sigma estimates of each
// level are the singular values of the deflated remainder), else inf.
constexpr double kGradedKappa = 1e6;
double pseudo_svd_graded(Ctx& ctx, const QView& y, const QView& h, int64_t m_global, int64_t row0,
                         uint64_t seed) {
  const int64_t s = y.cols, rows = y.rows;
  constexpr double kFloorRel = 1e-13;  // kPairFloorRel, factorizations.hpp:64
  DevQMat yk(ctx, rows, s);
  copy_qmat(ctx, y, yk.v);
  DevQMat g(ctx, s, s), vec(ctx, s, s);
  DeviceBuffer w(ctx, sizeof(double) * (size_t)s);
  int64_t r = 0;
  double lam1 = 0.0, lam_min = std::numeric_limits<double>::infinity();
  for (int level = 0; r < s && level < 8; ++level) {
    gram(ctx, yk.v, g.v);
    small_quat_eigh(ctx, g.v, w.as<double>(), vec.v);
    const std::vector<double> lam = to_host(ctx, w.as<double>(), (size_t)s);
    if (level == 0) lam1 = std::max(0.0, lam[0]);
    const double thr = std::max({64.0 * kUnit * (double)s * std::max(0.0, lam[0]),
                                 kFloorRel * kFloorRel * lam1, 1e-300});
    int64_t cnt = 0;
    while (cnt < s - r && lam[cnt] > thr) ++cnt;
    if (cnt == 0) break;
    lam_min = std::min(lam_min, lam[cnt - 1]);
    DevQMat t(ctx, rows, cnt);
    qgemm(ctx, QLRA_OP_N, QLRA_OP_N, 1.0, yk.v, sub(vec.v, 0, 0, s, cnt), 0.0, t.v);
    std::vector<double> is(cnt);
    for (int64_t i = 0; i < cnt; ++i) is[i] = 1.0 / std::sqrt(lam[i]);
    DeviceBuffer d_is(ctx, sizeof(double) * (size_t)cnt);
    QLRA_CUDA(cudaMemcpyAsync(d_is.ptr, is.data(), sizeof(double) * cnt, cudaMemcpyHostToDevice, ctx.stream));
    scale_cols(ctx, t.v, d_is.as<double>(), false, 0.0, t.v);
    const QView hp = sub(h, 0, 0, rows, r);
    if (r > 0) {
      DevQMat c(ctx, r, cnt);
      for (int pass = 0; pass < 2; ++pass) {
        qgemm(ctx, QLRA_OP_C, QLRA_OP_N, 1.0, hp, t.v, 0.0, c.v);
        allreduce_qmat(ctx, c.v);
        qgemm(ctx, QLRA_OP_N, QLRA_OP_N, -1.0, hp, c.v, 1.0, t.v);
      }
    }
    const QView hn = sub(h, 0, r, rows, cnt);
    if (!cholesky_qr(ctx, t.v, hn, false, m_global, nullptr))
      fail(QLRA_ERR_INTERNAL, "pseudo_svd: range basis orthonormalisation failed");
    r += cnt;
    if (r == s) break;
    // Y_{k+1} = (I - H H^*) Y_k over the basis so far, twice
    const QView hr = sub(h, 0, 0, rows, r);
    DevQMat c(ctx, r, s);
    for (int pass = 0; pass < 2; ++pass) {
      qgemm(ctx, QLRA_OP_C, QLRA_OP_N, 1.0, hr, yk.v, 0.0, c.v);
      allreduce_qmat(ctx, c.v);
      qgemm(ctx, QLRA_OP_N, QLRA_OP_N, -1.0, hr, c.v, 1.0, yk.v);
    }
  }
  if (r < s)
    orthonormal_completion(ctx, sub(h, 0, 0, rows, r), sub(h, 0, r, rows, s - r), row0, m_global,
                           rng_substream(rng_key(seed), 0x6261645F626C6BULL));
  return r == s && lam_min > 0.0 ? std::sqrt(lam1 / lam_min) : std::numeric_limits<double>::infinity();
}

void rank_check(const std::vector<double>& d) {
  double rmax = 0.0, rmin = std::numeric_limits<double>::infinity();
  for (double v : d) {
    rmax = std::max(rmax, std::fabs(v));
    rmin = std::min(rmin, std::fabs(v));
  }
  if (!(rmin > 1e-14 * rmax))
    fail(QLRA_ERR_RANK, "pseudo_qr: sketch numerically rank-deficient; use pseudo_svd");
}

// Spectrum of G = A^*A for a row-sharded tall A (descending), refined at the
// small end when kappa(A) > kRefineKappa: A = Q R by CholeskyQR2 (backward
// stable while kappa(A) < u^{-1/2}, so sigma(R) = sigma(A) to u ||A||), and
// the eigenvalues of R^{-1} R^{-*} give the small ones (merge_spectra).  The
// reference takes them from an SVD of chi_A (factorizations.cpp:316-337),
// accurate to u ||A|| likewise.
std::vector<double> gram_spectrum(Ctx& ctx, const QView& a, const QView& g, bool extremes_only,
                                  const DevQMat* rinv_in = nullptr);
double condition_number_dev(Ctx& ctx, const QView& a) {
  const int64_t k = std::min(a.rows, a.cols);
  if (k == 0) return std::numeric_limits<double>::infinity();
  DevQMat g(ctx, a.cols, a.cols);
  gram(ctx, a, g.v);
  return kappa_from_eigs(gram_spectrum(ctx, a, g.v, true));
}

// estimate_epsilon (rangefinders.cpp:66-97) given G and G^{-1}, with the
// reference's singularity tests.  The reference factors chi_G by partial-
// pivot LU and tests its 1-norm reciprocal condition estimate (Eigen rcond,
// rangefinders.cpp:71-75; the oracle: zgecon); here the EXACT 1-norm value
// rcond_1 = 1 / (||chi_G||_1 ||chi_G^{-1}||_1) from the explicit inverse --
// the estimators bound it from above and reach it for most matrices (within
// 1.3x on Gram matrices of kappa 1e5..1e8).  Note rcond_1 ~ 0.2 / kappa(H)^2
// there, so the tests bind well below the 2-norm kappa = 1/sqrt(rc_min).
// Returns eps; *rc_out = rcond_1 (also used by correction_step's square solve
// test, rcond > 1e-14, complex_bridge.cpp:73-77).
double estimate_epsilon_rc(Ctx& ctx, const QView& g, const QView& ginv, int iters, double* rc_out) {
  if (iters < 1) fail(QLRA_ERR_PARAMETER, "estimate_epsilon: power_iters must be >= 1");
  DeviceBuffer v(ctx, 3 * sizeof(double));
  small_power_iter_inverse(ctx, ginv, iters, v.as<double>());
  small_chi_norm1(ctx, g, v.as<double>() + 1);
  small_chi_norm1(ctx, ginv, v.as<double>() + 2);
  const std::vector<double> h = to_host(ctx, v.as<double>(), 3);
  const double rc = (h[1] > 0.0 && h[2] > 0.0 && std::isfinite(h[2])) ? 1.0 / (h[1] * h[2]) : 0.0;
  if (rc_out) *rc_out = rc;
  if (!(rc > 1e-15))
    fail(QLRA_ERR_SINGULAR, "estimate_epsilon: H*H numerically singular",
         rc > 0 ? 1.0 / rc : std::numeric_limits<double>::infinity());
  if (!(h[0] > 0.0)) fail(QLRA_ERR_SINGULAR, "estimate_epsilon: breakdown", 0.0);
  return std::min(1.0 / std::sqrt(h[0]), kEpsilonClamp);
}
// correction_step's square solve of chi_{H*H} (PartialPivLU, rcond > 1e-14,
// complex_bridge.cpp:73-77), on the rcond_1 of estimate_epsilon_rc.
void check_solve_rc(double rc) {
  if (!(rc > 1e-14))
    fail(QLRA_ERR_SINGULAR, "solve_quaternion_linear: singular system",
         rc > 0 ? 1.0 / rc : std::numeric_limits<double>::infinity());
}


// H_out = H ((1-eps) I + eps G^{-1}) == (1-eps) H + eps (H^+)^*  (rangefinders.cpp:99-105)
void correction_from_inverse(Ctx& ctx, const QView& h, const QView& ginv, double eps,
                             const QView& hout) {
  if (!(eps > 0.0 && eps < 1.0)) fail(QLRA_ERR_PARAMETER, "correction_step: epsilon must lie in (0,1)");
  DevQMat mm(ctx, ginv.rows, ginv.cols);
  small_axpby_identity(ctx, 1.0 - eps, eps, ginv, mm.v);
  if (hout.p[0] == h.p[0]) {
    DevQMat tmp(ctx, h.rows, h.cols);
    qgemm(ctx, QLRA_OP_N, QLRA_OP_N, 1.0, h, mm.v, 0.0, tmp.v);
    copy_qmat(ctx, tmp.v, hout);
  } else {
    qgemm(ctx, QLRA_OP_N, QLRA_OP_N, 1.0, h, mm.v, 0.0, hout);
  }
}

// Least squares X = argmin ||P X - B|| for replicated P (l x s, l >= s),
// B (l x n), through a QR of P as the reference does (ColPivHouseholderQR,
// complex_bridge.cpp:80-90): P = Q R by CholeskyQR2 (shifted CholeskyQR3 if
// needed), T = Q R^{-*} (small), X = T^* B = R^{-1} Q^* B -- one wide product.
// Accuracy ~ u kappa(P) like a Householder solve (no normal equations).
DevQMat lstsq_operator(Ctx& ctx, const QView& p);
void lstsq(Ctx& ctx, const QView& p, const QView& b, const QView& x) {
  DevQMat t = lstsq_operator(ctx, p);
  qgemm(ctx, QLRA_OP_C, QLRA_OP_N, 1.0, t.v, b, 0.0, x);
}
// T (l x s) with argmin ||P X - B|| = T^* B.
DevQMat lstsq_operator(Ctx& ctx, const QView& p) {
  const int64_t s = p.cols, l = p.rows;
  DevQMat q(ctx, l, s), rinv;
  std::vector<double> rd;
  // Rank test of ColPivHouseholderQR, |r_min| > 1e-14 |r_max|
  // (complex_bridge.cpp:80-85), on the diagonal of R.
  if (!cholesky_qr(ctx, p, q.v, /*complex_mode=*/false, l, &rd, /*distributed=*/false, &rinv))
    fail(QLRA_ERR_SINGULAR, "solve_quaternion_linear: rank-deficient system",
         std::numeric_limits<double>::infinity());
  double rmax = 0.0, rmin = std::numeric_limits<double>::infinity();
  for (double v : rd) {
    rmax = std::max(rmax, std::fabs(v));
    rmin = std::min(rmin, std::fabs(v));
  }
  if (!(rmin > 1e-14 * rmax))
    fail(QLRA_ERR_SINGULAR, "solve_quaternion_linear: rank-deficient system",
         rmin > 0 ? rmax / rmin : std::numeric_limits<double>::infinity());
  DevQMat t(ctx, l, s);
  qgemm(ctx, QLRA_OP_N, QLRA_OP_C, 1.0, q.v, rinv.v, 0.0, t.v);
  return t;
}

// Launches below go to stream `s` (and its own split-K counters) until the
// guard ends; stream-ordered buffers created meanwhile live on `s`.
struct StreamSwap {
  Ctx& c;
  cudaStream_t saved;
  StreamSwap(Ctx& ctx, cudaStream_t s) : c(ctx), saved(ctx.stream) {
    c.stream = s;
    std::swap(c.tile_cnt, c.tile_cnt2);
    std::swap(c.tile_cnt_n, c.tile_cnt2_n);
  }
  ~StreamSwap() {
    std::swap(c.tile_cnt, c.tile_cnt2);
    std::swap(c.tile_cnt_n, c.tile_cnt2_n);
    c.stream = saved;
  }
};

// The core solve started inside pseudo-QR.  H = Q0 C_k with Q0 = base *
// rinv_last orthonormal (pseudo_qr_dev), so P = Psi H = P0 C_k with
// P0 = Psi Q0, and X = P^+ W = C_k^{-1} X0, X0 = P0^+ W.  X0 (Psi, the tall
// product, CholeskyQR2 of P0 and the wide product) runs on a second stream
// while the s x s pseudo-QR work runs on the main one; the close is
// X = (C_k^* C_k)^{-1} C_k^* X0 through the normal equations of the small
// C_k, whose condition number is kappa_after (exact, by the spectral map),
// taken only when kappa_after <= kEarlyKappaMax (error ~ u kappa^2 <= 1e-12
// relative).  Otherwise -- and whenever P0's factorisation or rank test is
// not clean -- the sequential solve runs and raises what it raises.
constexpr double kEarlyKappaMax = 100.0;
struct EarlySolve {
  Ctx* c = nullptr;
  const qlra_spec_t* psi = nullptr;
  int64_t row0 = 0;
  QView w{};
  // set by the one-pass entries, whose Y = A Omega and W = Psi A come from
  // the same A in the same call: then Psi Y = W Omega (below)
  const qlra_spec_t* omega = nullptr;
  bool started = false;
  DeferredQ q0;     // Q0 = base * rinv_last (read by both streams)
  Cqr2Pending cqr;  // P0 = Q_p R_p
  DevQMat x0;       // P0^+ W (s x n)
  DevQMat ck;       // C_k
  DevQMat coef;     // rinv_last C_k (H = base coef, formed on the second stream)
  DevQMat rinv;     // R1^{-1} R2^{-1} (the W Omega route; copied on main before the fork)
  double kappa = std::numeric_limits<double>::infinity();
  // x0_ready: X0 done; done: everything on the second stream (X0, then H)
  cudaEvent_t x0_ready = nullptr, coef_ready = nullptr, done = nullptr;
  EarlySolve(Ctx& ctx, const qlra_spec_t& p, int64_t r0, const QView& wv) : c(&ctx), psi(&p), row0(r0), w(wv) {}
  // main waits for the second stream (before anything it uses is freed)
  void join() {
    if (done) QLRA_CUDA(cudaStreamWaitEvent(c->stream, done, 0));
  }
  ~EarlySolve() {
    if (done) cudaStreamWaitEvent(c->stream, done, 0);
    for (cudaEvent_t e : {x0_ready, coef_ready, done})
      if (e) cudaEventDestroy(e);
  }
  EarlySolve(const EarlySolve&) = delete;
  EarlySolve& operator=(const EarlySolve&) = delete;
};

// Psi Y = W Omega is used for P0 when n <= rows / 2 (the product over n
// instead of over the local rows; C5: 80 x 300 x 40 instead of the 6.9 ms
// 80 x 2097152 x 40 Psi Q0).  P0 = (W Omega) R^{-1} with R^{-1} = R1^{-1}
// R2^{-1} the chained CholeskyQR2 inverse; it differs from Psi (Y R1^{-1})
// R2^{-1} by rounding of the order u kappa(Y) relative, the same order as
// the explicit product's own (T1 = Y R1^{-1} carries that error).
bool womega_applies(const EarlySolve& es, int64_t rows) {
  static const bool off = std::getenv("QLRA_NO_WOMEGA") != nullptr;
  return es.omega && !off && 2 * es.w.cols <= rows;
}

void early_solve_start(Ctx& c, EarlySolve& es, const DeferredQ& q0, const QView& rinv_full) {
  const int64_t s = q0.base.v.cols, rows = q0.base.v.rows, l = es.psi->rows, n = es.w.cols;
  if (!c.side2) {
    int lo = 0, hi = 0;
    QLRA_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    QLRA_CUDA(cudaStreamCreateWithPriority(&c.side2, cudaStreamNonBlocking, lo));  // lowest priority
  }
  es.x0 = DevQMat(c, s, n);  // crosses streams: allocated on main before the fork
  const bool wom = womega_applies(es, rows);
  if (wom) {
    es.rinv = DevQMat(c, s, s);
    copy_qmat(c, rinv_full, es.rinv.v);
  }
  cudaEvent_t fork = nullptr;
  QLRA_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  QLRA_CUDA(cudaEventCreateWithFlags(&es.done, cudaEventDisableTiming));
  QLRA_CUDA(cudaEventCreateWithFlags(&es.x0_ready, cudaEventDisableTiming));
  QLRA_CUDA(cudaEventCreateWithFlags(&es.coef_ready, cudaEventDisableTiming));
  QLRA_CUDA(cudaEventRecord(fork, c.stream));
  QLRA_CUDA(cudaStreamWaitEvent(c.side2, fork, 0));
  QLRA_CUDA(cudaEventDestroy(fork));
  {
    StreamSwap on(c, c.side2);
    DevQMat ps_tmp, pb(c, l, s), p0(c, l, s);
    if (wom) {
      DevQMat om(c, n, s);
      launch_gen(c.stream, *es.omega, 0, 0, n, s, om.v, false);
      qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, es.w, om.v, 0.0, pb.v);  // Psi Y
      qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, pb.v, es.rinv.v, 0.0, p0.v);
    } else {
      if (!psi8_gemm(c, *es.psi, es.row0, q0.base.v, pb.v)) {
        const QView ps = psi_for_solve(c, *es.psi, es.row0, rows, ps_tmp);
        qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, ps, q0.base.v, 0.0, pb.v);
      }
      qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, pb.v, q0.rinv_last.v, 0.0, p0.v);
    }
    cqr2_enqueue(c, p0.v, QView{}, /*complex_mode=*/false, /*distributed=*/false, nullptr, /*form_q=*/false,
                 es.cqr);
    // X0 = R_p^{-1} Q_p^* W with Q_p = t1 R2^{-1}, R_p^{-1} = R1^{-1} R2^{-1}:
    // T0 = t1 (R2^{-1} (R1^{-1} R2^{-1})^*), X0 = T0^* W
    DevQMat rinv(c, s, s), mm(c, s, s), t0(c, l, s);
    qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, es.cqr.r1inv.v, es.cqr.r2inv.v, 0.0, rinv.v);
    qgemm(c, QLRA_OP_N, QLRA_OP_C, 1.0, es.cqr.r2inv.v, rinv.v, 0.0, mm.v);
    qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, es.cqr.t1.v, mm.v, 0.0, t0.v);
    qgemm(c, QLRA_OP_C, QLRA_OP_N, 1.0, t0.v, es.w, 0.0, es.x0.v);
  }
  QLRA_CUDA(cudaEventRecord(es.x0_ready, c.side2));
  QLRA_CUDA(cudaEventRecord(es.done, c.side2));
  es.started = true;
}

// X = C_k^{-1} X0 expressed as X = Z X0 (Z = (C_k^* C_k)^{-1} C_k^*, s x s).
// False (nothing usable) unless every condition of the early path holds.
bool early_solve_close(Ctx& c, EarlySolve& es, DevQMat& z) {
  if (!es.started) return false;
  QLRA_CUDA(cudaStreamWaitEvent(c.stream, es.x0_ready, 0));
  if (!(es.kappa <= kEarlyKappaMax) || !es.ck.buf.ptr) return false;
  const int64_t s = es.ck.v.rows;
  DevQMat g(c, s, s), r(c, s, s), ri(c, s, s), ginv(c, s, s);
  DeviceBuffer info(c, sizeof(int)), dg(c, sizeof(double) * (size_t)s);
  qgemm(c, QLRA_OP_C, QLRA_OP_N, 1.0, es.ck.v, es.ck.v, 0.0, g.v);
  chol_inv_any(c, g.v, r.v, ri.v, info.as<int>(), dg.as<double>());
  qgemm(c, QLRA_OP_N, QLRA_OP_C, 1.0, ri.v, ri.v, 0.0, ginv.v);
  z = DevQMat(c, s, s);
  qgemm(c, QLRA_OP_N, QLRA_OP_C, 1.0, ginv.v, es.ck.v, 0.0, z.v);
  int inf = 0;
  QLRA_CUDA(cudaMemcpyAsync(&inf, info.ptr, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  std::vector<double> rd;
  if (cqr2_status(c, es.cqr, &rd) != 0 || inf != 0) return false;  // (one sync: the status read)
  double rmax = 0.0, rmin = std::numeric_limits<double>::infinity();
  for (double v : rd) {
    rmax = std::max(rmax, std::fabs(v));
    rmin = std::min(rmin, std::fabs(v));
  }
  // P0's rank test with margin; borderline systems take the sequential
  // solve and its exact rank test (|r_min| > 1e-14 |r_max| on R of P)
  return rmin > 1e-10 * rmax;
}

// X = op(T) B over column blocks: the sequential solve (T (l x s), X = T^* W)
// or the early one (Z (s x s), X = Z X0).
struct CoreSolve {
  DevQMat t;
  bool adj = true;
  DevQMat b_own;
  QView b{};
  void cols(Ctx& c, int64_t j0, int64_t nj, const QView& x) const {
    qgemm(c, adj ? QLRA_OP_C : QLRA_OP_N, QLRA_OP_N, 1.0, t.v, sub(b, 0, j0, b.rows, nj), 0.0,
          sub(x, 0, j0, x.rows, nj));
  }
};

// ------------------------------------------------- rangefinders, solve ---
// Device bodies of pseudo_qr / pseudo_svd / qb_solve (Y, H row-sharded over
// the ranks; shapes validated by the callers).
// pseudo-QR's two factorisations for s <= the single-launch Cholesky limit:
// Y = Q0 R_q (quaternion CholeskyQR2, Q0 deferred) and R_q = C R_c (complex
// CholeskyQR2).  The complex pass-1 factor is the Cholesky factor of the
// complex part of R_q^* R_q = Y^* Y, so it is taken from the quaternion
// pass-1 Gram on the side stream while quaternion pass 2 runs; pass 2 on
// R_q R1c^{-1} removes its error as usual.  False if quaternion pass 1 broke
// down (the caller takes the general path); a complex breakdown reruns the
// complex CholeskyQR2 of R_q the general way.
bool pqr_factors_fast(Ctx& c, const QView& Y, DeferredQ& q0, DevQMat& rq, DevQMat& rq_inv, DevQMat& cm,
                      DevQMat& rc, std::vector<double>& rd, EarlySolve* es) {
  const int64_t s = Y.cols;
  if (!c.side) QLRA_CUDA(create_main_stream(&c.side));
  DevQMat gy(c, s, s), gc(c, s, s), r1c(c, s, s), r1c_inv(c, s, s);
  DeviceBuffer info_c(c, 2 * sizeof(int)), dg_c(c, 2 * sizeof(double) * (size_t)s);
  gram(c, Y, gy.v);
  copy_qmat(c, gy.v, gc.v);
  zero_jk_planes(c, gc.v);
  cudaEvent_t fork = nullptr, cdone = nullptr;
  QLRA_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  QLRA_CUDA(cudaEventCreateWithFlags(&cdone, cudaEventDisableTiming));
  QLRA_CUDA(cudaEventRecord(fork, c.stream));
  QLRA_CUDA(cudaStreamWaitEvent(c.side, fork, 0));
  const bool side_chol = s <= chol_inv_async_max();
  if (side_chol) {
    const cudaStream_t main = c.stream;
    c.stream = c.side;  // one launch, no split-K counters involved
    try {
      chol_inv_launch(c, gc.v, r1c.v, r1c_inv.v, info_c.as<int>(), dg_c.as<double>());
    } catch (...) {
      c.stream = main;
      throw;
    }
    c.stream = main;
  }
  QLRA_CUDA(cudaEventRecord(cdone, c.side));
  QLRA_CUDA(cudaEventDestroy(fork));
  struct Join {  // main waits for the side launch before its buffers are used or freed
    Ctx& c;
    cudaEvent_t e;
    ~Join() {
      cudaStreamWaitEvent(c.stream, e, 0);
      cudaEventDestroy(e);
    }
  } join{c, cdone};
  Cqr2Pending p;
  cqr2_enqueue(c, Y, QView{}, /*complex_mode=*/false, /*distributed=*/true, &gy.v, /*form_q=*/false, p);
  if (cqr2_status(c, p, nullptr) != 0) return false;
  rq = std::move(p.r1);
  chain_r(c, rq, p.r2.v);
  rq_inv = std::move(p.r1inv);
  chain_rinv(c, rq_inv, p.r2inv.v);
  q0.base = std::move(p.t1);
  q0.rinv_last = std::move(p.r2inv);
  if (es && c.nranks == 1 && es->psi->rows >= s && !std::getenv("QLRA_NO_EARLY_SOLVE"))
    early_solve_start(c, *es, q0, rq_inv.v);
  QLRA_CUDA(cudaStreamWaitEvent(c.stream, cdone, 0));
  // (s past the single-launch Cholesky: the blocked form needs the main
  // stream's split-K counters, so the complex pass-1 factor is taken here)
  if (!side_chol) chol_inv_any(c, gc.v, r1c.v, r1c_inv.v, info_c.as<int>(), dg_c.as<double>());
  DevQMat t1c(c, s, s), g2(c, s, s), r2c(c, s, s), r2c_inv(c, s, s);
  qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, rq.v, r1c_inv.v, 0.0, t1c.v);
  qgemm(c, QLRA_OP_C, QLRA_OP_N, 1.0, t1c.v, t1c.v, 0.0, g2.v);
  zero_jk_planes(c, g2.v);
  chol_inv_any(c, g2.v, r2c.v, r2c_inv.v, info_c.as<int>() + 1, dg_c.as<double>() + s);
  qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, t1c.v, r2c_inv.v, 0.0, cm.v);
  int inf[2] = {0, 0};
  std::vector<double> d((size_t)(2 * s));
  QLRA_CUDA(cudaMemcpyAsync(inf, info_c.ptr, 2 * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  QLRA_CUDA(cudaMemcpyAsync(d.data(), dg_c.ptr, 2 * sizeof(double) * (size_t)s, cudaMemcpyDeviceToHost, c.stream));
  QLRA_CUDA(cudaStreamSynchronize(c.stream));
  if (inf[0] != 0 || inf[1] != 0) {
    if (!cholesky_qr(c, rq.v, cm.v, /*complex_mode=*/true, s, &rd, /*distributed=*/false, nullptr, &rc))
      fail(QLRA_ERR_RANK, "pseudo_qr: sketch numerically rank-deficient; use pseudo_svd");
    return true;
  }
  rd.resize((size_t)s);
  for (int64_t k = 0; k < s; ++k) rd[k] = d[k] * d[s + k];
  rc = std::move(r1c);
  chain_r(c, rc, r2c.v);
  return true;
}

void pseudo_qr_dev(Ctx& c, const QView& Y, const QView& H, const qlra_pseudo_qr_config_t& cfg,
                   qlra_rangefinder_report_t* rep, EarlySolve* es = nullptr) {
  const int64_t s = Y.cols;
  const int64_t m = global_rows(c, Y.rows);
  if (m <= s) fail(QLRA_ERR_PARAMETER, "pseudo_qr: sketch must be tall (rows > cols)");
  if (cfg.max_correction_steps < 0) fail(QLRA_ERR_PARAMETER, "pseudo_qr: negative correction step count");
  if (!(cfg.delta_budget >= 1.0 && cfg.delta_budget <= std::sqrt(7.0) / 2.0 + 1e-12))
    fail(QLRA_ERR_PARAMETER, "pseudo_qr: delta_budget outside [1, sqrt(7)/2]");
  // Y = Q0 R_q by quaternion CholeskyQR2 -- the only factorisation of the
  // tall sketch.  Writing Y = Q0 R_q in compact form, compact(Y) =
  // U compact(R_q) with U (2m x 2s) the compact image of Q0, orthonormal
  // columns; so the reference's complex_qr(to_compact(Y))
  // (rangefinders.cpp:117) has the R factor R_c of compact(R_q), and its
  // basis is H0 = Q0 C with C = R_q R_c^{-1}: a complex-mode CholeskyQR2 of
  // the small s x s R_q.  Every correction step then acts on the s x s
  // coefficient matrix (H_k = Q0 C_k, kappa(H_k) = kappa(C_k) because Q0 is
  // orthonormal), and one tall product H = Q0 C_k closes the pass.  H lies in
  // range(Q0) = range(H0) to rounding, which is what the reference's
  // re-projection (rangefinders.cpp:142-153) restores.
  // Q0 itself is never formed: Q0 = base * rinv_last, and the pass closes
  // with H = base * (rinv_last * C_k) -- one tall product fewer, same
  // accuracy (rinv_last is the well-conditioned last CholeskyQR factor).
  DevQMat rq, rq_inv;
  DeferredQ q0_local;
  // with an early solve, q0 is read by the second stream: the EarlySolve owns
  // it (freed after its final join)
  DeferredQ& q0 = es ? es->q0 : q0_local;
  DevQMat cm(c, s, s), rc;
  std::vector<double> rd;
  if (!pqr_factors_fast(c, Y, q0, rq, rq_inv, cm, rc, rd, es)) {
    if (!cholesky_qr(c, Y, QView{}, /*complex_mode=*/false, m, nullptr, /*distributed=*/true, &rq_inv, &rq, &q0))
      fail(QLRA_ERR_RANK, "pseudo_qr: sketch numerically rank-deficient; use pseudo_svd");
    if (!cholesky_qr(c, rq.v, cm.v, /*complex_mode=*/true, s, &rd, /*distributed=*/false, nullptr, &rc))
      fail(QLRA_ERR_RANK, "pseudo_qr: sketch numerically rank-deficient; use pseudo_svd");
  }
  rank_check(rd);  // |diag R_c|, rangefinders.cpp:118-126
  qlra_rangefinder_report_t r{};
  r.method = QLRA_PSEUDO_QR;
  DevQMat g(c, s, s), mk(c, s, s);
  qgemm(c, QLRA_OP_C, QLRA_OP_N, 1.0, cm.v, cm.v, 0.0, g.v);  // H0^* H0 = C^* C
  // All eigenvalues of G_0 once.  M_k = (1-eps) I + eps G_k^{-1} is a function
  // of G_k, so G_{k+1} = M_k G_k M_k has the eigenvalues
  // lambda ((1-eps) + eps / lambda)^2: kappa(H_k) after every correction step
  // follows from G_0's spectrum (exact identity; the reference recomputes it
  // from H_k, rangefinders.cpp:136, which agrees to rounding).
  //
  // G_0's spectrum is computed on a side stream while the first two
  // correction steps (inverse, epsilon and the next coefficient matrix) are
  // computed speculatively here (almost every sketch needs them); they are
  // discarded where kappa says stop, and any error they raised surfaces only
  // where the sequential order would raise it.
  struct Spec {
    bool ok = false;
    int code = 0;
    std::string msg;
    double cond = 0.0;
    double eps = 0.0;
    DevQMat gk;    // G_k = C_k^* C_k (k >= 1; G_0 is g)
    DevQMat ginv;  // G_k^{-1}
    DevQMat next;  // C_{k+1} = C_k ((1-eps) I + eps G_k^{-1})
  };
  Spec spec[2];
  const int nspec = std::min(2, cfg.max_correction_steps);
  std::vector<double> lam;
  // One correction step on the coefficient matrix: G = C^*C, its inverse,
  // estimate_epsilon's power iteration and rcond test, correction_step's
  // solve test, then the next coefficient matrix (rangefinders.cpp:66-105).
  auto step = [&](const QView& ck, const QView& gk, DevQMat& ginv, DevQMat& next) -> double {
    double rc = 0.0;
    const double eps = estimate_epsilon_rc(c, gk, ginv.v, cfg.power_iters_for_epsilon, &rc);
    check_solve_rc(rc);
    if (!(eps > 0.0 && eps < 1.0)) fail(QLRA_ERR_PARAMETER, "correction_step: epsilon must lie in (0,1)");
    // H_{k+1} = H_k ((1-eps) I + eps G_k^{-1})  (rangefinders.cpp:99-105)
    small_axpby_identity(c, 1.0 - eps, eps, ginv.v, mk.v);
    next = DevQMat(c, s, s);
    qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, ck, mk.v, 0.0, next.v);
    return eps;
  };
  {
    SideEigs eig(c, g.v);
    for (int k = 0; k < nspec; ++k) {
      Spec& sp = spec[k];
      try {
        sp.ginv = DevQMat(c, s, s);
        const QView ck = k == 0 ? cm.v : spec[0].next.v;
        DevQMat& gk = sp.gk;
        if (k == 0) {
          // G_0^{-1} from the factors already at hand: C = R_q R_c^{-1}, so
          // G_0^{-1} = K K^* with K = R_c R_q^{-1} (no factorisation; the
          // reference's singularity tests are applied from its rcond below)
          DevQMat kf(c, s, s);
          qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, rc.v, rq_inv.v, 0.0, kf.v);
          qgemm(c, QLRA_OP_N, QLRA_OP_C, 1.0, kf.v, kf.v, 0.0, sp.ginv.v);
        } else {
          gk = DevQMat(c, s, s);
          qgemm(c, QLRA_OP_C, QLRA_OP_N, 1.0, ck, ck, 0.0, gk.v);
          if (!hpd_inverse(c, gk.v, sp.ginv.v, nullptr))
            fail(QLRA_ERR_SINGULAR, "estimate_epsilon: H*H numerically singular",
                 std::numeric_limits<double>::infinity());
        }
        sp.eps = step(ck, k == 0 ? g.v : gk.v, sp.ginv, sp.next);
        sp.ok = true;
      } catch (const Status& e) {
        // only the numerical outcomes of the sequential flow are deferred
        if (e.code != QLRA_ERR_SINGULAR && e.code != QLRA_ERR_PARAMETER) throw;
        sp.code = e.code;
        sp.msg = e.what();
        sp.cond = e.cond;
        break;
      }
    }
    lam = eig.get();
  }
  // G_0's small eigenvalues carry ~u kappa^2 relative error; refine them from
  // G_0^{-1} = K K^* (formed without squaring kappa) when it matters
  if (kappa_from_eigs(lam) > kRefineKappa && nspec > 0 && spec[0].ginv.buf.ptr)
    lam = merge_spectra(lam, quat_eigs(c, spec[0].ginv.v, /*extremes_only=*/false));
  r.kappa_before = kappa_from_eigs(lam);
  double kappa = r.kappa_before;
  if (std::getenv("QLRA_DEBUG_PQR")) {
    std::fprintf(stderr, "[pqr] s=%lld kappa0=%.6e lam=[%.3e..%.3e] rd=[%.3e..%.3e]", (long long)s, kappa,
                 lam.empty() ? 0.0 : lam.back(), lam.empty() ? 0.0 : lam.front(),
                 *std::min_element(rd.begin(), rd.end()), *std::max_element(rd.begin(), rd.end()));
    for (int k = 0; k < nspec; ++k)
      std::fprintf(stderr, " spec%d ok=%d eps=%.6e code=%d %s", k, (int)spec[k].ok, spec[k].eps, spec[k].code,
                   spec[k].msg.c_str());
    std::fprintf(stderr, "\n");
  }
  try {
    while (r.correction_steps_used < cfg.max_correction_steps && kappa > kKappaTarget) {
      // one inverse serves estimate_epsilon and correction_step (both
      // factor the same H^*H, rangefinders.cpp:68,102)
      const int k = r.correction_steps_used;
      double eps = 0.0;
      if (k < nspec) {
        Spec& sp = spec[k];
        if (!sp.ok) fail(sp.code, sp.msg, sp.cond);
        eps = sp.eps;
        cm = std::move(sp.next);
      } else {
        qgemm(c, QLRA_OP_C, QLRA_OP_N, 1.0, cm.v, cm.v, 0.0, g.v);
        DevQMat ginv(c, s, s), cn;
        if (!hpd_inverse(c, g.v, ginv.v, nullptr))
          fail(QLRA_ERR_SINGULAR, "estimate_epsilon: H*H numerically singular",
               std::numeric_limits<double>::infinity());
        eps = step(cm.v, g.v, ginv, cn);
        cm = std::move(cn);
      }
      double lmax = 0.0, lmin = std::numeric_limits<double>::infinity();
      for (double& v : lam) {
        const double f = (1.0 - eps) + eps / v;
        v = v * f * f;
        lmax = std::max(lmax, v);
        lmin = std::min(lmin, v);
      }
      kappa = lmin > 0.0 ? std::sqrt(lmax / lmin) : std::numeric_limits<double>::infinity();
      ++r.correction_steps_used;
    }
  } catch (const Status& e) {
    if (e.code != QLRA_ERR_SINGULAR) throw;
    fail(QLRA_ERR_RANK, "pseudo_qr: sketch numerically rank-deficient; use pseudo_svd");
  }
  r.kappa_after = kappa;
  if (es && es->started) {
    // H = base (rinv_last C_k) on the second stream, overlapping the close
    // of the early solve on this one (EarlySolve::done covers it)
    es->coef = DevQMat(c, s, s);
    qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, q0.rinv_last.v, cm.v, 0.0, es->coef.v);
    es->ck = std::move(cm);
    es->kappa = kappa;
    QLRA_CUDA(cudaEventRecord(es->coef_ready, c.stream));
    QLRA_CUDA(cudaStreamWaitEvent(c.side2, es->coef_ready, 0));
    {
      StreamSwap on(c, c.side2);
      qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, q0.base.v, es->coef.v, 0.0, H);
    }
    QLRA_CUDA(cudaEventRecord(es->done, c.side2));
  } else {
    DevQMat coef(c, s, s);
    qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, q0.rinv_last.v, cm.v, 0.0, coef.v);
    qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, q0.base.v, coef.v, 0.0, H);
  }
  if (rep) *rep = r;
}

// kappa_after_async (optional): leave kappa(H) to the caller as a pending
// side-stream eigenvalue computation instead of waiting for it here.
// range_only: orthonormal_range (rangefinders.cpp:160-164: rows >= cols
// allowed, no report).
// pseudo-SVD's report computations left to the caller: the refinement of
// kappa(Y) and kappa(H) run on the side stream while the caller's next work
// (the core solve) runs; finish() fills the report.
struct PsvdDeferred {
  std::vector<double> lam;          // spectrum of Y^*Y
  std::unique_ptr<SideEigs> refine;  // of (R^*R)^{-1}: kappa(Y) to ~u kappa(Y)
  std::unique_ptr<SideEigs> after;   // of H^*H: kappa(H)
  void finish(qlra_rangefinder_report_t* rep) {
    if (!rep) return;
    if (refine) rep->kappa_before = kappa_from_eigs(merge_spectra(lam, refine->get()));
    if (after) rep->kappa_after = kappa_from_eigs(after->get());
    refine.reset();
    after.reset();
  }
};

void pseudo_svd_dev(Ctx& c, const QView& Y, const QView& H, uint64_t seed, qlra_rangefinder_report_t* rep,
                    PsvdDeferred* deferred = nullptr, bool range_only = false) {
  const int64_t s = Y.cols;
  const int64_t m = global_rows(c, Y.rows);
  if (range_only) {
    if (m < s) fail(QLRA_ERR_PARAMETER, "orthonormal_range: requires rows >= cols");
  } else if (m <= s) {
    fail(QLRA_ERR_PARAMETER, "pseudo_svd: sketch must be tall (rows > cols)");
  }
  if (s == 0) return;
  qlra_rangefinder_report_t r{};
  r.method = QLRA_PSEUDO_SVD;
  // Full-rank sketches: quaternion CholeskyQR2 (shifted CholeskyQR3 when
  // needed).  Others: graded eigen route + orthonormal completion.
  // kappa(Y) comes from the eigenvalues of the same Gram CholeskyQR2 starts
  // from, computed on the side stream while CholeskyQR2 runs; a non-finite
  // kappa (kappa^2 past 1/u) or a CholeskyQR breakdown takes the graded route.
  DevQMat g(c, s, s), rinv;
  gram(c, Y, g.v);
  bool qr_ok = false;
  std::vector<double> lam;
  {
    SideEigs eig(c, g.v);
    qr_ok = cholesky_qr(c, Y, H, /*complex_mode=*/false, m, nullptr, /*distributed=*/true, &rinv, nullptr,
                        nullptr, &g.v);
    lam = eig.get();
  }
  r.kappa_before = kappa_from_eigs(lam);
  static const bool force_graded = [] {  // QLRA_PSVD_GRADED=1: A/B of the graded route only
    const char* e = std::getenv("QLRA_PSVD_GRADED");
    return e && std::atoi(e) != 0;
  }();
  if (!std::isfinite(r.kappa_before) || !qr_ok) {
    r.kappa_before = pseudo_svd_graded(c, Y, H, m, global_row0(c, Y.rows), seed);
  } else {
    // Past kappa(Y) ~ 1e6 the CholeskyQR2 basis is still orthonormal and
    // spans range(Y) to ~u kappa(Y), like any backward-stable method, but
    // its error is shaped by the product Y R^{-1}: at C3 (kappa 6e7) its QB
    // error differs from the reference's (SVD basis) by 8e-10 relative where
    // two runs of the reference differ by <1e-10.  The graded route (Gram
    // eigenvectors in levels, re-projected) lands within 5e-11 of it
    // (tools/diag_c3_psvd.py): take it there.
    const bool graded = r.kappa_before > kGradedKappa || force_graded;
    if (r.kappa_before > kRefineKappa && !range_only) {  // kappa(Y) to ~u kappa(Y), not u kappa(Y)^2
      if (deferred) {
        DevQMat pm(c, s, s);
        qgemm(c, QLRA_OP_N, QLRA_OP_C, 1.0, rinv.v, rinv.v, 0.0, pm.v);  // (R^* R)^{-1}
        deferred->lam = lam;
        deferred->refine.reset(new SideEigs(c, pm.v));
      } else {
        r.kappa_before = kappa_from_eigs(refine_with_rinv(c, lam, rinv.v));
      }
    }
    if (graded) pseudo_svd_graded(c, Y, H, m, global_row0(c, Y.rows), seed);
  }
  if (range_only) return;
  if (deferred) {
    // kappa(H)'s eigenvalues overlap the caller's next work
    DevQMat gh(c, s, s);
    gram(c, H, gh.v);
    deferred->after.reset(new SideEigs(c, gh.v));
  } else {
    r.kappa_after = condition_number_dev(c, H);
  }
  if (rep) *rep = r;
}

// The core solve's operator T (l x s): X = T^* W (qb_stage_with_psi,
// sketching.cpp:184-185: P = Psi H, X = P \ W through a QR of P).
DevQMat qb_solve_operator(Ctx& c, const qlra_spec_t& psi, int64_t row0, const QView& H) {
  const int64_t s = H.cols, l = psi.rows;
  DevQMat ps_tmp;
  DevQMat p(c, l, s);
  if (!psi8_gemm(c, psi, row0, H, p.v)) {
    const QView ps = psi_for_solve(c, psi, row0, H.rows, ps_tmp);
    qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, ps, H, 0.0, p.v);
  }
  allreduce_qmat(c, p.v);
  return lstsq_operator(c, p.v);
}
void qb_solve_dev(Ctx& c, const qlra_spec_t& psi, int64_t row0, const QView& H, const QView& W, const QView& X) {
  DevQMat t = qb_solve_operator(c, psi, row0, H);
  qgemm(c, QLRA_OP_C, QLRA_OP_N, 1.0, t.v, W, 0.0, X);
}
// The QB stage's core solve after a rangefinder that may have started it early.
CoreSolve core_solve(Ctx& c, EarlySolve* es, const qlra_spec_t& psi, int64_t row0, const QView& H,
                     const QView& W) {
  CoreSolve cs;
  if (es && early_solve_close(c, *es, cs.t)) {
    cs.adj = false;
    cs.b_own = std::move(es->x0);
    cs.b = cs.b_own.v;
    return cs;
  }
  if (es) es->join();  // H may come from the second stream
  cs.t = qb_solve_operator(c, psi, row0, H);
  cs.adj = true;
  cs.b = W;
  return cs;
}

void check_view(const qlra_qmat_t* m, const char* who) {
  if (!m) fail(QLRA_ERR_PARAMETER, std::string(who) + ": null matrix");
  if (m->rows < 0 || m->cols < 0 || m->ld < m->cols)
    fail(QLRA_ERR_SHAPE, std::string(who) + ": bad matrix view");
}

void validate_spec(const qlra_spec_t* s) {
  if (!s) fail(QLRA_ERR_PARAMETER, "test matrix: null spec");
  if (s->rows < 0 || s->cols < 0) fail(QLRA_ERR_PARAMETER, "test matrix: negative dims");
  if (!(s->density > 0.0 && s->density <= 1.0))
    fail(QLRA_ERR_PARAMETER, "test matrix: density must lie in (0,1]");
  if (s->kind < 0 || s->kind > 3) fail(QLRA_ERR_PARAMETER, "test matrix: unknown kind");
}

}  // namespace
}  // namespace qlra_dev

using namespace qlra_dev;

// The device's stream-ordered pool: no release to the driver between calls,
// and no reuse of a block freed on ANOTHER stream that is not yet complete
// (by default the pool would make this stream wait for that one -- it
// serialised the pseudo-QR close on the main stream behind the closing tall
// product on the second stream, 4 ms at C4).  Reuse of completed frees stays.
static void setup_pool(int device) {
  cudaMemPool_t pool;
  QLRA_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = UINT64_MAX;
  QLRA_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  int no = 0;
  QLRA_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no));
}

template <class F>
static int guarded(qlra_ctx_t* ctx, F&& f) {
  try {
    if (!ctx) return QLRA_ERR_PARAMETER;
    QLRA_CUDA(cudaSetDevice(ctx->c.device));
    f(ctx->c);
    return QLRA_OK;
  } catch (const Status& s) {
    ctx->c.last_error = s.what();
    ctx->c.last_cond = s.cond;
    return s.code;
  } catch (const std::exception& e) {
    ctx->c.last_error = e.what();
    return QLRA_ERR_INTERNAL;
  }
}

extern "C" {

int qlra_nccl_unique_id(void* out) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return QLRA_ERR_NCCL;
  std::memcpy(out, &id, sizeof(id));
  return QLRA_OK;
}

int qlra_ctx_create(qlra_ctx_t** out, int device, int rank, int nranks, const void* nccl_id) {
  if (!out) return QLRA_ERR_PARAMETER;
  *out = nullptr;
  qlra_ctx_t* ctx = new qlra_ctx_t();
  ctx->c.device = device;
  ctx->c.rank = rank;
  ctx->c.nranks = nranks < 1 ? 1 : nranks;
  const int rc = guarded(ctx, [&](Ctx& c) {
    QLRA_CUDA(create_main_stream(&c.stream));
    c.own_stream = true;
    setup_pool(device);
    QLRA_CUDA(cudaMallocHost(&c.pinned, 4096));
    if (c.nranks > 1) {
      if (!nccl_id) fail(QLRA_ERR_PARAMETER, "qlra_ctx_create: nranks > 1 needs an NCCL id");
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      const ncclResult_t r = ncclCommInitRank(&c.comm, c.nranks, id, rank);
      if (r != ncclSuccess) fail(QLRA_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
  });
  if (rc != QLRA_OK) {
    delete ctx;
    return rc;
  }
  *out = ctx;
  return QLRA_OK;
}

int qlra_ctx_create_local(qlra_ctx_t** out, int device, qlra_group_t* group, int rank) {
  if (!out) return QLRA_ERR_PARAMETER;
  *out = nullptr;
  qlra_ctx_t* ctx = new qlra_ctx_t();
  ctx->c.device = device;
  const int rc = guarded(ctx, [&](Ctx& c) {
    QLRA_CUDA(create_main_stream(&c.stream));
    c.own_stream = true;
    setup_pool(device);
    QLRA_CUDA(cudaMallocHost(&c.pinned, 4096));
    group_attach(c, group, rank);
  });
  if (rc != QLRA_OK) {
    if (ctx->c.stream) cudaStreamDestroy(ctx->c.stream);
    if (ctx->c.pinned) cudaFreeHost(ctx->c.pinned);
    delete ctx;
    return rc;
  }
  *out = ctx;
  return QLRA_OK;
}

static void drop_events(Ctx& c) {
  for (auto& e : c.ktimer.ev) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  c.ktimer.ev.clear();
  c.ktimer.flops = c.ktimer.a_bytes = c.ktimer.int8_ops = 0.0;
  c.ktimer.launches = 0;
  c.ktimer.engines = 0;
}

int qlra_ctx_destroy(qlra_ctx_t* ctx) {
  if (!ctx) return QLRA_OK;
  cudaSetDevice(ctx->c.device);
  if (ctx->c.stream) {
    psi_keep_release(ctx->c);
    try {
      oz_release(ctx->c);
    } catch (...) {
    }
    cudaStreamSynchronize(ctx->c.stream);
  }
  if (ctx->c.comm) ncclCommDestroy(ctx->c.comm);
  group_detach(ctx->c);
  if (ctx->c.own_stream && ctx->c.stream) cudaStreamDestroy(ctx->c.stream);
  if (ctx->c.pinned) cudaFreeHost(ctx->c.pinned);
  if (ctx->c.tile_cnt) cudaFree(ctx->c.tile_cnt);
  if (ctx->c.side) {
    cudaStreamSynchronize(ctx->c.side);
    cudaStreamDestroy(ctx->c.side);
  }
  if (ctx->c.staging) cudaFreeHost(ctx->c.staging);
  if (ctx->c.side2) {
    cudaStreamSynchronize(ctx->c.side2);
    cudaStreamDestroy(ctx->c.side2);
  }
  if (ctx->c.tile_cnt2) cudaFree(ctx->c.tile_cnt2);
  drop_events(ctx->c);
  for (auto& e : ctx->c.ktimer.pool) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  delete ctx;
  return QLRA_OK;
}

int qlra_ctx_set_stream(qlra_ctx_t* ctx, void* stream) {
  return guarded(ctx, [&](Ctx& c) {
    if (c.own_stream && c.stream) {
      QLRA_CUDA(cudaStreamSynchronize(c.stream));
      QLRA_CUDA(cudaStreamDestroy(c.stream));
      c.own_stream = false;
    }
    // Used as given; NULL is the legacy default stream (torch's default).
    c.stream = static_cast<cudaStream_t>(stream);
  });
}

int qlra_ctx_synchronize(qlra_ctx_t* ctx) {
  return guarded(ctx, [&](Ctx& c) { QLRA_CUDA(cudaStreamSynchronize(c.stream)); });
}

const char* qlra_last_error(const qlra_ctx_t* ctx, double* cond) {
  if (!ctx) return "null context";
  if (cond) *cond = ctx->c.last_cond;
  return ctx->c.last_error.c_str();
}

int64_t qlra_ctx_launch_count(const qlra_ctx_t*) { return launch_counter().load(); }

int qlra_ctx_kernel_timing(qlra_ctx_t* ctx, int enable) {
  return guarded(ctx, [&](Ctx& c) {
    drop_events(c);
    c.ktimer.on = enable != 0;
    if (c.ktimer.on)  // events for up to 256 launches created now, outside any timed region
      while (c.ktimer.pool.size() < 256) {
        cudaEvent_t a = nullptr, b = nullptr;
        QLRA_CUDA(cudaEventCreate(&a));
        QLRA_CUDA(cudaEventCreate(&b));
        c.ktimer.pool.emplace_back(a, b);
      }
  });
}

int qlra_ctx_kernel_stats(qlra_ctx_t* ctx, double* ms, int64_t* launches, double* flops,
                          double* a_bytes) {
  return guarded(ctx, [&](Ctx& c) {
    double total = 0.0;
    for (auto& e : c.ktimer.ev) {
      QLRA_CUDA(cudaEventSynchronize(e.second));
      float t = 0.f;
      QLRA_CUDA(cudaEventElapsedTime(&t, e.first, e.second));
      total += t;
    }
    if (ms) *ms = total;
    if (launches) *launches = c.ktimer.launches;
    if (flops) *flops = c.ktimer.flops;
    if (a_bytes) *a_bytes = c.ktimer.a_bytes;
  });
}

int qlra_ctx_kernel_engines(qlra_ctx_t* ctx, int* engines, double* int8_ops) {
  return guarded(ctx, [&](Ctx& c) {
    if (engines) *engines = c.ktimer.engines;
    if (int8_ops) *int8_ops = c.ktimer.int8_ops;
  });
}

int qlra_measure_int8_peak(qlra_ctx_t* ctx, double ms, double* tops) {
  return guarded(ctx, [&](Ctx& c) { *tops = oz_measure_int8_peak(c, ms); });
}

const char* qlra_int8_engine_name(void) { return oz_kernel_name(); }

int qlra_i8gemm_batched(qlra_ctx_t* ctx, int mode, int64_t m, int64_t n, int64_t k, const int8_t* a, int64_t lda,
                        int64_t stride_a, const int8_t* b, int64_t ldb, int64_t stride_b, int32_t* c_out, int64_t ldc,
                        int64_t stride_c, int batch, int beta) {
  return guarded(ctx, [&](Ctx& c) {
    i8gemm_batched(c, mode, m, n, k, a, lda, stride_a, b, ldb, stride_b, c_out, ldc, stride_c, batch, beta, c.stream);
  });
}
const char* qlra_i8gemm_kernel_name(void) { return i8gemm_kernel_name(); }

int qlra_ctx_set_sketch_engine(qlra_ctx_t* ctx, int engine) {
  return guarded(ctx, [&](Ctx& c) {
    if (engine != QLRA_SKETCH_AUTO && engine != QLRA_SKETCH_DMMA && engine != QLRA_SKETCH_INT8)
      fail(QLRA_ERR_PARAMETER, "sketch engine must be QLRA_SKETCH_AUTO, _DMMA or _INT8");
    c.sketch_engine = engine;
  });
}

int qlra_gen_test_matrix_block(qlra_ctx_t* ctx, const qlra_spec_t* spec, int64_t r0, int64_t c0,
                               qlra_qmat_t* out) {
  return guarded(ctx, [&](Ctx& c) {
    validate_spec(spec);
    check_view(out, "gen_test_matrix");
    if (r0 < 0 || c0 < 0 || r0 + out->rows > spec->rows || c0 + out->cols > spec->cols)
      fail(QLRA_ERR_SHAPE, "test matrix: block out of range");
    launch_gen(c.stream, *spec, r0, c0, out->rows, out->cols, view_of(out), false);
  });
}

int qlra_sketch_update_rows(qlra_ctx_t* ctx, const qlra_spec_t* omega, const qlra_spec_t* psi,
                            int64_t row0, const qlra_qmat_t* block, qlra_qmat_t* y_rows,
                            qlra_qmat_t* w) {
  return guarded(ctx, [&](Ctx& c) {
    validate_spec(omega);
    validate_spec(psi);
    check_view(block, "sketch_update_rows");
    check_view(y_rows, "sketch_update_rows");
    check_view(w, "sketch_update_rows");
    const int64_t n = w->cols;
    if (block->cols != n || omega->rows != n)
      fail(QLRA_ERR_SHAPE, "sketch_update_rows: column count mismatch");
    if (y_rows->rows != block->rows || y_rows->cols != omega->cols || w->rows != psi->rows)
      fail(QLRA_ERR_SHAPE, "sketch_update_rows: sketch shape mismatch");
    if (row0 < 0 || row0 + block->rows > psi->cols)
      fail(QLRA_ERR_SHAPE, "sketch_update_rows: row range out of bounds");
    sketch_update_rows(c, *omega, *psi, row0, view_of(block), view_of(y_rows), view_of(w));
  });
}

int qlra_sketch_update_rows_host(qlra_ctx_t* ctx, const qlra_spec_t* omega,
                                 const qlra_spec_t* psi, int64_t row0,
                                 const qlra_qmat_t* host_block, qlra_qmat_t* y_rows,
                                 qlra_qmat_t* w, int64_t block_rows) {
  return guarded(ctx, [&](Ctx& c) {
    validate_spec(omega);
    validate_spec(psi);
    check_view(host_block, "sketch_update_rows");
    check_view(y_rows, "sketch_update_rows");
    check_view(w, "sketch_update_rows");
    const int64_t n = w->cols;
    if (host_block->cols != n || omega->rows != n)
      fail(QLRA_ERR_SHAPE, "sketch_update_rows: column count mismatch");
    if (y_rows->rows != host_block->rows || y_rows->cols != omega->cols || w->rows != psi->rows)
      fail(QLRA_ERR_SHAPE, "sketch_update_rows: sketch shape mismatch");
    if (row0 < 0 || row0 + host_block->rows > psi->cols)
      fail(QLRA_ERR_SHAPE, "sketch_update_rows: row range out of bounds");
    if (block_rows < 0) fail(QLRA_ERR_PARAMETER, "sketch_from_source: block_rows must be >= 1");
    sketch_update_rows_host(c, *omega, *psi, row0, view_of(host_block), view_of(y_rows),
                            view_of(w), block_rows);
  });
}

int qlra_sketch_allreduce(qlra_ctx_t* ctx, qlra_qmat_t* w) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(w, "sketch_allreduce");
    allreduce_qmat(c, view_of(w));
  });
}

int qlra_qmat_mul(qlra_ctx_t* ctx, int op_a, int op_b, double alpha, const qlra_qmat_t* a,
                  const qlra_qmat_t* b, double beta, qlra_qmat_t* cm) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(a, "qmat_mul");
    check_view(b, "qmat_mul");
    check_view(cm, "qmat_mul");
    qgemm(c, op_a, op_b, alpha, view_of(a), view_of(b), beta, view_of(cm));
  });
}

int qlra_gram(qlra_ctx_t* ctx, const qlra_qmat_t* h, qlra_qmat_t* g) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(h, "gram");
    check_view(g, "gram");
    if (g->rows != h->cols || g->cols != h->cols) fail(QLRA_ERR_SHAPE, "gram: output shape mismatch");
    gram(c, view_of(h), view_of(g));
  });
}

int qlra_condition_number(qlra_ctx_t* ctx, const qlra_qmat_t* h, double* kappa) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(h, "condition_number");
    if (h->rows < h->cols && c.nranks == 1) {
      // wide: singular values of A^* (tall)
      if (h->rows == 0) {
        *kappa = std::numeric_limits<double>::infinity();
        return;
      }
      DevQMat at(c, h->cols, h->rows);
      qgemm(c, QLRA_OP_C, QLRA_OP_N, 1.0, view_of(h), identity_like(c, h->rows).v, 0.0, at.v);
      *kappa = condition_number_dev(c, at.v);
    } else {
      *kappa = condition_number_dev(c, view_of(h));
    }
  });
}

int qlra_singular_values(qlra_ctx_t* ctx, const qlra_qmat_t* a, double* sv) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(a, "singular_values");
    const bool wide = a->rows < a->cols && c.nranks == 1;
    const int64_t k = wide ? a->rows : a->cols;
    if (k == 0) return;
    DevQMat g(c, k, k);
    std::vector<double> ev;
    if (wide) {  // (the wide form refines through the tall A^*)
      DevQMat at(c, a->cols, a->rows);
      qgemm(c, QLRA_OP_C, QLRA_OP_N, 1.0, view_of(a), identity_like(c, a->rows).v, 0.0, at.v);
      gram(c, at.v, g.v);
      ev = gram_spectrum(c, at.v, g.v, /*extremes_only=*/false);
    } else {
      gram(c, view_of(a), g.v);
      ev = gram_spectrum(c, view_of(a), g.v, /*extremes_only=*/false);
    }
    for (int64_t i = 0; i < k; ++i) sv[i] = std::sqrt(std::max(0.0, ev[i]));
  });
}

int qlra_solve_quaternion_linear(qlra_ctx_t* ctx, const qlra_qmat_t* a, const qlra_qmat_t* b,
                                 qlra_qmat_t* x) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(a, "solve_quaternion_linear");
    check_view(b, "solve_quaternion_linear");
    check_view(x, "solve_quaternion_linear");
    if (a->rows != b->rows) fail(QLRA_ERR_SHAPE, "solve_quaternion_linear: row mismatch");
    if (a->rows < a->cols)
      fail(QLRA_ERR_SHAPE, "solve_quaternion_linear: underdetermined system not supported");
    if (x->rows != a->cols || x->cols != b->cols)
      fail(QLRA_ERR_SHAPE, "solve_quaternion_linear: output shape mismatch");
    const QView A = view_of(a), B = view_of(b), X = view_of(x);
    if (a->rows == a->cols) {
      if (a->rows == 0) return;
      DevQMat ainv(c, a->rows, a->cols);
      const std::vector<double> st = quat_inverse(c, A, ainv.v);
      if (st[0] != 0.0)
        fail(QLRA_ERR_SINGULAR, "solve_quaternion_linear: singular system",
             std::numeric_limits<double>::infinity());
      DeviceBuffer nrm(c, 2 * sizeof(double));
      small_chi_norm1(c, A, nrm.as<double>());
      small_chi_norm1(c, ainv.v, nrm.as<double>() + 1);
      const std::vector<double> nn = to_host(c, nrm.as<double>(), 2);
      const double rc = (nn[0] > 0 && nn[1] > 0) ? 1.0 / (nn[0] * nn[1]) : 0.0;
      if (!(rc > 1e-14))
        fail(QLRA_ERR_SINGULAR, "solve_quaternion_linear: singular system",
             rc > 0 ? 1.0 / rc : std::numeric_limits<double>::infinity());
      qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, ainv.v, B, 0.0, X);
    } else {
      lstsq(c, A, B, X);
    }
  });
}

int qlra_estimate_epsilon(qlra_ctx_t* ctx, const qlra_qmat_t* h, int power_iters, double* eps) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(h, "estimate_epsilon");
    if (power_iters < 1) fail(QLRA_ERR_PARAMETER, "estimate_epsilon: power_iters must be >= 1");
    const int64_t s = h->cols;
    DevQMat g(c, s, s), ginv(c, s, s);
    gram(c, view_of(h), g.v);
    if (!hpd_inverse(c, g.v, ginv.v, nullptr))
      fail(QLRA_ERR_SINGULAR, "estimate_epsilon: H*H numerically singular",
           std::numeric_limits<double>::infinity());
    *eps = estimate_epsilon_rc(c, g.v, ginv.v, power_iters, nullptr);
  });
}

int qlra_correction_step(qlra_ctx_t* ctx, const qlra_qmat_t* h, double epsilon, qlra_qmat_t* hout) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(h, "correction_step");
    check_view(hout, "correction_step");
    if (!(epsilon > 0.0 && epsilon < 1.0))
      fail(QLRA_ERR_PARAMETER, "correction_step: epsilon must lie in (0,1)");
    const int64_t s = h->cols;
    DevQMat g(c, s, s), ginv(c, s, s);
    gram(c, view_of(h), g.v);
    if (!hpd_inverse(c, g.v, ginv.v, nullptr))
      fail(QLRA_ERR_SINGULAR, "solve_quaternion_linear: singular system",
           std::numeric_limits<double>::infinity());
    // the square solve's rcond test (complex_bridge.cpp:73-77) on rcond_1
    DeviceBuffer nr(c, 2 * sizeof(double));
    small_chi_norm1(c, g.v, nr.as<double>());
    small_chi_norm1(c, ginv.v, nr.as<double>() + 1);
    const std::vector<double> nn = to_host(c, nr.as<double>(), 2);
    check_solve_rc((nn[0] > 0 && nn[1] > 0) ? 1.0 / (nn[0] * nn[1]) : 0.0);
    correction_from_inverse(c, view_of(h), ginv.v, epsilon, view_of(hout));
  });
}

int qlra_pseudo_qr(qlra_ctx_t* ctx, const qlra_qmat_t* y, const qlra_pseudo_qr_config_t* cfg_in,
                   qlra_qmat_t* h, qlra_rangefinder_report_t* rep) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(y, "pseudo_qr");
    check_view(h, "pseudo_qr");
    qlra_pseudo_qr_config_t cfg{3, 3, 1.2};
    if (cfg_in) cfg = *cfg_in;
    if (h->rows != y->rows || h->cols != y->cols) fail(QLRA_ERR_SHAPE, "pseudo_qr: output shape mismatch");
    pseudo_qr_dev(c, view_of(y), view_of(h), cfg, rep);
  });
}

int qlra_pseudo_svd(qlra_ctx_t* ctx, const qlra_qmat_t* y, uint64_t seed, qlra_qmat_t* h,
                    qlra_rangefinder_report_t* rep) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(y, "pseudo_svd");
    check_view(h, "pseudo_svd");
    if (h->rows != y->rows || h->cols != y->cols) fail(QLRA_ERR_SHAPE, "pseudo_svd: output shape mismatch");
    pseudo_svd_dev(c, view_of(y), view_of(h), seed, rep);
  });
}

int qlra_orthonormal_range(qlra_ctx_t* ctx, const qlra_qmat_t* y, uint64_t seed, qlra_qmat_t* h) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(y, "orthonormal_range");
    check_view(h, "orthonormal_range");
    if (h->rows != y->rows || h->cols != y->cols) fail(QLRA_ERR_SHAPE, "orthonormal_range: output shape mismatch");
    pseudo_svd_dev(c, view_of(y), view_of(h), seed, nullptr, nullptr, /*range_only=*/true);
  });
}

void check_solve_shapes(const qlra_spec_t* psi, int64_t row0, const qlra_qmat_t* h, const qlra_qmat_t* w,
                        const qlra_qmat_t* x) {
  const int64_t s = h->cols, l = psi->rows, n = w->cols;
  if (w->rows != l || x->rows != s || x->cols != n) fail(QLRA_ERR_SHAPE, "qb_stage: shape mismatch");
  if (row0 < 0 || row0 + h->rows > psi->cols) fail(QLRA_ERR_SHAPE, "qb_stage: Psi shape mismatch");
}

int qlra_qb_solve(qlra_ctx_t* ctx, const qlra_spec_t* psi, int64_t row0, const qlra_qmat_t* h,
                  const qlra_qmat_t* w, qlra_qmat_t* x) {
  return guarded(ctx, [&](Ctx& c) {
    validate_spec(psi);
    check_view(h, "qb_solve");
    check_view(w, "qb_solve");
    check_view(x, "qb_solve");
    check_solve_shapes(psi, row0, h, w, x);
    qb_solve_dev(c, *psi, row0, view_of(h), view_of(w), view_of(x));
  });
}

// qb_stage_with_psi (sketching.cpp:169-194) in one call: rangefinder on Y,
// then X = (Psi H) \ W; with pseudo-QR the solve starts inside the
// rangefinder (EarlySolve).
int qlra_qb_stage(qlra_ctx_t* ctx, const qlra_spec_t* psi, int64_t row0, const qlra_qmat_t* y,
                  const qlra_qmat_t* w, int method, uint64_t rangefinder_seed, const qlra_pseudo_qr_config_t* cfg_in,
                  qlra_qmat_t* h, qlra_qmat_t* x, qlra_rangefinder_report_t* rep) {
  return guarded(ctx, [&](Ctx& c) {
    validate_spec(psi);
    check_view(y, "qb_stage");
    check_view(w, "qb_stage");
    check_view(h, "qb_stage");
    check_view(x, "qb_stage");
    if (h->rows != y->rows || h->cols != y->cols) fail(QLRA_ERR_SHAPE, "qb_stage: output shape mismatch");
    check_solve_shapes(psi, row0, h, w, x);
    if (method != QLRA_PSEUDO_QR && method != QLRA_PSEUDO_SVD) fail(QLRA_ERR_PARAMETER, "qb_stage: unknown rangefinder");
    qlra_pseudo_qr_config_t cfg{3, 3, 1.2};
    if (cfg_in) cfg = *cfg_in;
    EarlySolve es(c, *psi, row0, view_of(w));
    PsvdDeferred pd;
    if (method == QLRA_PSEUDO_QR) pseudo_qr_dev(c, view_of(y), view_of(h), cfg, rep, &es);
    else pseudo_svd_dev(c, view_of(y), view_of(h), rangefinder_seed, rep, &pd);
    const CoreSolve cs = core_solve(c, &es, *psi, row0, view_of(h), view_of(w));
    cs.cols(c, 0, x->cols, view_of(x));
    pd.finish(rep);
  });
}

// one_pass_approx through the QB stage (sketching.cpp:250-263) on a
// device-resident row shard, in one call: the sketch into y, w (zeroed
// here), the rangefinder into h, the core solve into x.
int qlra_one_pass_qb(qlra_ctx_t* ctx, const qlra_qmat_t* a, int64_t row0, const qlra_spec_t* omega,
                     const qlra_spec_t* psi, int method, uint64_t rangefinder_seed,
                     const qlra_pseudo_qr_config_t* cfg_in, qlra_qmat_t* y, qlra_qmat_t* w, qlra_qmat_t* h,
                     qlra_qmat_t* x, qlra_rangefinder_report_t* rep) {
  return guarded(ctx, [&](Ctx& c) {
    validate_spec(omega);
    validate_spec(psi);
    for (const qlra_qmat_t* m : {a, (const qlra_qmat_t*)y, (const qlra_qmat_t*)w, (const qlra_qmat_t*)h,
                                 (const qlra_qmat_t*)x})
      check_view(m, "one_pass_qb");
    const int64_t rows = a->rows, n = a->cols, s = omega->cols, l = psi->rows;
    if (omega->rows != n || row0 < 0 || psi->cols < row0 + rows)
      fail(QLRA_ERR_SHAPE, "one_pass_qb: test matrix shape mismatch");
    if (y->rows != rows || y->cols != s || w->rows != l || w->cols != n || h->rows != rows || h->cols != s ||
        x->rows != s || x->cols != n)
      fail(QLRA_ERR_SHAPE, "one_pass_qb: output shape mismatch");
    if (method != QLRA_PSEUDO_QR && method != QLRA_PSEUDO_SVD) fail(QLRA_ERR_PARAMETER, "qb_stage: unknown rangefinder");
    qlra_pseudo_qr_config_t cfg{3, 3, 1.2};
    if (cfg_in) cfg = *cfg_in;
    const QView yv = view_of(y), wv = view_of(w);
    for (const QView* v : {&yv, &wv})
      for (int p = 0; p < 4; ++p)
        if (v->rows * v->cols > 0)
          QLRA_CUDA(cudaMemset2DAsync(v->p[p], sizeof(double) * v->ld, 0, sizeof(double) * v->cols, (size_t)v->rows,
                                      c.stream));
    sketch_update_rows(c, *omega, *psi, row0, view_of(a), yv, wv);
    allreduce_qmat(c, wv);
    EarlySolve es(c, *psi, row0, wv);
    es.omega = omega;
    PsvdDeferred pd;
    if (method == QLRA_PSEUDO_QR) pseudo_qr_dev(c, yv, view_of(h), cfg, rep, &es);
    else pseudo_svd_dev(c, yv, view_of(h), rangefinder_seed, rep, &pd);
    const CoreSolve cs = core_solve(c, &es, *psi, row0, view_of(h), wv);
    cs.cols(c, 0, x->cols, view_of(x));
    pd.finish(rep);
  });
}

// qb_stage_with_psi (sketching.cpp:169-188) with an explicitly supplied Psi:
// psi is the rank's column slice Psi(:, row0 : row0 + y.rows) in device
// memory (l x y.rows); the reference's own tests inject structured ones
// (test_sketching.cpp:170-183).  Rangefinder, then P = Psi H (all-reduced
// over the ranks) and X = P \ W through a QR of P.
int qlra_qb_stage_with_psi(qlra_ctx_t* ctx, const qlra_qmat_t* psi, const qlra_qmat_t* y, const qlra_qmat_t* w,
                           int method, uint64_t rangefinder_seed, const qlra_pseudo_qr_config_t* cfg_in,
                           qlra_qmat_t* h, qlra_qmat_t* x, qlra_rangefinder_report_t* rep) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(psi, "qb_stage_with_psi");
    check_view(y, "qb_stage_with_psi");
    check_view(w, "qb_stage_with_psi");
    check_view(h, "qb_stage_with_psi");
    check_view(x, "qb_stage_with_psi");
    if (h->rows != y->rows || h->cols != y->cols) fail(QLRA_ERR_SHAPE, "qb_stage: output shape mismatch");
    // qmat_mul(psi, h) (sketching.cpp:184): inner dimensions must agree
    if (psi->cols != y->rows) fail(QLRA_ERR_SHAPE, "qmat_mul: inner dimensions differ");
    if (w->rows != psi->rows) fail(QLRA_ERR_SHAPE, "solve_quaternion_linear: row mismatch");
    if (x->rows != y->cols || x->cols != w->cols) fail(QLRA_ERR_SHAPE, "qb_stage: shape mismatch");
    if (method != QLRA_PSEUDO_QR && method != QLRA_PSEUDO_SVD) fail(QLRA_ERR_PARAMETER, "qb_stage: unknown rangefinder");
    qlra_pseudo_qr_config_t cfg{3, 3, 1.2};
    if (cfg_in) cfg = *cfg_in;
    if (method == QLRA_PSEUDO_QR) pseudo_qr_dev(c, view_of(y), view_of(h), cfg, rep);
    else pseudo_svd_dev(c, view_of(y), view_of(h), rangefinder_seed, rep);
    const int64_t s = y->cols, l = psi->rows;
    if (l < s) fail(QLRA_ERR_SHAPE, "solve_quaternion_linear: underdetermined system not supported");
    DevQMat p(c, l, s);
    qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, view_of(psi), view_of(h), 0.0, p.v);
    allreduce_qmat(c, p.v);
    DevQMat t = lstsq_operator(c, p.v);
    qgemm(c, QLRA_OP_C, QLRA_OP_N, 1.0, t.v, view_of(w), 0.0, view_of(x));
  });
}

void* qlra_ctx_stream(const qlra_ctx_t* ctx) { return ctx ? static_cast<void*>(ctx->c.stream) : nullptr; }

// Host in, host out: one_pass_approx through the QB stage
// (sketching.cpp:250-263) on a host row shard.  A streams through the
// overlapped H2D + fused-sketch pipeline; H is copied back on a side stream
// while the core solve runs; X follows.
int qlra_one_pass_qb_host(qlra_ctx_t* ctx, const qlra_qmat_t* a_host, int64_t row0, const qlra_spec_t* omega,
                          const qlra_spec_t* psi, int method, uint64_t rangefinder_seed,
                          const qlra_pseudo_qr_config_t* cfg_in, int64_t block_rows, qlra_qmat_t* h_host,
                          qlra_qmat_t* x_host, qlra_rangefinder_report_t* rep) {
  return guarded(ctx, [&](Ctx& c) {
    validate_spec(omega);
    validate_spec(psi);
    check_view(a_host, "one_pass_qb");
    check_view(h_host, "one_pass_qb");
    check_view(x_host, "one_pass_qb");
    const int64_t rows = a_host->rows, n = a_host->cols, s = omega->cols, l = psi->rows;
    if (omega->rows != n || psi->cols < row0 + rows || row0 < 0)
      fail(QLRA_ERR_SHAPE, "one_pass_qb: test matrix shape mismatch");
    if (h_host->rows != rows || h_host->cols != s || x_host->rows != s || x_host->cols != n)
      fail(QLRA_ERR_SHAPE, "one_pass_qb: output shape mismatch");
    if (block_rows < 0) fail(QLRA_ERR_PARAMETER, "sketch_from_source: block_rows must be >= 1");
    if (method != QLRA_PSEUDO_QR && method != QLRA_PSEUDO_SVD)
      fail(QLRA_ERR_PARAMETER, "one_pass_qb: unknown rangefinder");
    qlra_pseudo_qr_config_t cfg{3, 3, 1.2};
    if (cfg_in) cfg = *cfg_in;
    DevQMat y(c, rows, s), w(c, l, n), h(c, rows, s), x(c, s, n);
    y.zero(c);
    w.zero(c);
    sketch_update_rows_host(c, *omega, *psi, row0, view_of(a_host), y.v, w.v, block_rows);
    allreduce_qmat(c, w.v);
    PsvdDeferred pd;  // pseudo-SVD: the kappa refinements overlapped with the solve
    qlra_rangefinder_report_t rr{};
    // No early solve here: H's read-back already hides the solve (C2:
    // 31.55 ms either way; C5: the early solve's side-stream work delays H
    // and so its 49 ms read-back, 433 -> 446 ms).
    EarlySolve* esp = nullptr;
    if (method == QLRA_PSEUDO_QR) pseudo_qr_dev(c, y.v, h.v, cfg, &rr, esp);
    else pseudo_svd_dev(c, y.v, h.v, rangefinder_seed, &rr, &pd);
    // H is final: copy it back on a side stream while the solve runs.  The
    // guard (declared after y, w, h, x) drains the side stream on every exit
    // -- a failing solve included -- before those buffers are released and
    // before the call returns, so no copy lands in the caller's buffers later.
    struct SideCopies {
      cudaStream_t s = nullptr;
      cudaEvent_t ready = nullptr, copied = nullptr;
      SideCopies() {
        QLRA_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        QLRA_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
        QLRA_CUDA(cudaEventCreateWithFlags(&copied, cudaEventDisableTiming));
      }
      ~SideCopies() {
        if (s) cudaStreamSynchronize(s);
        if (ready) cudaEventDestroy(ready);
        if (copied) cudaEventDestroy(copied);
        if (s) cudaStreamDestroy(s);
      }
    } sc;
    cudaStream_t side = sc.s;
    cudaEvent_t ready = sc.ready, copied = sc.copied;
    QLRA_CUDA(cudaEventRecord(ready, c.stream));
    QLRA_CUDA(cudaStreamWaitEvent(side, ready, 0));
    const QView hv = view_of(h_host), xv = view_of(x_host);
    for (int p = 0; p < 4; ++p) {
      if (hv.ld == s)  // contiguous: one linear DMA (h is dense)
        QLRA_CUDA(cudaMemcpyAsync(hv.p[p], h.v.p[p], sizeof(double) * (size_t)(rows * s), cudaMemcpyDeviceToHost,
                                  side));
      else
        QLRA_CUDA(cudaMemcpy2DAsync(hv.p[p], sizeof(double) * hv.ld, h.v.p[p], sizeof(double) * h.v.ld,
                                    sizeof(double) * s, (size_t)rows, cudaMemcpyDeviceToHost, side));
    }
    // X = T^* W in column blocks; each block is copied back on the side
    // stream while the next one is computed
    const CoreSolve cs = core_solve(c, esp, *psi, row0, h.v, w.v);
    const int64_t nblk = n >= 2048 ? 4 : 1;
    const int64_t bw = (n + nblk - 1) / nblk;
    for (int64_t j0 = 0; j0 < n; j0 += bw) {
      const int64_t nj = std::min(bw, n - j0);
      cs.cols(c, j0, nj, x.v);
      QLRA_CUDA(cudaEventRecord(ready, c.stream));
      QLRA_CUDA(cudaStreamWaitEvent(side, ready, 0));
      for (int p = 0; p < 4; ++p)
        QLRA_CUDA(cudaMemcpy2DAsync(xv.p[p] + j0, sizeof(double) * xv.ld, x.v.p[p] + j0, sizeof(double) * x.v.ld,
                                    sizeof(double) * nj, (size_t)s, cudaMemcpyDeviceToHost, side));
    }
    QLRA_CUDA(cudaEventRecord(copied, side));
    pd.finish(&rr);
    if (rep) *rep = rr;
    // device buffers are released on c.stream: order that after the copies
    QLRA_CUDA(cudaStreamWaitEvent(c.stream, copied, 0));
    QLRA_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int qlra_residual_fro(qlra_ctx_t* ctx, const qlra_qmat_t* a, const qlra_qmat_t* h,
                      const qlra_qmat_t* x, double* res_fro, double* a_fro) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(a, "residual");
    check_view(h, "residual");
    check_view(x, "residual");
    DeviceBuffer out(c, 2 * sizeof(double));
    qgemm_residual(c, view_of(a), view_of(h), view_of(x), out.as<double>());
    allreduce_sum(c, out.as<double>(), 2);
    const std::vector<double> v = to_host(c, out.as<double>(), 2);
    if (res_fro) *res_fro = std::sqrt(v[0]);
    if (a_fro) *a_fro = std::sqrt(v[1]);
  });
}

// qsvd of a replicated wide-or-tall A (factorizations.cpp:166-295) through the
// Hermitian eigendecomposition of the smaller Gram.  u: m x k, v: n x k,
// sigma: k host values (k = min(m, n)), nonincreasing.
static void qsvd_dev(Ctx& c, const QView& a, const QView& u, const QView& v, double* sigma_host,
                     bool complex_only = false) {
  const int64_t m = a.rows, n = a.cols, k = std::min(m, n);
  if (k == 0) return;
  const bool wide = m < n;  // reference: qsvd(A^*) then swap (factorizations.cpp:167-170)
  // small side eigenvectors E (k x k): of A A^* when wide (-> U), of A^*A when tall (-> V)
  DevQMat g(c, k, k), e(c, k, k);
  if (wide)
    qgemm(c, QLRA_OP_N, QLRA_OP_C, 1.0, a, a, 0.0, g.v);
  else
    qgemm(c, QLRA_OP_C, QLRA_OP_N, 1.0, a, a, 0.0, g.v);
  DeviceBuffer w(c, sizeof(double) * (size_t)k);
  small_quat_eigh(c, g.v, w.as<double>(), e.v);
  // Second pass: B = E^* A (wide; A E when tall) has nearly orthogonal rows
  // (columns) of norms sigma_i, computed with absolute error ~u sigma_1, so
  // the eigenvalues of its (nearly diagonal) Gram carry sigma_i to relative
  // accuracy ~u sigma_1 / sigma_i -- an SVD's accuracy -- where the first
  // Gram's carry u (sigma_1 / sigma_i)^2.  E <- E E2 (the reference takes
  // the factors from an SVD of chi(A), factorizations.cpp:166-295).
  {
    DevQMat b(c, wide ? k : m, wide ? n : k), e2(c, k, k), e12(c, k, k);
    if (wide) {
      qgemm(c, QLRA_OP_C, QLRA_OP_N, 1.0, e.v, a, 0.0, b.v);
      qgemm(c, QLRA_OP_N, QLRA_OP_C, 1.0, b.v, b.v, 0.0, g.v);
    } else {
      qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, a, e.v, 0.0, b.v);
      qgemm(c, QLRA_OP_C, QLRA_OP_N, 1.0, b.v, b.v, 0.0, g.v);
    }
    small_quat_eigh(c, g.v, w.as<double>(), e2.v);
    qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, e.v, e2.v, 0.0, e12.v);
    e = std::move(e12);
  }
  std::vector<double> lam = to_host(c, w.as<double>(), (size_t)k);
  std::vector<double> sg(k);
  for (int64_t i = 0; i < k; ++i) sg[i] = std::sqrt(std::max(0.0, lam[i]));
  const double tiny = 1e-13 * sg[0];
  int64_t good = 0;
  while (good < k && sg[good] > tiny) ++good;
  DeviceBuffer d_sg(c, sizeof(double) * (size_t)k);
  QLRA_CUDA(cudaMemcpyAsync(d_sg.ptr, sg.data(), sizeof(double) * k, cudaMemcpyHostToDevice, c.stream));
  // big side: A^* U / sigma (wide) or A V / sigma (tall)
  const QView small = wide ? u : v, big = wide ? v : u;
  copy_qmat(c, e.v, small);
  DevQMat t(c, big.rows, k);
  if (wide)
    qgemm(c, QLRA_OP_C, QLRA_OP_N, 1.0, a, e.v, 0.0, t.v);
  else
    qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, a, e.v, 0.0, t.v);
  scale_cols(c, t.v, d_sg.as<double>(), true, tiny, t.v);
  // Polish (factorizations.cpp:245-260): Gram-Schmidt in sigma order strips
  // the eps/gap leakage; CholeskyQR spans the same nested column spaces.
  if (good > 0 && !cholesky_qr(c, sub(t.v, 0, 0, big.rows, good), sub(big, 0, 0, big.rows, good),
                               false, big.rows, nullptr))
    copy_qmat(c, sub(t.v, 0, 0, big.rows, good), sub(big, 0, 0, big.rows, good));
  if (good < k)  // zero singular values: orthonormal completion (factorizations.cpp:224-236)
    orthonormal_completion(c, sub(big, 0, 0, big.rows, good), sub(big, 0, good, big.rows, k - good), 0,
                           big.rows, rng_substream(rng_key(0x715D), (uint64_t)(m * 131 + n)), complex_only);
  // phase convention on the tall factorization's V: the small side in both
  // orientations (for wide A the reference factors A^*, factorizations.cpp:167-170)
  qsvd_phase(c, big, small);
  for (int64_t i = 0; i < k; ++i) sigma_host[i] = sg[i];
}

int qlra_qsvd(qlra_ctx_t* ctx, const qlra_qmat_t* a, qlra_qmat_t* u, double* sigma, qlra_qmat_t* v) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(a, "qsvd");
    check_view(u, "qsvd");
    check_view(v, "qsvd");
    const int64_t k = std::min(a->rows, a->cols);
    if (u->rows != a->rows || u->cols != k || v->rows != a->cols || v->cols != k)
      fail(QLRA_ERR_SHAPE, "qsvd: output shape mismatch");
    qsvd_dev(c, view_of(a), view_of(u), view_of(v), sigma);
  });
}

int qlra_truncate_stage(qlra_ctx_t* ctx, const qlra_qmat_t* h, const qlra_qmat_t* x, int64_t r,
                        qlra_qmat_t* h_out, double* sigma, qlra_qmat_t* v) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(h, "truncate_stage");
    check_view(x, "truncate_stage");
    check_view(h_out, "truncate_stage");
    check_view(v, "truncate_stage");
    if (h->cols != x->rows) fail(QLRA_ERR_SHAPE, "truncate_stage: H and X do not conform");
    if (r < 1 || r > x->rows) fail(QLRA_ERR_PARAMETER, "truncate_stage: need 1 <= r <= s");
    if (h_out->rows != h->rows || h_out->cols != r || v->rows != x->cols || v->cols != r)
      fail(QLRA_ERR_SHAPE, "truncate_stage: output shape mismatch");
    const int64_t s = x->rows, n = x->cols, k = std::min(s, n);
    DevQMat uu(c, s, k), vv(c, n, k);
    std::vector<double> sg(k);
    qsvd_dev(c, view_of(x), uu.v, vv.v, sg.data());
    qgemm(c, QLRA_OP_N, QLRA_OP_N, 1.0, view_of(h), sub(uu.v, 0, 0, s, r), 0.0, view_of(h_out));
    copy_qmat(c, sub(vv.v, 0, 0, n, r), view_of(v));
    for (int64_t i = 0; i < r; ++i) sigma[i] = sg[i];
  });
}

int qlra_approx_residual_fro(qlra_ctx_t* ctx, const qlra_qmat_t* a, const qlra_qmat_t* h,
                             const double* sigma, const qlra_qmat_t* v, double* res_fro,
                             double* a_fro) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(a, "relative_error");
    check_view(h, "relative_error");
    check_view(v, "relative_error");
    const int64_t r = h->cols, n = v->rows;
    DeviceBuffer d_s(c, sizeof(double) * (size_t)std::max<int64_t>(1, r));
    QLRA_CUDA(cudaMemcpyAsync(d_s.ptr, sigma, sizeof(double) * r, cudaMemcpyHostToDevice, c.stream));
    DevQMat xr(c, r, n);
    sigma_vadj(c, d_s.as<double>(), view_of(v), xr.v);
    DeviceBuffer out(c, 2 * sizeof(double));
    qgemm_residual(c, view_of(a), view_of(h), xr.v, out.as<double>());
    allreduce_sum(c, out.as<double>(), 2);
    const std::vector<double> vals = to_host(c, out.as<double>(), 2);
    if (res_fro) *res_fro = std::sqrt(vals[0]);
    if (a_fro) *a_fro = std::sqrt(vals[1]);
  });
}

static void check_cview(const qlra_cmat_t* m, const char* who) {
  if (!m) fail(QLRA_ERR_PARAMETER, std::string(who) + ": null matrix");
  if (m->rows < 0 || m->cols < 0 || m->ld < std::max<int64_t>(1, m->rows) ||
      (m->rows * m->cols > 0 && !m->data))
    fail(QLRA_ERR_SHAPE, std::string(who) + ": bad matrix view");
}

int qlra_to_compact(qlra_ctx_t* ctx, const qlra_qmat_t* a, qlra_cmat_t* out) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(a, "to_compact");
    check_cview(out, "to_compact");
    if (out->rows != 2 * a->rows || out->cols != a->cols) fail(QLRA_ERR_SHAPE, "to_compact: output shape mismatch");
    to_complex(c, view_of(a), cview_of(out), false);
  });
}

int qlra_to_full(qlra_ctx_t* ctx, const qlra_qmat_t* a, qlra_cmat_t* out) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(a, "to_full");
    check_cview(out, "to_full");
    if (out->rows != 2 * a->rows || out->cols != 2 * a->cols) fail(QLRA_ERR_SHAPE, "to_full: output shape mismatch");
    to_complex(c, view_of(a), cview_of(out), true);
  });
}

int qlra_from_compact(qlra_ctx_t* ctx, const qlra_cmat_t* z, qlra_qmat_t* out) {
  return guarded(ctx, [&](Ctx& c) {
    check_cview(z, "from_compact");
    check_view(out, "from_compact");
    if (z->rows % 2 != 0) fail(QLRA_ERR_SHAPE, "from_compact: odd row count");  // complex_bridge.cpp:38
    if (out->rows != z->rows / 2 || out->cols != z->cols) fail(QLRA_ERR_SHAPE, "from_compact: output shape mismatch");
    from_compact(c, cview_of(z), view_of(out));
  });
}

int qlra_j_mul_conj(qlra_ctx_t* ctx, const qlra_cmat_t* u, qlra_cmat_t* out) {
  return guarded(ctx, [&](Ctx& c) {
    check_cview(u, "j_mul_conj");
    check_cview(out, "j_mul_conj");
    if (u->rows % 2 != 0) fail(QLRA_ERR_SHAPE, "j_mul_conj: odd row count");  // complex_bridge.cpp:55
    if (out->rows != u->rows || out->cols != u->cols) fail(QLRA_ERR_SHAPE, "j_mul_conj: output shape mismatch");
    if (out->data == u->data) fail(QLRA_ERR_PARAMETER, "j_mul_conj: output must not alias the input");
    j_mul_conj(c, cview_of(u), cview_of(out));
  });
}

int qlra_complex_qr(qlra_ctx_t* ctx, const qlra_cmat_t* m, qlra_cmat_t* q, qlra_cmat_t* r) {
  return guarded(ctx, [&](Ctx& c) {
    check_cview(m, "complex_qr");
    check_cview(q, "complex_qr");
    check_cview(r, "complex_qr");
    const int64_t p = m->rows, n = m->cols;
    if (p < n) fail(QLRA_ERR_SHAPE, "complex_qr: requires rows >= cols");  // factorizations.cpp:34
    if (q->rows != p || q->cols != n || r->rows != n || r->cols != n)
      fail(QLRA_ERR_SHAPE, "complex_qr: output shape mismatch");
    if (n == 0) return;
    // The complex matrix as a quaternion one (y = z = 0): the complex-mode
    // CholeskyQR2 (Gram's j, k planes zeroed) never leaves the complex
    // subalgebra, and its R has a real positive diagonal -- the reference's
    // phase convention (factorizations.cpp:40-49) -- so Q is the same
    // unique Q up to rounding.
    DevQMat e(c, p, n), qe(c, p, n), rf;
    cmat_to_quat(c, cview_of(m), e.v);
    std::vector<double> rd;
    if (!cholesky_qr(c, e.v, qe.v, /*complex_mode=*/true, p, &rd, /*distributed=*/false, nullptr, &rf))
      fail(QLRA_ERR_RANK, "complex_qr: numerically rank-deficient input (CholeskyQR route)");
    quat_to_cmat(c, qe.v, cview_of(q));
    quat_to_cmat(c, rf.v, cview_of(r));
    QLRA_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int qlra_complex_svd(qlra_ctx_t* ctx, const qlra_cmat_t* m, qlra_cmat_t* u, double* s, qlra_cmat_t* v) {
  return guarded(ctx, [&](Ctx& c) {
    check_cview(m, "complex_svd");
    check_cview(u, "complex_svd");
    check_cview(v, "complex_svd");
    const int64_t p = m->rows, n = m->cols, k = std::min(p, n);
    if (u->rows != p || u->cols != k || v->rows != n || v->cols != k)
      fail(QLRA_ERR_SHAPE, "complex_svd: output shape mismatch");
    if (k == 0) return;
    DevQMat e(c, p, n), uq(c, p, k), vq(c, n, k);
    cmat_to_quat(c, cview_of(m), e.v);
    qsvd_dev(c, e.v, uq.v, vq.v, s, /*complex_only=*/true);
    quat_to_cmat(c, uq.v, cview_of(u));
    quat_to_cmat(c, vq.v, cview_of(v));
    QLRA_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int qlra_qmat_pinv(qlra_ctx_t* ctx, const qlra_qmat_t* a, qlra_qmat_t* out) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(a, "qmat_pinv");
    check_view(out, "qmat_pinv");
    const int64_t m = a->rows, n = a->cols, k = std::min(m, n);
    if (out->rows != n || out->cols != m) fail(QLRA_ERR_SHAPE, "qmat_pinv: output shape mismatch");
    if (k == 0) return;
    DevQMat uu(c, m, k), vv(c, n, k);
    std::vector<double> sg((size_t)k);
    qsvd_dev(c, view_of(a), uu.v, vv.v, sg.data());
    // factorizations.cpp:303-314: sigma <= max(m, n) eps sigma_max -> 0
    const double tol = (double)std::max(m, n) * std::numeric_limits<double>::epsilon() * sg[0];
    std::vector<double> inv((size_t)k);
    for (int64_t i = 0; i < k; ++i) inv[i] = sg[i] > tol ? 1.0 / sg[i] : 0.0;
    DeviceBuffer d_inv(c, sizeof(double) * (size_t)k);
    QLRA_CUDA(cudaMemcpyAsync(d_inv.ptr, inv.data(), sizeof(double) * k, cudaMemcpyHostToDevice, c.stream));
    scale_cols(c, vv.v, d_inv.as<double>(), false, 0.0, vv.v);
    qgemm(c, QLRA_OP_N, QLRA_OP_C, 1.0, vv.v, uu.v, 0.0, view_of(out));
    QLRA_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int qlra_spectral_norm(qlra_ctx_t* ctx, const qlra_qmat_t* a, double* norm) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(a, "spectral_norm");
    *norm = 0.0;
    const int64_t k = std::min(a->rows, a->cols);
    if (k == 0) return;
    // lambda_max of the smaller Gram: relative accuracy u at the top
    DevQMat g(c, k, k);
    if (a->rows < a->cols && c.nranks == 1)
      qgemm(c, QLRA_OP_N, QLRA_OP_C, 1.0, view_of(a), view_of(a), 0.0, g.v);
    else
      gram(c, view_of(a), g.v);
    *norm = std::sqrt(std::max(0.0, quat_eigs(c, g.v, /*extremes_only=*/true)[0]));
  });
}

int qlra_write_qmat(qlra_ctx_t* ctx, const char* path, const qlra_qmat_t* m) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(m, "write_qmat");
    write_qmat(c, path, view_of(m));
  });
}

int qlra_qmat_file_shape(const char* path, int64_t* rows, int64_t* cols) {
  try {
    qmat_header(path, rows, cols);
    return QLRA_OK;
  } catch (const Status& s) {
    return s.code;
  } catch (...) {
    return QLRA_ERR_IO;
  }
}

int qlra_read_qmat(qlra_ctx_t* ctx, const char* path, qlra_qmat_t* m) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(m, "read_qmat");
    read_qmat(c, path, view_of(m));
  });
}

int qlra_write_sketch(qlra_ctx_t* ctx, const char* path, const qlra_spec_t* omega,
                      const qlra_spec_t* psi, int64_t r, int64_t s, int64_t l,
                      const qlra_qmat_t* y, const qlra_qmat_t* w) {
  return guarded(ctx, [&](Ctx& c) {
    validate_spec(omega);
    validate_spec(psi);
    check_view(y, "write_sketch");
    check_view(w, "write_sketch");
    write_sketch(c, path, *omega, *psi, r, s, l, view_of(y), view_of(w));
  });
}

int qlra_sketch_file_header(const char* path, qlra_spec_t* omega, qlra_spec_t* psi, int64_t* rsl) {
  try {
    sketch_header(path, omega, psi, rsl);
    return QLRA_OK;
  } catch (const Status& s) {
    return s.code;
  } catch (...) {
    return QLRA_ERR_IO;
  }
}

int qlra_sketch_file_dims(const char* path, int64_t* dims) {
  try {
    sketch_dims(path, dims);
    return QLRA_OK;
  } catch (const Status& s) {
    return s.code;
  } catch (...) {
    return QLRA_ERR_IO;
  }
}

int qlra_read_sketch(qlra_ctx_t* ctx, const char* path, qlra_qmat_t* y, qlra_qmat_t* w) {
  return guarded(ctx, [&](Ctx& c) {
    check_view(y, "read_sketch");
    check_view(w, "read_sketch");
    read_sketch(c, path, view_of(y), view_of(w));
  });
}

int qlra_sketch_from_qmat_file(qlra_ctx_t* ctx, const char* path, const qlra_spec_t* omega,
                               const qlra_spec_t* psi, qlra_qmat_t* y, qlra_qmat_t* w,
                               int64_t block_rows) {
  return guarded(ctx, [&](Ctx& c) {
    validate_spec(omega);
    validate_spec(psi);
    check_view(y, "sketch_from_source");
    check_view(w, "sketch_from_source");
    sketch_from_qmat_file(c, path, *omega, *psi, view_of(y), view_of(w), block_rows);
  });
}

int qlra_measure_fp64_peak(qlra_ctx_t* ctx, int mode, double ms, double* tflops) {
  return guarded(ctx, [&](Ctx& c) { *tflops = measure_fp64_peak(c, mode, ms); });
}

const char* qlra_sketch_kernel_name(void) { return sketch_kernel_name(); }

}  // extern "C"
