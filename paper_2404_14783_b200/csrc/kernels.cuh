// kernels.cuh -- host-side declarations shared by the qlra CUDA sources.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace qlra_dev {

// Launch counter (evidence of device work; exported via qlra_ctx_launch_count).
std::atomic<int64_t>& launch_counter();
// thread-safe, per-device cudaFuncSetAttribute (largest value wins)
void set_func_attr(const void* func, cudaFuncAttribute attr, int value);
inline void count_launch() { launch_counter().fetch_add(1, std::memory_order_relaxed); }

// One context per (host thread, device): stream, NCCL communicator, errors.
struct Ctx {
  int device = 0;
  int rank = 0, nranks = 1;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ncclComm_t comm = nullptr;
  std::string last_error;
  double last_cond = 0.0;
  double* pinned = nullptr;  // small host staging buffer (syncs)
  // per-tile arrival counters of the split-K small GEMM (self-resetting:
  // the last CTA of a tile sets its counter back to 0)
  unsigned* tile_cnt = nullptr;
  int64_t tile_cnt_n = 0;
  // side stream for overlapped small work, and its pinned read-back buffer
  // (created on first use, kept for the context's lifetime)
  cudaStream_t side = nullptr;
  double* side_pinned = nullptr;
  size_t side_pinned_n = 0;
  // second side stream (the core solve started inside pseudo-QR) with its own
  // split-K arrival counters (StreamSwap exchanges them with tile_cnt)
  cudaStream_t side2 = nullptr;
  unsigned* tile_cnt2 = nullptr;
  int64_t tile_cnt2_n = 0;
  // Optional per-launch timing of the fused sketch kernel (bench evidence):
  // CUDA events bracket every launch on the launching stream.
  struct KernelTimer {
    bool on = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;  // recorded pairs
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool;  // created up front (no driver call per launch)
    double flops = 0.0, a_bytes = 0.0;
    int64_t launches = 0;
  } ktimer;
};

// Stream-ordered device allocation (cudaMallocAsync from the device's default
// pool, whose release threshold is raised at ctx creation so steady-state
// calls do not hit the driver).
struct DeviceBuffer {
  Ctx* ctx = nullptr;
  void* ptr = nullptr;
  size_t bytes = 0;
  DeviceBuffer() = default;
  DeviceBuffer(Ctx& c, size_t n) : ctx(&c), bytes(n) {
    if (n) QLRA_CUDA(cudaMallocAsync(&ptr, n, c.stream));
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : ctx(o.ctx), ptr(o.ptr), bytes(o.bytes) { o.ptr = nullptr; }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      release();
      ctx = o.ctx;
      ptr = o.ptr;
      bytes = o.bytes;
      o.ptr = nullptr;
    }
    return *this;
  }
  void release() {
    if (ptr) cudaFreeAsync(ptr, ctx->stream);
    ptr = nullptr;
  }
  ~DeviceBuffer() { release(); }
  template <class T>
  T* as() const { return static_cast<T*>(ptr); }
};

// Owned device quaternion matrix (4 planes in one allocation, ld = cols).
struct DevQMat {
  DeviceBuffer buf;
  QView v{};
  DevQMat() = default;
  DevQMat(Ctx& c, int64_t rows, int64_t cols) : buf(c, (size_t)4 * rows * cols * sizeof(double)) {
    double* base = buf.as<double>();
    for (int p = 0; p < 4; ++p) v.p[p] = base + (size_t)p * rows * cols;
    v.rows = rows;
    v.cols = cols;
    v.ld = cols;
  }
  void zero(Ctx& c) {
    if (buf.bytes) QLRA_CUDA(cudaMemsetAsync(buf.ptr, 0, buf.bytes, c.stream));
  }
};

// Sub-block view (rows [r0, r0+nr), cols [c0, c0+nc)).
inline QView sub(const QView& a, int64_t r0, int64_t c0, int64_t nr, int64_t nc) {
  QView v = a;
  for (int p = 0; p < 4; ++p) v.p[p] = a.p[p] + r0 * a.ld + c0;
  v.rows = nr;
  v.cols = nc;
  return v;
}

// ------------------------------------------------------------ embed.cu ---
void launch_gen(cudaStream_t st, const qlra_spec_t& spec, int64_t r0, int64_t c0, int64_t nrows,
                int64_t ncols, const QView& out, bool transposed);

// ------------------------------------------------------------ qgemm.cu ---
void qgemm(Ctx& ctx, int op_a, int op_b, double alpha, const QView& A, const QView& B,
           double beta, const QView& C, int force_splits = 0);
// Split count filling whole waves for `tiles` 64x64 tiles over K (plus
// `other_ctas` CTAs sharing the launch).
int64_t choose_splits(int64_t tiles, int64_t K, int64_t other_ctas);
// C = alpha * sum_{z<nz} ws[z] + beta * C  (ws: [nz][4][rows][cols], fixed order)
void splitk_reduce(Ctx& ctx, const double* ws, int nz, const QView& C, double alpha, double beta);
// d_out2[0] = ||R - H X||_F^2, d_out2[1] = ||R||_F^2 (device pointer)
void qgemm_residual(Ctx& ctx, const QView& R, const QView& H, const QView& X, double* d_out2);

// ----------------------------------------------------------- sketch.cu ---
void sketch_update_rows(Ctx& ctx, const qlra_spec_t& omega, const qlra_spec_t& psi, int64_t row0,
                        const QView& block, const QView& y_rows, const QView& w);
// Same with the block in HOST memory (pinned for full overlap): row panels
// are streamed H2D on a copy stream, double-buffered against the sketch.
void sketch_update_rows_host(Ctx& ctx, const qlra_spec_t& omega, const qlra_spec_t& psi,
                             int64_t row0, const QView& host_block, const QView& y_rows,
                             const QView& w, int64_t block_rows);
const char* sketch_kernel_name();

// Gauss-Jordan with partial pivoting on quaternion A (n x n): B <- A^{-1} B,
// A destroyed.  d_stat[0] = info (0 ok, k+1 = zero pivot at k),
// d_stat[1..2] = min/max pivot norm (doubles via reinterpret).
void small_quat_solve(Ctx& ctx, const QView& a, const QView& b, double* d_stat, bool pivot = true);
// Eigenvalues (descending, n values) of a quaternion Hermitian matrix (a is
// destroyed); extremes_only computes only w[0] (max) and w[n-1] (min).
void small_quat_herm_eigvals(Ctx& ctx, const QView& a, double* d_w, bool extremes_only);
// ||chi_A||_1 into *d_out (device).
void small_chi_norm1(Ctx& ctx, const QView& a, double* d_out);
// out = alpha * I + beta * a   (square)
void small_axpby_identity(Ctx& ctx, double alpha, double beta, const QView& a, const QView& out);
void small_set_identity(Ctx& ctx, const QView& out);
// estimate_epsilon power iterations on chi_{Ginv}: *d_rho (device).
void small_power_iter_inverse(Ctx& ctx, const QView& ginv, int iters, double* d_rho);
// Eigendecomposition of a quaternion Hermitian matrix (a destroyed):
// eigenvalues descending into d_w (device, n), eigenvectors into the columns
// of vecs (n x n, quaternion-orthonormal); parallel cyclic Jacobi, one CTA.
void small_quat_eigh(Ctx& ctx, const QView& a, double* d_w, const QView& vecs, int max_sweeps = 30);
// out(:, j) = a(:, j) * f[j]  (or / f[j] when invert; 0 where f[j] <= floor)
void scale_cols(Ctx& ctx, const QView& a, const double* d_f, bool invert, double floor_v,
                const QView& out);
// out (r x n) = diag(sigma) V^*
void sigma_vadj(Ctx& ctx, const double* d_sigma, const QView& v, const QView& out);
// qsvd phase convention on (U, V) columns (factorizations.cpp:273-293)
void qsvd_phase(Ctx& ctx, const QView& u, const QView& v);
// Blocked quaternion Cholesky G = R^*R (R upper) returning R^{-1} in rinv
// (s x s, fully written), diag(R) and optionally R itself; false if G is not
// numerically PD.
bool blocked_chol_inv(Ctx& ctx, const QView& g, const QView& rinv, std::vector<double>* rdiag,
                      const QView* r_out = nullptr);
// Single-launch cluster Cholesky+inverse for s <= chol_inv_async_max(), no
// host sync: *d_info = 0 or the first failing column (1-based); r may be a
// workspace (R is written there); d_rdiag = diag(R).
int64_t chol_inv_async_max();
void chol_inv_launch(Ctx& ctx, const QView& g, const QView& r, const QView& rinv, int* d_info, double* d_rdiag);
// zero the j, k planes (restrict a quaternion matrix to its complex part)
void zero_jk_planes(Ctx& ctx, const QView& g);
void small_add_diag(Ctx& ctx, const QView& g, double shift);
// dst = src (same shape)
void copy_qmat(Ctx& ctx, const QView& src, const QView& dst);
void scale_add_qmat(Ctx& ctx, double a, const QView& x, double b, const QView& y,
                    const QView& out);  // out = a x + b y

// --------------------------------------------------------------- io.cu ---
void write_qmat(Ctx& ctx, const std::string& path, const QView& m);
void qmat_header(const std::string& path, int64_t* rows, int64_t* cols);
void read_qmat(Ctx& ctx, const std::string& path, const QView& m);
void write_sketch(Ctx& ctx, const std::string& path, const qlra_spec_t& om, const qlra_spec_t& ps,
                  int64_t r, int64_t s, int64_t l, const QView& y, const QView& w);
void sketch_header(const std::string& path, qlra_spec_t* om, qlra_spec_t* ps, int64_t* rsl);
void read_sketch(Ctx& ctx, const std::string& path, const QView& y, const QView& w);
void sketch_from_qmat_file(Ctx& ctx, const std::string& path, const qlra_spec_t& omega,
                           const qlra_spec_t& psi, const QView& y, const QView& w, int64_t block_rows);

// ------------------------------------------------------------- peak.cu ---
double measure_fp64_peak(Ctx& ctx, int mode, double ms);

// ---------------------------------------------------------- collective ---
void allreduce_sum(Ctx& ctx, double* buf, size_t count);
void allreduce_qmat(Ctx& ctx, const QView& m);  // contiguous-ld views only

}  // namespace qlra_dev
