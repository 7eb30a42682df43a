// qgemm.cu -- FP64 quaternion GEMM on the B200 FP64 tensor pipe (DMMA).
//
//   C = alpha * op(A) op(B) + beta * C,   op in {identity, adjoint}
//
// Replaces the 16 real plane GEMMs of qmat_mul (proj/src/qmatrix.cpp:165-197)
// and the ordered triple loop qmat_mul_accumulate_ordered
// (proj/src/qmatrix.cpp:203-242).  The tile core is qtile.cuh (64x64
// quaternion tile per CTA, DMMA.8x8x4, 3-stage cp.async ring).  Split-K
// writes per-split partials to a workspace reduced in fixed split order
// (deterministic, no atomics).  Epilogue variants: store, or residual (sum of
// squares of R - op(A)op(B) and of R, for ||A - HX||_F without forming HX).
#include "common.cuh"
#include "kernels.cuh"
#include "qtile.cuh"

namespace qlra_dev {

namespace {

using qt::BM;
using qt::BN;
using qt::BK;
using qt::NT;

struct GemmArgs {
  qt::Operands op;
  double* c[4];
  const double* r[4];   // residual reference (mode 1)
  int64_t K;
  int64_t ldc, ldr;
  double alpha, beta;
  int64_t kchunk;       // k range per split (multiple of BK)
  double* ws;           // split partials [z][4][M][N]  (nullptr if gridDim.z == 1)
  double* red;          // residual partials [blocks][2]
};

template <bool CA, bool CB, int MODE>
__global__ void __launch_bounds__(NT, 1) qgemm_kernel(GemmArgs g) {
  extern __shared__ __align__(16) double smem[];
  const int64_t M = g.op.M, N = g.op.N;
  const int64_t i0 = (int64_t)blockIdx.y * BM, j0 = (int64_t)blockIdx.x * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * g.kchunk;
  const int64_t kend = min(g.K, kbeg + g.kchunk);
  qt::Acc acc;
  qt::zero_acc(acc);
  qt::mma_tile<CA, CB>(g.op, smem, i0, j0, kbeg, kend, acc);

  if (MODE == 0) {
    const bool split = gridDim.z > 1;
#pragma unroll
    for (int rb = 0; rb < qt::WRB; ++rb) {
      const int64_t gi = i0 + qt::acc_row(rb);
      if (gi >= M) continue;
#pragma unroll
      for (int cb = 0; cb < qt::WCB; ++cb)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t gj = j0 + qt::acc_col(cb) + h;
          if (gj >= N) continue;
          if (split) {
            double* w = g.ws + (int64_t)blockIdx.z * 4 * M * N;
#pragma unroll
            for (int p = 0; p < 4; ++p) w[(int64_t)p * M * N + gi * N + gj] = acc[rb][cb][p][h];
          } else {
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              double* dst = g.c[p] + gi * g.ldc + gj;
              const double v = g.alpha * acc[rb][cb][p][h];
              *dst = g.beta != 0.0 ? fma(g.beta, *dst, v) : v;
            }
          }
        }
    }
  } else {
    // residual epilogue: sum over the tile of (R - alpha*acc)^2 and R^2.
    double rs = 0.0, as = 0.0;
#pragma unroll
    for (int rb = 0; rb < qt::WRB; ++rb) {
      const int64_t gi = i0 + qt::acc_row(rb);
#pragma unroll
      for (int cb = 0; cb < qt::WCB; ++cb)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t gj = j0 + qt::acc_col(cb) + h;
          if (gi < M && gj < N) {
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              const double ref = g.r[p][gi * g.ldr + gj];
              const double d = ref - g.alpha * acc[rb][cb][p][h];
              rs = fma(d, d, rs);
              as = fma(ref, ref, as);
            }
          }
        }
    }
    __syncthreads();  // smem ring reused as reduction scratch
    double* red = smem;
    const int tid = threadIdx.x;
    red[tid] = rs;
    red[NT + tid] = as;
    __syncthreads();
    for (int w = NT / 2; w > 0; w >>= 1) {
      if (tid < w) {
        red[tid] += red[tid + w];
        red[NT + tid] += red[NT + tid + w];
      }
      __syncthreads();
    }
    if (tid == 0) {
      const int64_t b = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
      g.red[2 * b] = red[0];
      g.red[2 * b + 1] = red[NT];
    }
  }
}

// C = alpha * sum_z ws[z] + beta * C, summed in ascending z (deterministic).
__global__ void splitk_reduce_kernel(const double* ws, int nz, int64_t M, int64_t N, double* c0,
                                     double* c1, double* c2, double* c3, int64_t ldc, double alpha,
                                     double beta) {
  const int64_t total = 4 * M * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(e / (M * N));
    const int64_t rem = e % (M * N);
    const int64_t i = rem / N, j = rem % N;
    double s = 0.0;
    for (int z = 0; z < nz; ++z) s += ws[(int64_t)z * 4 * M * N + e];
    double* c = p == 0 ? c0 : p == 1 ? c1 : p == 2 ? c2 : c3;
    double* dst = c + i * ldc + j;
    const double v = alpha * s;
    *dst = beta != 0.0 ? fma(beta, *dst, v) : v;
  }
}

__global__ void residual_finish_kernel(const double* red, int64_t nblocks, double* out) {
  // single thread, fixed order
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double rs = 0.0, as = 0.0;
    for (int64_t b = 0; b < nblocks; ++b) {
      rs += red[2 * b];
      as += red[2 * b + 1];
    }
    out[0] = rs;
    out[1] = as;
  }
}

template <bool CA, bool CB, int MODE>
void set_attr() {
  static bool done = false;
  if (!done) {
    QLRA_CUDA(cudaFuncSetAttribute(qgemm_kernel<CA, CB, MODE>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qt::SMEM_BYTES));
    done = true;
  }
}

template <int MODE>
void dispatch(bool ca, bool cb, dim3 grid, cudaStream_t st, const GemmArgs& g) {
  if (!ca && !cb) { set_attr<false, false, MODE>(); qgemm_kernel<false, false, MODE><<<grid, NT, qt::SMEM_BYTES, st>>>(g); }
  else if (ca && !cb) { set_attr<true, false, MODE>(); qgemm_kernel<true, false, MODE><<<grid, NT, qt::SMEM_BYTES, st>>>(g); }
  else if (!ca && cb) { set_attr<false, true, MODE>(); qgemm_kernel<false, true, MODE><<<grid, NT, qt::SMEM_BYTES, st>>>(g); }
  else { set_attr<true, true, MODE>(); qgemm_kernel<true, true, MODE><<<grid, NT, qt::SMEM_BYTES, st>>>(g); }
  QLRA_LAUNCH_CHECK();
  count_launch();
}

GemmArgs make_args(int op_a, int op_b, double alpha, const QView& A, const QView& B, double beta,
                   int64_t& M, int64_t& N, int64_t& K) {
  GemmArgs g{};
  M = op_a == QLRA_OP_N ? A.rows : A.cols;
  K = op_a == QLRA_OP_N ? A.cols : A.rows;
  const int64_t Kb = op_b == QLRA_OP_N ? B.rows : B.cols;
  N = op_b == QLRA_OP_N ? B.cols : B.rows;
  if (K != Kb) fail(QLRA_ERR_SHAPE, "qmat_mul: inner dimensions differ");
  for (int p = 0; p < 4; ++p) {
    g.op.a[p] = A.p[p];
    g.op.b[p] = B.p[p];
  }
  if (op_a == QLRA_OP_N) { g.op.a_si = A.ld; g.op.a_sk = 1; } else { g.op.a_si = 1; g.op.a_sk = A.ld; }
  if (op_b == QLRA_OP_N) { g.op.b_sk = B.ld; g.op.b_sj = 1; } else { g.op.b_sk = 1; g.op.b_sj = B.ld; }
  g.op.M = M;
  g.op.N = N;
  g.K = K;
  g.alpha = alpha;
  g.beta = beta;
  return g;
}

}  // namespace

int64_t choose_splits(int64_t tiles, int64_t K, int64_t other_ctas) {
  // Split K so the launch fills whole waves of 148 SMs (1 CTA/SM): maximise
  // ctas / (waves * 148) with a small per-split penalty, >= 24 k-steps each.
  const int64_t maxs = std::max<int64_t>(1, std::min<int64_t>(64, K / (24 * BK)));
  int64_t best = 1;
  double best_score = -1.0;
  for (int64_t z = 1; z <= maxs; ++z) {
    const int64_t ctas = tiles * z + other_ctas;
    const int64_t waves = (ctas + 147) / 148;
    const double score = (double)ctas / (double)(waves * 148) - 0.004 * (double)(z - 1);
    if (score > best_score + 1e-12) {
      best_score = score;
      best = z;
    }
  }
  return best;
}

void splitk_reduce(Ctx& ctx, const double* ws, int nz, const QView& C, double alpha, double beta) {
  const int64_t total = 4 * C.rows * C.cols;
  if (total == 0) return;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((total + threads - 1) / threads, 148 * 8);
  splitk_reduce_kernel<<<(unsigned)blocks, threads, 0, ctx.stream>>>(
      ws, nz, C.rows, C.cols, C.p[0], C.p[1], C.p[2], C.p[3], C.ld, alpha, beta);
  QLRA_LAUNCH_CHECK();
  count_launch();
}

void qgemm(Ctx& ctx, int op_a, int op_b, double alpha, const QView& A, const QView& B,
           double beta, const QView& C, int force_splits) {
  int64_t M, N, K;
  GemmArgs g = make_args(op_a, op_b, alpha, A, B, beta, M, N, K);
  if (C.rows != M || C.cols != N) fail(QLRA_ERR_SHAPE, "qmat_mul: output shape mismatch");
  if (M == 0 || N == 0) return;
  for (int p = 0; p < 4; ++p) g.c[p] = C.p[p];
  g.ldc = C.ld;
  const int64_t tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
  const int64_t tiles = tm * tn;
  int64_t nsplit = 1;
  if (force_splits > 0) {
    nsplit = force_splits;
  } else if (K > 0) {
    nsplit = choose_splits(tiles, K, 1);
  }
  int64_t kchunk = (K + nsplit - 1) / nsplit;
  kchunk = ((kchunk + BK - 1) / BK) * BK;
  if (kchunk == 0) kchunk = BK;
  nsplit = K > 0 ? (K + kchunk - 1) / kchunk : 1;
  g.kchunk = kchunk;
  dim3 grid((unsigned)tn, (unsigned)tm, (unsigned)nsplit);
  if (nsplit > 1) {
    DeviceBuffer ws(ctx, (size_t)nsplit * 4 * M * N * sizeof(double));
    g.ws = ws.as<double>();
    dispatch<0>(op_a == QLRA_OP_C, op_b == QLRA_OP_C, grid, ctx.stream, g);
    splitk_reduce(ctx, g.ws, (int)nsplit, C, alpha, beta);
  } else {
    dispatch<0>(op_a == QLRA_OP_C, op_b == QLRA_OP_C, grid, ctx.stream, g);
  }
}

void qgemm_residual(Ctx& ctx, const QView& R, const QView& H, const QView& X, double* d_out2) {
  int64_t M, N, K;
  GemmArgs g = make_args(QLRA_OP_N, QLRA_OP_N, 1.0, H, X, 0.0, M, N, K);
  if (R.rows != M || R.cols != N) fail(QLRA_ERR_SHAPE, "residual: A and HX differ in shape");
  for (int p = 0; p < 4; ++p) g.r[p] = R.p[p];
  g.ldr = R.ld;
  const int64_t tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
  g.kchunk = ((K + BK - 1) / BK) * BK;
  if (g.kchunk == 0) g.kchunk = BK;
  DeviceBuffer red(ctx, (size_t)tm * tn * 2 * sizeof(double));
  g.red = red.as<double>();
  dim3 grid((unsigned)tn, (unsigned)tm, 1);
  if (M > 0 && N > 0) dispatch<1>(false, false, grid, ctx.stream, g);
  residual_finish_kernel<<<1, 32, 0, ctx.stream>>>(g.red, tm * tn, d_out2);
  QLRA_LAUNCH_CHECK();
  count_launch();
}

}  // namespace qlra_dev
