// qgemm.cu -- FP64 quaternion GEMM on the B200 DFMA pipe.
//
//   C = alpha * op(A) op(B) + beta * C,   op in {identity, adjoint}
//
// Replaces the 16 real plane GEMMs of qmat_mul (proj/src/qmatrix.cpp:165-197)
// and the ordered triple loop qmat_mul_accumulate_ordered
// (proj/src/qmatrix.cpp:203-242) used by both sketches.  One qMAC is the
// Hamilton product table (proj/include/qlra/quaternion.hpp:33-38) = 16 DFMAs
// whose operand negations are free SASS modifiers, so the quaternion product
// costs exactly the reference's 32 flop/qMAC with no sign materialisation.
// (tcgen05 has no f64 kind and DMMA.8x8x4 would need negated operand copies;
// SURVEY.md F7 / H1.)
//
// Tiling: 64x64 quaternion output tile per 256-thread CTA, 4x4 quaternion
// micro-tile per thread (64 FP64 accumulators), BK = 8 quaternion k-steps per
// stage, 3-stage cp.async pipeline, operands staged k-major in shared memory
// so every compute-side read is an LDS.128.  Split-K writes per-split
// partials to a workspace reduced in fixed split order (deterministic, no
// atomics).  Epilogue variants: store, or residual (sum of squares of
// R - op(A)op(B) and of R, for ||A - HX||_F without materialising HX).
#include "common.cuh"
#include "kernels.cuh"

namespace qlra_dev {

namespace {

constexpr int BM = 64, BN = 64, BK = 8, TM = 4, TN = 4, NT = 256, STAGES = 3;
constexpr int A_STAGE = 4 * BK * BM;  // doubles per stage
constexpr int B_STAGE = 4 * BK * BN;
constexpr size_t SMEM_BYTES = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double);

struct GemmArgs {
  const double* a[4];
  const double* b[4];
  double* c[4];
  const double* r[4];   // residual reference (mode 1)
  int64_t M, N, K;
  int64_t a_si, a_sk;   // op(A)(i,k) = A.p[.][i*a_si + k*a_sk]
  int64_t b_sk, b_sj;   // op(B)(k,j) = B.p[.][k*b_sk + j*b_sj]
  int64_t ldc, ldr;
  double alpha, beta;
  int64_t kchunk;       // k range per split (multiple of BK)
  double* ws;           // split partials [z][4][M][N]  (nullptr if gridDim.z == 1)
  double* red;          // residual partials [blocks][2]
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Loads one BK-slice of op(A) (BM x BK) and op(B) (BK x BN) into a stage.
__device__ __forceinline__ void load_stage(const GemmArgs& g, double* As, double* Bs, int64_t i0,
                                           int64_t j0, int64_t k0, int64_t kend, int tid) {
  // A: 4 planes x BM x BK = 2048 doubles, 8 per thread.
  const bool a_kfast = (g.a_sk == 1);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int e = tid + NT * r;
    const int p = e >> 9;  // / 512
    const int idx = e & 511;
    int i, k;
    if (a_kfast) { i = idx >> 3; k = idx & 7; }
    else         { i = idx & 63; k = idx >> 6; }
    const int64_t gi = i0 + i, gk = k0 + k;
    const bool ok = gi < g.M && gk < kend;
    const double* src = ok ? g.a[p] + gi * g.a_si + gk * g.a_sk : g.a[p];
    cp_async8(As + (p * BK + k) * BM + i, src, ok);
  }
  const bool b_jfast = (g.b_sj == 1);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int e = tid + NT * r;
    const int p = e >> 9;
    const int idx = e & 511;
    int j, k;
    if (b_jfast) { j = idx & 63; k = idx >> 6; }
    else         { j = idx >> 3; k = idx & 7; }
    const int64_t gj = j0 + j, gk = k0 + k;
    const bool ok = gj < g.N && gk < kend;
    const double* src = ok ? g.b[p] + gk * g.b_sk + gj * g.b_sj : g.b[p];
    cp_async8(Bs + (p * BK + k) * BN + j, src, ok);
  }
}

template <bool CA, bool CB, int MODE>
__global__ void __launch_bounds__(NT, 1) qgemm_kernel(GemmArgs g) {
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = smem + STAGES * A_STAGE;

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t i0 = (int64_t)blockIdx.y * BM, j0 = (int64_t)blockIdx.x * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * g.kchunk;
  const int64_t kend = min(g.K, kbeg + g.kchunk);
  const int nk = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;

  double acc[4][TM][TN];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int r = 0; r < TM; ++r)
#pragma unroll
      for (int c = 0; c < TN; ++c) acc[p][r][c] = 0.0;

  // prologue
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(g, As + s * A_STAGE, Bs + s * B_STAGE, i0, j0, kbeg + s * BK, kend, tid);
    cp_async_commit();
  }

  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kt + STAGES - 1;
      if (nxt < nk) {
        const int s = nxt % STAGES;
        load_stage(g, As + s * A_STAGE, Bs + s * B_STAGE, i0, j0, kbeg + (int64_t)nxt * BK, kend, tid);
      }
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * A_STAGE;
    const double* bs = Bs + (kt % STAGES) * B_STAGE;
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      double a[4][TM], b[4][TN];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const double2* ap = reinterpret_cast<const double2*>(as + (p * BK + k) * BM + ty * TM);
        const double2* bp = reinterpret_cast<const double2*>(bs + (p * BK + k) * BN + tx * TN);
        const double2 a01 = ap[0], a23 = ap[1], b01 = bp[0], b23 = bp[1];
        a[p][0] = a01.x; a[p][1] = a01.y; a[p][2] = a23.x; a[p][3] = a23.y;
        b[p][0] = b01.x; b[p][1] = b01.y; b[p][2] = b23.x; b[p][3] = b23.y;
      }
      if (CA) {
#pragma unroll
        for (int r = 0; r < TM; ++r) { a[1][r] = -a[1][r]; a[2][r] = -a[2][r]; a[3][r] = -a[3][r]; }
      }
      if (CB) {
#pragma unroll
        for (int c = 0; c < TN; ++c) { b[1][c] = -b[1][c]; b[2][c] = -b[2][c]; b[3][c] = -b[3][c]; }
      }
#pragma unroll
      for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int c = 0; c < TN; ++c) {
          const double aw = a[0][r], ax = a[1][r], ay = a[2][r], az = a[3][r];
          const double bw = b[0][c], bx = b[1][c], by = b[2][c], bz = b[3][c];
          acc[0][r][c] = fma(aw, bw, acc[0][r][c]);
          acc[0][r][c] = fma(-ax, bx, acc[0][r][c]);
          acc[0][r][c] = fma(-ay, by, acc[0][r][c]);
          acc[0][r][c] = fma(-az, bz, acc[0][r][c]);
          acc[1][r][c] = fma(aw, bx, acc[1][r][c]);
          acc[1][r][c] = fma(ax, bw, acc[1][r][c]);
          acc[1][r][c] = fma(ay, bz, acc[1][r][c]);
          acc[1][r][c] = fma(-az, by, acc[1][r][c]);
          acc[2][r][c] = fma(aw, by, acc[2][r][c]);
          acc[2][r][c] = fma(-ax, bz, acc[2][r][c]);
          acc[2][r][c] = fma(ay, bw, acc[2][r][c]);
          acc[2][r][c] = fma(az, bx, acc[2][r][c]);
          acc[3][r][c] = fma(aw, bz, acc[3][r][c]);
          acc[3][r][c] = fma(ax, by, acc[3][r][c]);
          acc[3][r][c] = fma(-ay, bx, acc[3][r][c]);
          acc[3][r][c] = fma(az, bw, acc[3][r][c]);
        }
    }
  }
  cp_async_wait<0>();

  if (MODE == 0) {
    const bool split = gridDim.z > 1;
#pragma unroll
    for (int r = 0; r < TM; ++r) {
      const int64_t gi = i0 + ty * TM + r;
      if (gi >= g.M) continue;
#pragma unroll
      for (int c = 0; c < TN; ++c) {
        const int64_t gj = j0 + tx * TN + c;
        if (gj >= g.N) continue;
        if (split) {
          double* w = g.ws + (int64_t)blockIdx.z * 4 * g.M * g.N;
#pragma unroll
          for (int p = 0; p < 4; ++p) w[(int64_t)p * g.M * g.N + gi * g.N + gj] = acc[p][r][c];
        } else {
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            double* dst = g.c[p] + gi * g.ldc + gj;
            const double v = g.alpha * acc[p][r][c];
            *dst = g.beta != 0.0 ? fma(g.beta, *dst, v) : v;
          }
        }
      }
    }
  } else {
    // residual epilogue: sum over the tile of (R - alpha*acc)^2 and R^2.
    double rs = 0.0, as = 0.0;
#pragma unroll
    for (int r = 0; r < TM; ++r) {
      const int64_t gi = i0 + ty * TM + r;
#pragma unroll
      for (int c = 0; c < TN; ++c) {
        const int64_t gj = j0 + tx * TN + c;
        if (gi < g.M && gj < g.N) {
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const double ref = g.r[p][gi * g.ldr + gj];
            const double d = ref - g.alpha * acc[p][r][c];
            rs = fma(d, d, rs);
            as = fma(ref, ref, as);
          }
        }
      }
    }
    __shared__ double red[2][NT];
    red[0][tid] = rs;
    red[1][tid] = as;
    __syncthreads();
    for (int w = NT / 2; w > 0; w >>= 1) {
      if (tid < w) {
        red[0][tid] += red[0][tid + w];
        red[1][tid] += red[1][tid + w];
      }
      __syncthreads();
    }
    if (tid == 0) {
      const int64_t b = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
      g.red[2 * b] = red[0][0];
      g.red[2 * b + 1] = red[1][0];
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
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES));
    done = true;
  }
}

template <int MODE>
void dispatch(bool ca, bool cb, dim3 grid, cudaStream_t st, const GemmArgs& g) {
  if (!ca && !cb) { set_attr<false, false, MODE>(); qgemm_kernel<false, false, MODE><<<grid, NT, SMEM_BYTES, st>>>(g); }
  else if (ca && !cb) { set_attr<true, false, MODE>(); qgemm_kernel<true, false, MODE><<<grid, NT, SMEM_BYTES, st>>>(g); }
  else if (!ca && cb) { set_attr<false, true, MODE>(); qgemm_kernel<false, true, MODE><<<grid, NT, SMEM_BYTES, st>>>(g); }
  else { set_attr<true, true, MODE>(); qgemm_kernel<true, true, MODE><<<grid, NT, SMEM_BYTES, st>>>(g); }
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
    g.a[p] = A.p[p];
    g.b[p] = B.p[p];
  }
  if (op_a == QLRA_OP_N) { g.a_si = A.ld; g.a_sk = 1; } else { g.a_si = 1; g.a_sk = A.ld; }
  if (op_b == QLRA_OP_N) { g.b_sk = B.ld; g.b_sj = 1; } else { g.b_sk = 1; g.b_sj = B.ld; }
  g.M = M; g.N = N; g.K = K;
  g.alpha = alpha;
  g.beta = beta;
  return g;
}

}  // namespace

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
    // Fill ~2 waves of 148 SMs while keeping >= 32 k-steps per split.
    const int64_t want = (2 * 148 + tiles - 1) / tiles;
    const int64_t maxs = std::max<int64_t>(1, K / (32 * BK));
    nsplit = std::min(want, maxs);
    if (nsplit < 1) nsplit = 1;
    if (nsplit > 64) nsplit = 64;
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
    const int64_t total = 4 * M * N;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((total + threads - 1) / threads, 148 * 8);
    splitk_reduce_kernel<<<(unsigned)blocks, threads, 0, ctx.stream>>>(
        g.ws, (int)nsplit, M, N, C.p[0], C.p[1], C.p[2], C.p[3], C.ld, alpha, beta);
    QLRA_LAUNCH_CHECK();
    count_launch();
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
