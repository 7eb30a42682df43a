// qgemm.cu -- FP64 quaternion GEMM on the B200 FP64 tensor pipe (DMMA).
//
//   C = alpha * op(A) op(B) + beta * C,   op in {identity, adjoint}
//
// Replaces the 16 real plane GEMMs of qmat_mul (proj/src/qmatrix.cpp:165-197)
// and the ordered triple loop qmat_mul_accumulate_ordered
// (proj/src/qmatrix.cpp:203-242).  The tile core is qtile.cuh (64x64
// quaternion tile per CTA, DMMA.8x8x4, 4-stage cp.async ring).  Split-K
// writes per-split partials to a workspace reduced in fixed split order
// (deterministic, no atomics).  Epilogue variants: store, or residual (sum of
// squares of R - op(A)op(B) and of R, for ||A - HX||_F without forming HX).
#include <algorithm>
#include <array>
#include <map>
#include <mutex>
#include <vector>
#include "common.cuh"
#include "kernels.cuh"
#include "ozaki.cuh"
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
  double* ws;           // split partials [z][4][M][N]  (nullptr if nsplit == 1)
  double* red;          // residual partials [tiles][2]
  // CTA order, longest first: up to 4 groups of tiles (full, then the tiles
  // padded along N / M / both, by decreasing cost), each group's CTAs =
  // its tiles x nsplit, split index fastest, then tile row
  int nsplit, ngroups, tn_all;
  int g_tm0[4], g_tm1[4], g_tn0[4], g_tn1[4];
  int64_t g_start[5];
};

// blockIdx.x -> (tile row, tile column, split)
__device__ __forceinline__ void gemm_task(const GemmArgs& g, int& tm, int& tn, int& z) {
  const int64_t t = blockIdx.x;
  int gi = 0;
  while (gi + 1 < g.ngroups && t >= g.g_start[gi + 1]) ++gi;
  int64_t local = t - g.g_start[gi];
  z = (int)(local % g.nsplit);
  local /= g.nsplit;
  const int nr = g.g_tm1[gi] - g.g_tm0[gi];
  tm = g.g_tm0[gi] + (int)(local % nr);
  tn = g.g_tn0[gi] + (int)(local / nr);
}

template <bool CA, bool CB, int MODE>
__global__ void __launch_bounds__(NT, 1) qgemm_kernel(GemmArgs g) {
  extern __shared__ __align__(16) double smem[];
  const int64_t M = g.op.M, N = g.op.N;
  int tm, tn, zs;
  gemm_task(g, tm, tn, zs);
  if (MODE == 0 && g.op.herm && tm > tn) return;  // lower tile of a Hermitian product: mirrored later
  const int64_t i0 = (int64_t)tm * BM, j0 = (int64_t)tn * BN;
  const int64_t kbeg = (int64_t)zs * g.kchunk;
  const int64_t kend = min(g.K, kbeg + g.kchunk);
  qt::Acc acc;
  qt::zero_acc(acc);
  qt::mma_tile<CA, CB>(g.op, smem, i0, j0, kbeg, kend, acc);

  if (MODE == 0) {
    const bool split = g.nsplit > 1;
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
            double* w = g.ws + (int64_t)zs * 4 * M * N;
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
      const int64_t b = (int64_t)tm * g.tn_all + tn;
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

// ---------------------------------------------------------------------------
// Small products (s x s blocks of the factorisations, s x s x l Grams): a
// 64x64 DMMA tile on one SM is bound by that SM's FP64 rate (~0.25 TF/s), so
// a 100x100x100 quaternion product on 4 CTAs takes ~30 us.  Here every CTA
// owns a 16x16 quaternion output tile (one element per thread, 16 FP64 FMA
// per quaternion MAC on the CUDA cores), K is staged through shared memory
// in chunks of SKC, and K is split over gridDim.z.  Split partials go to a
// workspace; the last CTA to arrive at a tile (per-tile counter) sums them in
// ascending split order -- deterministic -- and applies alpha/beta.
constexpr int STL = 16;   // output tile edge (quaternions)
constexpr int SKC = 32;   // k chunk staged in shared memory

struct SmallArgs {
  qt::Operands op;
  double* c[4];
  int64_t ldc, K, kchunk;
  double alpha, beta;
  double* ws;        // [z][tile][4][256] partials (split only)
  unsigned* cnt;     // [tile] arrival counters
};

template <bool CA, bool CB>
__global__ void __launch_bounds__(256) qgemm_small_kernel(SmallArgs g) {
  __shared__ double as[4][STL][SKC + 1];
  __shared__ double bs[4][SKC][STL + 1];
  __shared__ unsigned s_last;
  const int t = threadIdx.x, ti = t >> 4, tj = t & 15;
  const int64_t M = g.op.M, N = g.op.N;
  const int64_t i0 = (int64_t)blockIdx.y * STL, j0 = (int64_t)blockIdx.x * STL;
  const int64_t kbeg = (int64_t)blockIdx.z * g.kchunk, kend = min(g.K, kbeg + g.kchunk);
  double aw = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
  const double sa = CA ? -1.0 : 1.0, sb = CB ? -1.0 : 1.0;
  for (int64_t k0 = kbeg; k0 < kend; k0 += SKC) {
    // op(A)(i, k) = A[i*a_si + k*a_sk] (conjugated when CA); coalesce along
    // the unit-stride index
    for (int e = t; e < STL * SKC; e += 256) {
      const int r = CA ? (e % STL) : (e / SKC), kk = CA ? (e / STL) : (e % SKC);
      const int64_t gi = i0 + r, gk = k0 + kk;
      const bool ok = gi < M && gk < kend;
      const int64_t o = gi * g.op.a_si + gk * g.op.a_sk;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const double v = ok ? g.op.a[p][o] : 0.0;
        as[p][r][kk] = p == 0 ? v : sa * v;
      }
    }
    for (int e = t; e < SKC * STL; e += 256) {
      const int kk = CB ? (e % SKC) : (e / STL), c = CB ? (e / SKC) : (e % STL);
      const int64_t gk = k0 + kk, gj = j0 + c;
      const bool ok = gk < kend && gj < N;
      const int64_t o = gk * g.op.b_sk + gj * g.op.b_sj;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const double v = ok ? g.op.b[p][o] : 0.0;
        bs[p][kk][c] = p == 0 ? v : sb * v;
      }
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < SKC; ++kk) {
      const double a0 = as[0][ti][kk], a1 = as[1][ti][kk], a2 = as[2][ti][kk], a3 = as[3][ti][kk];
      const double b0 = bs[0][kk][tj], b1 = bs[1][kk][tj], b2 = bs[2][kk][tj], b3 = bs[3][kk][tj];
      aw = fma(a0, b0, aw); aw = fma(-a1, b1, aw); aw = fma(-a2, b2, aw); aw = fma(-a3, b3, aw);
      ax = fma(a0, b1, ax); ax = fma(a1, b0, ax); ax = fma(a2, b3, ax); ax = fma(-a3, b2, ax);
      ay = fma(a0, b2, ay); ay = fma(-a1, b3, ay); ay = fma(a2, b0, ay); ay = fma(a3, b1, ay);
      az = fma(a0, b3, az); az = fma(a1, b2, az); az = fma(-a2, b1, az); az = fma(a3, b0, az);
    }
    __syncthreads();
  }
  const int64_t gi = i0 + ti, gj = j0 + tj;
  const bool in = gi < M && gj < N;
  if (gridDim.z == 1) {
    if (in) {
      const double v[4] = {aw, ax, ay, az};
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        double* dst = g.c[p] + gi * g.ldc + gj;
        const double r = g.alpha * v[p];
        *dst = g.beta != 0.0 ? fma(g.beta, *dst, r) : r;
      }
    }
    return;
  }
  const int64_t tile = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
  const int64_t ntile = (int64_t)gridDim.x * gridDim.y;
  double* w = g.ws + (((int64_t)blockIdx.z * ntile + tile) * 4) * 256;
  w[0 * 256 + t] = aw;
  w[1 * 256 + t] = ax;
  w[2 * 256 + t] = ay;
  w[3 * 256 + t] = az;
  __threadfence();
  __syncthreads();
  if (t == 0) s_last = atomicAdd(&g.cnt[tile], 1u) == gridDim.z - 1 ? 1u : 0u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (in) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      double s = 0.0;
      for (unsigned z = 0; z < gridDim.z; ++z) s += __ldcg(g.ws + ((z * ntile + tile) * 4 + p) * 256 + t);
      double* dst = g.c[p] + gi * g.ldc + gj;
      const double r = g.alpha * s;
      *dst = g.beta != 0.0 ? fma(g.beta, *dst, r) : r;
    }
  }
  if (t == 0) g.cnt[tile] = 0u;  // ready for the next launch on this stream
}

void small_gemm(Ctx& ctx, bool ca, bool cb, const GemmArgs& ga, int64_t M, int64_t N, int64_t K,
                const QView& C) {
  SmallArgs g{};
  g.op = ga.op;
  for (int p = 0; p < 4; ++p) g.c[p] = C.p[p];
  g.ldc = C.ld;
  g.K = K;
  g.alpha = ga.alpha;
  g.beta = ga.beta;
  const int64_t tm = (M + STL - 1) / STL, tn = (N + STL - 1) / STL, tiles = tm * tn;
  // split K to reach about two CTAs per SM, >= 2 chunks of SKC per split
  int64_t z = std::max<int64_t>(1, std::min<int64_t>((296 + tiles - 1) / tiles, K / (2 * SKC)));
  z = std::min<int64_t>(z, 64);
  int64_t kchunk = (K + z - 1) / z;
  kchunk = std::max<int64_t>(SKC, ((kchunk + SKC - 1) / SKC) * SKC);
  z = K > 0 ? (K + kchunk - 1) / kchunk : 1;
  g.kchunk = std::max<int64_t>(kchunk, 1);
  DeviceBuffer ws;
  if (z > 1) {
    if (ctx.tile_cnt_n < tiles) {
      if (ctx.tile_cnt) {
        QLRA_CUDA(cudaStreamSynchronize(ctx.stream));
        QLRA_CUDA(cudaFree(ctx.tile_cnt));
      }
      ctx.tile_cnt_n = std::max<int64_t>(tiles, 4096);
      QLRA_CUDA(cudaMalloc(&ctx.tile_cnt, sizeof(unsigned) * (size_t)ctx.tile_cnt_n));
      QLRA_CUDA(cudaMemsetAsync(ctx.tile_cnt, 0, sizeof(unsigned) * (size_t)ctx.tile_cnt_n, ctx.stream));
    }
    ws = DeviceBuffer(ctx, sizeof(double) * (size_t)(z * tiles * 4 * 256));
    g.ws = ws.as<double>();
    g.cnt = ctx.tile_cnt;
  }
  dim3 grid((unsigned)tn, (unsigned)tm, (unsigned)z);
  if (!ca && !cb) qgemm_small_kernel<false, false><<<grid, 256, 0, ctx.stream>>>(g);
  else if (ca && !cb) qgemm_small_kernel<true, false><<<grid, 256, 0, ctx.stream>>>(g);
  else if (!ca && cb) qgemm_small_kernel<false, true><<<grid, 256, 0, ctx.stream>>>(g);
  else qgemm_small_kernel<true, true><<<grid, 256, 0, ctx.stream>>>(g);
  QLRA_LAUNCH_CHECK();
  count_launch();
}

template <bool CA, bool CB, int MODE>
void set_attr() {
  set_func_attr((const void*)qgemm_kernel<CA, CB, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                (int)qt::SMEM_BYTES);
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
  const int64_t maxs = std::max<int64_t>(1, std::min<int64_t>(296, K / (24 * BK)));
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

namespace {

// Tile groups of an M x N output in 64x64 tiles, by decreasing cost: full
// tiles, then those padded along N / M / both (cost = the fraction of 8x8
// blocks inside M x N -- padded blocks issue no DMMA, qtile.cuh).
struct TileGroup {
  int tm0, tm1, tn0, tn1;
  double cost;
};
std::vector<TileGroup> tile_groups(int64_t M, int64_t N) {
  const int tm = (int)((M + BM - 1) / BM), tn = (int)((N + BN - 1) / BN);
  const int tmf = (int)(M / BM), tnf = (int)(N / BN);
  auto frac = [](int64_t valid) { return (double)((valid + 7) / 8) / 8.0; };
  const double fr = frac(M - (int64_t)tmf * BM), fc = frac(N - (int64_t)tnf * BN);
  std::vector<TileGroup> g;
  if (tmf > 0 && tnf > 0) g.push_back({0, tmf, 0, tnf, 1.0});
  if (tn > tnf && tmf > 0) g.push_back({0, tmf, tnf, tn, fc});
  if (tm > tmf && tnf > 0) g.push_back({tmf, tm, 0, tnf, fr});
  if (tm > tmf && tn > tnf) g.push_back({tmf, tm, tnf, tn, fr * fc});
  std::stable_sort(g.begin(), g.end(), [](const TileGroup& a, const TileGroup& b) { return a.cost > b.cost; });
  return g;
}

// Makespan (in k-steps of a full tile) of the launch under greedy list
// scheduling on 148 SMs, CTAs in kernel order; plus the split-K reduction.
double simulate_gemm(const std::vector<TileGroup>& groups, int64_t M, int64_t N, int64_t K, int64_t z) {
  const int64_t kc = ((K + z - 1) / z + BK - 1) / BK * BK;
  const int64_t nz = (K + kc - 1) / kc;
  std::map<double, int64_t> sm{{0.0, 148}};
  for (const TileGroup& g : groups) {
    const double d = (double)(kc / BK) * g.cost + 3.0;  // + prologue / epilogue
    int64_t c = (int64_t)(g.tm1 - g.tm0) * (g.tn1 - g.tn0) * nz;
    while (c > 0) {
      auto it = sm.begin();
      const double t0 = it->first;
      const int64_t k = it->second;
      sm.erase(it);
      const int64_t take = std::min(c, k);
      if (k > take) sm[t0] += k - take;
      sm[t0 + d] += take;
      c -= take;
    }
  }
  const double red = nz > 1 ? (double)nz * (double)M * (double)N * 32.0 / 25e6 : 0.0;
  return sm.rbegin()->first + red;
}

int64_t choose_gemm_splits(int64_t M, int64_t N, int64_t K) {
  static std::mutex mu;
  static std::map<std::array<int64_t, 3>, int64_t> cache;
  const std::array<int64_t, 3> key{M, N, K};
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  const std::vector<TileGroup> groups = tile_groups(M, N);
  const int64_t maxs = std::max<int64_t>(1, std::min<int64_t>(296, K / (8 * BK)));
  int64_t best = 1;
  double best_t = 1e300;
  for (int64_t z = 1; z <= maxs; z = z < 16 ? z + 1 : std::max(z + 1, z * 9 / 8)) {
    const double t = simulate_gemm(groups, M, N, K, z);
    if (t < best_t - 1e-9) {
      best_t = t;
      best = z;
    }
  }
  std::lock_guard<std::mutex> lock(mu);
  cache[key] = best;
  return best;
}

// Fill the CTA schedule of g (groups in cost order, nsplit CTAs per tile);
// returns the number of CTAs.
int64_t fill_schedule(GemmArgs& g, int64_t M, int64_t N, int nsplit) {
  const std::vector<TileGroup> groups = tile_groups(M, N);
  g.nsplit = nsplit;
  g.ngroups = (int)groups.size();
  g.tn_all = (int)((N + BN - 1) / BN);
  int64_t start = 0;
  for (int i = 0; i < g.ngroups; ++i) {
    g.g_tm0[i] = groups[i].tm0;
    g.g_tm1[i] = groups[i].tm1;
    g.g_tn0[i] = groups[i].tn0;
    g.g_tn1[i] = groups[i].tn1;
    g.g_start[i] = start;
    start += (int64_t)(groups[i].tm1 - groups[i].tm0) * (groups[i].tn1 - groups[i].tn0) * nsplit;
  }
  g.g_start[g.ngroups] = start;
  return start;
}

}  // namespace

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

// C(i, j) = conj(C(j, i)) for i > j: completes a Hermitian product of
// which only the upper triangle was computed.
__global__ void k_mirror_upper(QView c) {
  const int64_t n = c.rows;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / n, j = t % n;
    if (i <= j) continue;
    const int64_t src = j * c.ld + i, dst = i * c.ld + j;
    c.p[0][dst] = c.p[0][src];
    c.p[1][dst] = -c.p[1][src];
    c.p[2][dst] = -c.p[2][src];
    c.p[3][dst] = -c.p[3][src];
  }
}

void qgemm(Ctx& ctx, int op_a, int op_b, double alpha, const QView& A, const QView& B,
           double beta, const QView& C, int force_splits) {
  qgemm_ex(ctx, op_a, op_b, alpha, A, B, beta, C, force_splits, false);
}

// C = A^* A (Hermitian): on the 64x64 DMMA path only the tiles and warp
// tiles on or above the diagonal are computed and the rest is mirrored
// (about half the tensor work of a Gram; exactly Hermitian result).
void qgemm_gram(Ctx& ctx, const QView& A, const QView& C) {
  if (oz_gemm_try(ctx, QLRA_OP_C, QLRA_OP_N, 1.0, A, A, 0.0, C)) return;  // long K: exact int8 products
  if (q8gram(ctx, A, C)) return;  // tall A: 8 real products per MAC (qtile8.cuh mode 4)
  qgemm_ex(ctx, QLRA_OP_C, QLRA_OP_N, 1.0, A, A, 0.0, C, 0, true);
}

void mirror_upper(Ctx& ctx, const QView& C) {
  const int64_t M = C.rows;
  k_mirror_upper<<<(unsigned)std::min<int64_t>((M * M + 255) / 256, 148 * 4), 256, 0, ctx.stream>>>(C);
  QLRA_LAUNCH_CHECK();
  count_launch();
}

void qgemm_ex(Ctx& ctx, int op_a, int op_b, double alpha, const QView& A, const QView& B,
              double beta, const QView& C, int force_splits, bool herm) {
  int64_t M, N, K;
  GemmArgs g = make_args(op_a, op_b, alpha, A, B, beta, M, N, K);
  if (C.rows != M || C.cols != N) fail(QLRA_ERR_SHAPE, "qmat_mul: output shape mismatch");
  if (M == 0 || N == 0) return;
  // long contractions (K >= 4096, large output): exact int8 products
  if (!herm && force_splits == 0 && oz_gemm_try(ctx, op_a, op_b, alpha, A, B, beta, C)) return;
  for (int p = 0; p < 4; ++p) g.c[p] = C.p[p];
  g.ldc = C.ld;
  const int64_t tm = (M + BM - 1) / BM, tn = (N + BN - 1) / BN;
  const int64_t tiles = tm * tn;
  // Small products: the 64x64 DMMA tiles (+ split-K of >= 24 k-steps) cannot
  // fill the GPU -- use the 16x16-tile path (CUDA cores), unless the product
  // is big enough for the tensor tiles to win anyway (C4's 500 x 500 x 500:
  // 240 us on the small path; QLRA_SMALL_GEMM_MAX tunes the cut in M N K)
  static const double small_max = [] {
    const char* e = std::getenv("QLRA_SMALL_GEMM_MAX");
    return e ? std::atof(e) : 6.4e7;
  }();
  if (force_splits <= 0 && K > 0 && tiles * std::max<int64_t>(1, K / (24 * BK)) < 148 &&
      (double)M * (double)N * (double)K < small_max) {
    small_gemm(ctx, op_a == QLRA_OP_C, op_b == QLRA_OP_C, g, M, N, K, C);
    return;
  }
  // tall x small / small x tall products (an adjoint only on the small
  // factor): 8 real products per quaternion MAC instead of 16 (qtile8.cuh)
  if (force_splits <= 0 && !herm && q8gemm_try(ctx, op_a, op_b, alpha, A, B, beta, C)) return;
  int64_t nsplit = 1;
  if (force_splits > 0) {
    nsplit = force_splits;
  } else if (K > 0) {
    nsplit = choose_gemm_splits(M, N, K);
  }
  int64_t kchunk = (K + nsplit - 1) / nsplit;
  kchunk = ((kchunk + BK - 1) / BK) * BK;
  if (kchunk == 0) kchunk = BK;
  nsplit = K > 0 ? (K + kchunk - 1) / kchunk : 1;
  g.kchunk = kchunk;
  const int64_t ctas = fill_schedule(g, M, N, (int)nsplit);
  dim3 grid((unsigned)ctas);
  g.op.herm = herm && M == N && beta == 0.0 ? 1 : 0;
  if (nsplit > 1) {
    DeviceBuffer ws(ctx, (size_t)nsplit * 4 * M * N * sizeof(double));
    g.ws = ws.as<double>();
    dispatch<0>(op_a == QLRA_OP_C, op_b == QLRA_OP_C, grid, ctx.stream, g);
    splitk_reduce(ctx, g.ws, (int)nsplit, C, alpha, beta);
  } else {
    dispatch<0>(op_a == QLRA_OP_C, op_b == QLRA_OP_C, grid, ctx.stream, g);
  }
  if (g.op.herm) {
    k_mirror_upper<<<(unsigned)std::min<int64_t>((M * M + 255) / 256, 148 * 4), 256, 0, ctx.stream>>>(C);
    QLRA_LAUNCH_CHECK();
    count_launch();
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
  if (M > 0 && N > 0) {
    dim3 grid((unsigned)fill_schedule(g, M, N, 1));
    dispatch<1>(false, false, grid, ctx.stream, g);
  }
  residual_finish_kernel<<<1, 32, 0, ctx.stream>>>(g.red, tm * tn, d_out2);
  QLRA_LAUNCH_CHECK();
  count_launch();
}

}  // namespace qlra_dev
