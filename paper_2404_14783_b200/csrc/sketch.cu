// sketch.cu -- K1+K2: the fused dual sketch  Y += A Omega,  W += Psi A.
//
// Replaces sketch_update_rows (proj/src/sketching.cpp:125-139):
// gen_test_matrix(Omega) + qmat_mul_accumulate_ordered(Y, A, Omega) +
// gen_test_matrix_cols(Psi, rows) + qmat_mul_accumulate_ordered(W, Psi, A).
//
// The block of A is walked in row panels of up to 2 GB (one launch for C2).
// Each panel is ONE launch of sketch8_kernel (8 real products per
// quaternion MAC, qtile8.cuh) whose CTAs are either Y-tasks (tiles of
// Y_panel = A_panel * Omega~ over a K-chunk of the n columns) or W-tasks
// (tiles of W += Psi~[:, panel] * A_panel over a chunk of the panel rows);
// Omega~ / Psi~ are the embeddings' 8 plane combinations, formed once per
// call.  A is never rewritten: its tiles are staged by TMA (one producer
// warp) and combined in registers.  The kernel does ~300 flop per byte of
// A, so the re-reads of an unsplit panel by the tiles that share it cost no
// time on this FP64-bound path.  Split-K partials go
// to workspaces reduced in fixed order afterwards: deterministic, no
// atomics.  Omega (n x s) and the Psi column slice (l x b) are generated on
// device by K1 (embed.cu) from the reference's counter RNG.  The same
// engine (launch8) runs the tall x small products of the rangefinders and
// the core solve, and the Grams (gram8_kernel).  (The 16-product sketch
// kernel of round 1 is gone: the 16-product engine, qtile.cuh, now only
// serves qgemm.cu's products.)
#include <array>
#include <cmath>
#include <cstring>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <type_traits>
#include <vector>

#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.cuh"
#include "ozaki.cuh"
#include "qtile.cuh"
#include "qtile8.cuh"

namespace qlra_dev {

namespace {

using qt::BK;
using qt::BM;
using qt::BN;
using qt::NT;

// ---- the 8-product path (qtile8.cuh) --------------------------------------
// Y-tasks: 64x32 tiles of A * Omega~; W-tasks: 32x64 tiles of Psi~ * A.
constexpr int Y8M = qt8::Cfg<0>::TM, Y8N = qt8::Cfg<0>::TN;
constexpr int W8M = qt8::Cfg<1>::TM, W8N = qt8::Cfg<1>::TN;
constexpr int YNM = qt8::Cfg<2>::TM, YNN = qt8::Cfg<2>::TN;  // narrow remainder tiles
constexpr int WNM = qt8::Cfg<3>::TM, WNN = qt8::Cfg<3>::TN;

struct Fused8Args {
  // TMA maps (sketch8_kernel<true>): Y left = A panel, Y right = Omega~,
  // W left = Psi~ panel, W right = A panel (3D: inner, rows, planes)
  CUtensorMap ylm, yrm, wlm, wrm;
  CUtensorMap ynlm, ynrm, wnlm, wnrm;  // the narrow remainder tiles (modes 2 / 3)
  int stages, stride;  // TMA ring slots and doubles per slot
  int yn_t, wn_t;  // narrow remainder tiles: YN row tiles, WN column tiles (0: none)
  int y_ilv;       // Y and YN tiles interleaved by 128-row block (QLRA_Y_INTERLEAVE)
  int y_rep;       // consecutive Y row tiles per CTA (stream_tiles, small K; 1: one tile)
  qt8::Operands yop;  // A_panel (k-fast) x Omega~ (8 planes, j-fast): M = panel rows, N = s, K = n
  qt8::Operands wop;  // Psi~_panel (8 planes, k-fast) x A_panel (j-fast): M = l, N = n, K = panel rows
  int64_t ky, kw;
  int y_tm, y_tn, zy;
  int64_t ky_chunk;
  int w_tm, w_tn, zw;
  int64_t kw_chunk;
  int y_tnf, w_tmf;
  double* y[4];
  int64_t ldy;
  double* yp;
  double* w[4];
  int64_t ldw;
  double* wp;
  double alpha, beta;  // C = alpha * product + beta * C (sketch: 1, 1); partials are plain
};

// Epilogue: the half-0 warps gather the other half's products (qtile8.cuh),
// form the quaternion planes and add them to C (or write the split-K partial).
template <int MODE>
__device__ __forceinline__ void store_slot8(const qt8::Acc& acc, const double* slot, int64_t i0, int64_t j0, int64_t M,
                                            int64_t N, double* const* c, int64_t ldc, double* part, double alpha,
                                            double beta) {
  if (!slot) return;
#pragma unroll
  for (int rb = 0; rb < 2; ++rb) {
    const int64_t gi = i0 + qt8::acc_row<MODE>(rb);
    if (gi >= M) continue;
#pragma unroll
    for (int cb = 0; cb < 2; ++cb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gj = j0 + qt8::acc_col<MODE>(cb) + h;
        if (gj >= N) continue;
        double m[8], q[4];
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
          m[ii] = acc[ii][rb][cb][h];
          m[4 + ii] = qt8::other_product(slot, ii, rb, cb, h);
          if constexpr (qt8::Cfg<MODE>::GRAM) m[4 + ii] *= 0.5;  // no combined side to carry the halves
        }
        qt8::combine(m, q);
        if (part) {
#pragma unroll
          for (int p = 0; p < 4; ++p) part[(int64_t)p * M * N + gi * N + gj] = q[p];
        } else {
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            double* dst = c[p] + gi * ldc + gj;
            *dst = beta == 1.0 && alpha == 1.0 ? *dst + q[p] : (beta != 0.0 ? fma(beta, *dst, alpha * q[p]) : alpha * q[p]);
          }
        }
      }
  }
}

template <int MODE>
__device__ __forceinline__ void store_tile8(const qt8::Acc& acc, double* xbuf, int64_t i0, int64_t j0, int64_t M,
                                            int64_t N, double* const* c, int64_t ldc, double* part, double alpha,
                                            double beta) {
  store_slot8<MODE>(acc, qt8::exchange_products(acc, xbuf), i0, j0, M, N, c, ldc, part, alpha, beta);
}

// One task of mode MODE (qtile8.cuh) at tile origin (i0, j0), split z.
template <int MODE, bool TMA>
__device__ __forceinline__ void run_task(const Fused8Args& f, double* smem, int64_t i0, int64_t j0, int z) {
  constexpr bool W = (MODE & 1) != 0;
  const qt8::Operands& op = W ? f.wop : f.yop;
  const int64_t kc = W ? f.kw_chunk : f.ky_chunk, K = W ? f.kw : f.ky;
  const int zs = W ? f.zw : f.zy;
  const int64_t kb = (int64_t)z * kc, ke = min(K, kb + kc);
  qt8::Acc acc;
  qt8::zero_acc(acc);
  if constexpr (TMA) {
    const CUtensorMap* lm = MODE == 0 ? &f.ylm : MODE == 1 ? &f.wlm : MODE == 2 ? &f.ynlm : &f.wnlm;
    const CUtensorMap* rm = MODE == 0 ? &f.yrm : MODE == 1 ? &f.wrm : MODE == 2 ? &f.ynrm : &f.wnrm;
    qt8::mma_tile_tma<MODE>(qt8::TmaOps{lm, rm, 0, f.stages, f.stride}, op, smem, i0, j0, kb, ke, acc);
  } else if constexpr (MODE < 2) {
    qt8::mma_tile<MODE>(op, smem, i0, j0, kb, ke, acc);
  }
  double* part = zs > 1 ? (W ? f.wp : f.yp) + (int64_t)z * 4 * op.M * op.N : nullptr;
  store_tile8<MODE>(acc, smem, i0, j0, op.M, op.N, W ? f.w : f.y, W ? f.ldw : f.ldy, part, f.alpha, f.beta);
}

// Y tiles g0 .. g0 + ntiles - 1 (row tiles of mode MODE) at column j0 as one
// TMA stage stream (stream_tiles); Y-only launches with small K and zy = 1.
template <int MODE>
__device__ __forceinline__ void run_stream(const Fused8Args& f, double* smem, int g0, int ntiles, int64_t j0) {
  constexpr int TM = qt8::Cfg<MODE>::TM;
  const CUtensorMap* lm = MODE == 0 ? &f.ylm : &f.ynlm;
  const CUtensorMap* rm = MODE == 0 ? &f.yrm : &f.ynrm;
  double* xbuf = smem + (size_t)f.stages * f.stride;
  qt8::stream_tiles<MODE>(qt8::TmaOps{lm, rm, 0, f.stages, f.stride}, f.yop, smem, xbuf, (int64_t)g0 * TM, ntiles, j0,
                          0, f.ky, [&](const qt8::Acc& acc, const double* slot, int64_t i0) {
                            store_slot8<MODE>(acc, slot, i0, j0, f.yop.M, f.yop.N, f.y, f.ldy, nullptr, f.alpha,
                                              f.beta);
                          });
}

// Task order, longest first: full W tiles, narrow W remainder tiles, Y
// tiles, narrow Y remainder tiles, padded W row tiles.  Within the groups
// the order is L2-aware: W CTAs sharing a K chunk are adjacent (the l-row
// tiles of an A column tile read the same A rows, the n-column tiles of a
// Psi~ row tile the same Psi~ columns), and the column tiles of a Y row tile
// are adjacent, so each A row tile comes from DRAM about once.
template <bool TMA>
__global__ void __launch_bounds__(TMA ? qt8::NT_TMA : qt8::NT, 1) sketch8_kernel(const __grid_constant__ Fused8Args f) {
  extern __shared__ __align__(128) double smem_raw[];
  // TMA destinations need 128-byte alignment (the launch adds the slack)
  // (offset arithmetic on the shared array keeps the accesses LDS, not generic)
  double* smem = smem_raw + ((128u - (qt::smem_u32(smem_raw) & 127u)) & 127u) / sizeof(double);
  const int wtf = f.w_tmf * f.w_tn, wtp = (f.w_tm - f.w_tmf) * f.w_tn;
  const int nwf = wtf * f.zw, nwn = f.wn_t * f.zw;
  const int yg = (f.y_tm + f.y_rep - 1) / f.y_rep, yng = (f.yn_t + f.y_rep - 1) / f.y_rep;
  const int nyr = yg * f.y_tn * f.zy, nyn = yng * f.zy;
  int t = blockIdx.x;
  if (t < nwf) {
    const int tile = t % wtf, z = t / wtf;
    run_task<1, TMA>(f, smem, (int64_t)(tile % f.w_tmf) * W8M, (int64_t)(tile / f.w_tmf) * W8N, z);
    return;
  }
  t -= nwf;
  if (TMA && t < nwn) {
    const int tile = t % f.wn_t, z = t / f.wn_t;
    run_task<3, TMA>(f, smem, (int64_t)f.w_tmf * W8M, (int64_t)tile * WNN, z);
    return;
  }
  t -= nwn;
  if (TMA && f.y_rep == 1 && f.yn_t > 0 && f.y_ilv && t < nyr + nyn) {
    // interleaved: each 128-row block's regular Y tiles, then its narrow
    // tile, so the block's A rows are re-read from L2 rather than DRAM
    const int per = (2 * f.y_tn + 1) * f.zy;  // tasks of a full block
    int blk = t / per, r = t % per;
    if (blk >= f.yn_t - 1) {  // the last block may hold one regular row tile
      blk = f.yn_t - 1;
      r = t - blk * per;
    }
    const int nreg = min(2, f.y_tm - 2 * blk) * f.y_tn * f.zy;
    if (r < nreg) {
      const int z = r % f.zy, q = r / f.zy;
      run_task<0, TMA>(f, smem, (int64_t)(2 * blk + q / f.y_tn) * Y8M, (int64_t)(q % f.y_tn) * Y8N, z);
    } else {
      run_task<2, TMA>(f, smem, (int64_t)blk * YNM, (int64_t)f.y_tnf * Y8N, r - nreg);
    }
    return;
  }
  if (t < nyr) {
    const int z = t % f.zy;
    t /= f.zy;
    const int tn = t % f.y_tn, g0 = (t / f.y_tn) * f.y_rep;
    if constexpr (TMA) {
      if (f.y_rep > 1) {
        run_stream<0>(f, smem, g0, min(f.y_rep, f.y_tm - g0), (int64_t)tn * Y8N);
        return;
      }
    }
    run_task<0, TMA>(f, smem, (int64_t)g0 * Y8M, (int64_t)tn * Y8N, z);
    return;
  }
  t -= nyr;
  if (TMA && t < nyn) {
    const int z = t % f.zy, g0 = (t / f.zy) * f.y_rep;
    if constexpr (TMA) {
      if (f.y_rep > 1) {
        run_stream<2>(f, smem, g0, min(f.y_rep, f.yn_t - g0), (int64_t)f.y_tnf * Y8N);
        return;
      }
    }
    run_task<2, TMA>(f, smem, (int64_t)g0 * YNM, (int64_t)f.y_tnf * Y8N, z);
    return;
  }
  t -= nyn;
  const int tile = t % wtp, z = t / wtp;
  run_task<1, TMA>(f, smem, (int64_t)(f.w_tmf + tile % (f.w_tm - f.w_tmf)) * W8M,
                   (int64_t)(tile / (f.w_tm - f.w_tmf)) * W8N, z);
}

// ---- Gram Y^* Y on the 8-product engine (mode 4) ---------------------------
constexpr int GRAM_MAXT = 160;  // upper tiles of an s x s Gram, s <= 512
struct Gram8Args {
  CUtensorMap lm, rm;  // both over Y: boxes {68, BK, 4} (adjoint side) / {36, BK, 4}
  int stages, stride;
  qt8::Operands op;    // M = N = s (bounds only; the data comes through the maps)
  int64_t K, kchunk;
  int ntiles, zk;
  unsigned short tm[GRAM_MAXT], tn[GRAM_MAXT];
  double* g[4];
  int64_t ldg;
  double* part;        // [zk][4][s][s] when zk > 1
};

template <int MODE>
__global__ void __launch_bounds__(qt8::NT_TMA, 1) gram8_kernel(const __grid_constant__ Gram8Args f) {
  extern __shared__ __align__(128) double smem_raw[];
  double* smem = smem_raw + ((128u - (qt::smem_u32(smem_raw) & 127u)) & 127u) / sizeof(double);
  const int tile = blockIdx.x % f.ntiles, z = blockIdx.x / f.ntiles;
  const int64_t i0 = (int64_t)f.tm[tile] * qt8::Cfg<MODE>::TM, j0 = (int64_t)f.tn[tile] * qt8::Cfg<MODE>::TN;
  const int64_t kb = (int64_t)z * f.kchunk, ke = min(f.K, kb + f.kchunk);
  qt8::Acc acc;
  qt8::zero_acc(acc);
  qt8::mma_tile_tma<MODE>(qt8::TmaOps{&f.lm, &f.rm, 0, f.stages, f.stride}, f.op, smem, i0, j0, kb, ke, acc);
  const int64_t s = f.op.M;
  double* part = f.zk > 1 ? f.part + (int64_t)z * 4 * s * s : nullptr;
  store_tile8<MODE>(acc, smem, i0, j0, s, s, f.g, f.ldg, part, 1.0, 0.0);
}

// out plane i (rows x cols, ld = cols) = combination i of in's planes, the
// left (Psi) or right (Omega) set, halves folded into i >= 4
__global__ void combine8_kernel(QView in, double* out, int64_t ld, int left, int adj) {
  // adj: combine op(in) = in^* (rows x cols of the adjoint)
  const int64_t rows = adj ? in.cols : in.rows, cols = adj ? in.rows : in.cols, total = rows * cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / cols, j = e % cols;
    double v[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const double x = adj ? in.p[p][j * in.ld + i] : in.p[p][i * in.ld + j];
      v[p] = adj && p > 0 ? -x : x;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double x = left ? qt8::lcomb(c, v) : qt8::rcomb(c, v);
      out[(int64_t)c * rows * ld + i * ld + j] = c >= 4 ? 0.5 * x : x;
    }
  }
}

}  // namespace

bool sketch_use8() { return true; }

const char* sketch_kernel_name() {
  return "sketch8_kernel(8-product quaternion GEMM on DMMA, 64x32/32x64 tiles, TMA + mbarrier ring, panels <= 2 GB)";
}

namespace {

struct SketchWork {
  DeviceBuffer yp, wp;  // split-K partial workspaces, grown on demand
};

// Tile geometry of a fused launch: Y tiles ym x yn, W tiles wm x wn, each
// made of 8x8 blocks (padded blocks cost nothing).
struct Geom {
  int ym, yn, wm, wn;
  bool ynarrow = false, wnarrow = false;  // remainder as 128x16 / 16x128 tiles (8-product TMA path)
};
constexpr Geom kGeom8{Y8M, Y8N, W8M, W8N};
// the narrow remainder tiles pay off when they hold at most half a regular
// tile's columns (Y) / rows (W)
inline bool narrow_rem(int64_t ext, int tile) { return ext % tile != 0 && ext % tile <= tile / 2; }

// Makespan of one fused launch under greedy list scheduling on 148 SMs
// (1 CTA per SM), tasks in kernel order.  Cost unit: one BK k-step of a full
// tile (both engines' Y and W tiles cost the same per k-step).
double simulate_panel(const Geom& G, int64_t rp, int64_t n, int64_t s, int64_t l, int zy, int zw) {
  const int64_t kyc = ((n + zy - 1) / zy + BK - 1) / BK * BK, kwc = ((rp + zw - 1) / zw + BK - 1) / BK * BK;
  const int64_t ny_chunks = (n + kyc - 1) / kyc, nw_chunks = (rp + kwc - 1) / kwc;
  const int64_t y_tm = (rp + G.ym - 1) / G.ym, y_tn = (s + G.yn - 1) / G.yn, w_tm = (l + G.wm - 1) / G.wm,
                w_tn = (n + G.wn - 1) / G.wn;
  const int64_t y_tnf = s / G.yn, w_tmf = l / G.wm;
  auto frac = [](int64_t valid, int dim) { return (double)((valid + 7) / 8) / (dim / 8); };
  const double y_part = frac(s - y_tnf * G.yn, G.yn), w_part = frac(l - w_tmf * G.wm, G.wm);
  // narrow remainder tiles: valid 8x8 blocks over a regular tile's 32
  const int64_t yn_t = G.ynarrow ? (rp + YNM - 1) / YNM : 0, wn_t = G.wnarrow ? (n + WNN - 1) / WNN : 0;
  const double yn_cost = (double)((s - y_tnf * G.yn + 7) / 8) * (YNM / 8) / 32.0;
  const double wn_cost = (double)((l - w_tmf * G.wm + 7) / 8) * (WNN / 8) / 32.0;
  struct Group { int64_t count; double cost; };
  const Group groups[6] = {{w_tmf * w_tn * nw_chunks, (double)(kwc / BK)},
                           {wn_t * nw_chunks, (double)(kwc / BK) * wn_cost},
                           {y_tm * y_tnf * ny_chunks, (double)(kyc / BK)},
                           {G.ynarrow ? 0 : y_tm * (y_tn - y_tnf) * ny_chunks, (double)(kyc / BK) * y_part},
                           {yn_t * ny_chunks, (double)(kyc / BK) * yn_cost},
                           {G.wnarrow ? 0 : (w_tm - w_tmf) * w_tn * nw_chunks, (double)(kwc / BK) * w_part}};
  // Greedy assignment on buckets of SMs that free at the same time (tasks of
  // a group cost the same, so whole buckets advance together): O(tasks/148)
  // per group instead of a heap operation per CTA.
  std::map<double, int64_t> sm{{0.0, 148}};
  for (const Group& g : groups) {
    const double d = g.cost + 2.0;  // + prologue/epilogue (~2 k-steps)
    int64_t c = g.count;
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
  const double mk = sm.rbegin()->first;
  // split-K partials cost a reduction pass over zy Y / zw W copies
  // (~1 k-step of a 64x64 tile per 25 MB of partials; scaled by tile area)
  const double red = (zy > 1 ? (double)zy * rp * s : 0.0) + (zw > 1 ? (double)zw * l * n : 0.0);
  return mk + red * 32.0 / 25e6 * (double)(BM * BN) / (double)(G.ym * G.yn);
}

std::pair<int, int> choose_panel_splits(const Geom& G, int64_t rp, int64_t n, int64_t s, int64_t l) {
  static std::mutex mu;
  static std::map<std::array<int64_t, 5>, std::pair<int, int>> cache;
  const std::array<int64_t, 5> key{rp, n, s, l, (int64_t)G.ym * 1000 + G.yn + (G.ynarrow ? 1000000 : 0) +
                                                  (G.wnarrow ? 2000000 : 0)};
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  const int64_t wt = ((l + G.wm - 1) / G.wm) * ((n + G.wn - 1) / G.wn);
  // W split-K only while W has fewer than 4 waves of tiles (its partials are
  // l x n each: 868 MB at C4)
  const int zw_max = wt >= 4 * 148 ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(wt >= 148 ? 8 : 64, rp / 64));
  const int zy_max = (int)std::max<int64_t>(1, std::min<int64_t>(256, n / 32));
  // candidates: every value up to 16, then geometric steps of ~12%
  auto candidates = [](int hi) {
    std::vector<int> v;
    for (int z = 1; z <= hi; z = z < 16 ? z + 1 : std::max(z + 1, z * 9 / 8)) v.push_back(z);
    if (v.back() != hi) v.push_back(hi);
    return v;
  };
  double best = 1e300;
  std::pair<int, int> arg{1, 1};
  for (int zw : candidates(zw_max))
    for (int zy : candidates(zy_max)) {
      const double mk = simulate_panel(G, rp, n, s, l, zy, zw);
      if (mk < best - 1e-9) { best = mk; arg = {zy, zw}; }
    }
  {
    std::lock_guard<std::mutex> lock(mu);
    cache[key] = arg;
  }
  if (std::getenv("QLRA_DEBUG_SPLITS")) {
    // ideal = total cost / 148 (perfect balance, no per-CTA overhead)
    const int64_t y_tm = (rp + G.ym - 1) / G.ym, y_tn = (s + G.yn - 1) / G.yn, w_tm = (l + G.wm - 1) / G.wm,
                  w_tn = (n + G.wn - 1) / G.wn;
    auto frac = [](int64_t valid, int dim) { return (double)((valid + 7) / 8) / (dim / 8); };
    const double yc = (double)y_tm * ((double)(s / G.yn) + (y_tn > s / G.yn ? frac(s - (s / G.yn) * G.yn, G.yn) : 0.0)) * (double)n / BK;
    const double wc = (double)w_tn * ((double)(l / G.wm) + (w_tm > l / G.wm ? frac(l - (l / G.wm) * G.wm, G.wm) : 0.0)) * (double)rp / BK;
    std::fprintf(stderr, "[qlra] panel %lldx%lld s=%lld l=%lld tiles %dx%d/%dx%d: zy=%d zw=%d makespan %.0f ideal %.0f (%.1f%%)\n",
                 (long long)rp, (long long)n, (long long)s, (long long)l, G.ym, G.yn, G.wm, G.wn, arg.first, arg.second,
                 best, (yc + wc) / 148.0, 100.0 * (yc + wc) / 148.0 / best);
  }
  return arg;
}

// The embeddings of one sketch call: Omega (n x s) and the Psi column block
// (l x b), plain (16-product engine) or as their 8 plane combinations
// (8-product engine; planes of rows x cols each, ld = cols).
struct Emb {
  QView om, ps;
  const double* om8 = nullptr;  // 8 planes of n x s, leading dimension om8_ld
  const double* ps8 = nullptr;  // 8 planes of l x b, leading dimension ps8_ld
  int64_t om8_ld = 0, ps8_ld = 0;  // even: 16-byte rows for TMA
};

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda
// link).  3D map over planes of row-major doubles: (inner, rows, planes).
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}
bool make_map3(CUtensorMap* m, const double* base, int64_t inner, int64_t rows, int64_t planes, int64_t ld,
               int64_t pstride, int box_inner, int box_rows, int box_planes) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)planes};
  const cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)pstride * 8};
  const cuuint32_t box[3] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows, (cuuint32_t)box_planes};
  const cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// A's planes as one 3D tensor: 16-byte aligned rows and a uniform positive
// plane stride (a (4, m, n) tensor with n even); else the cp.async path
bool tma_layout(const QView& a, int64_t* pstride) {
  const int64_t d = a.p[1] - a.p[0];
  if (d <= 0 || d % 2 || a.ld % 2 || (reinterpret_cast<uintptr_t>(a.p[0]) & 15)) return false;
  for (int q = 2; q < 4; ++q)
    if (a.p[q] - a.p[0] != q * d) return false;
  *pstride = d;
  return true;
}
// TMA ring slots (QLRA_Q8_STAGES overrides; the producer warp refills a slot as soon as it is released)
// dynamic shared memory of the TMA kernel: 227 KB less its static barriers
constexpr size_t kDynSmemMax = 227 * 1024 - 1024;
int tma_stages(int stride, size_t extra_bytes) {
  static const int req = [] {
    const char* e = std::getenv("QLRA_Q8_STAGES");
    return e ? std::atoi(e) : 4;
  }();
  return std::max(2, std::min(req, std::min(qt8::MAX_STAGES, (int)((kDynSmemMax - 128 - extra_bytes) / (stride * sizeof(double))))));
}
bool sketch_tma_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("QLRA_SKETCH_TMA");
    return !(e && std::atoi(e) == 0);
  }();
  return v;
}

template <class Args>
void set_splits(Args& f, const Geom& G, int64_t rp, int64_t n, int64_t s, int64_t l, Ctx& ctx, SketchWork& ws) {
  f.y_tm = (int)((rp + G.ym - 1) / G.ym);
  f.y_tn = (int)((s + G.yn - 1) / G.yn);
  f.w_tm = (int)((l + G.wm - 1) / G.wm);
  f.w_tn = (int)((n + G.wn - 1) / G.wn);
  f.y_tnf = (int)(s / G.yn);
  f.w_tmf = (int)(l / G.wm);
  if constexpr (std::is_same_v<Args, Fused8Args>) {  // narrow remainder tiles: 8-product engine only
    if (G.ynarrow) {
      f.y_tn = f.y_tnf;
      f.yn_t = (int)((rp + YNM - 1) / YNM);
    }
    if (G.wnarrow) {
      f.w_tm = f.w_tmf;
      f.wn_t = (int)((n + WNN - 1) / WNN);
    }
  }
  // Split counts (zy over n, zw over the panel rows) from a simulation of
  // the dispatcher: CTAs in kernel order (longest first) go to the SM that
  // frees first; cost = k-steps x fraction of 8x8 blocks inside M x N.
  // Cached per panel shape.
  const auto choice = choose_panel_splits(G, rp, n, s, l);
  f.kw_chunk = ((rp + choice.second - 1) / choice.second + BK - 1) / BK * BK;
  f.zw = (int)((rp + f.kw_chunk - 1) / f.kw_chunk);
  f.ky_chunk = ((n + choice.first - 1) / choice.first + BK - 1) / BK * BK;
  f.zy = (int)((n + f.ky_chunk - 1) / f.ky_chunk);
  if (f.zy > 1) {
    const size_t need = (size_t)f.zy * 4 * rp * s * sizeof(double);
    if (ws.yp.bytes < need) ws.yp = DeviceBuffer(ctx, need);
    f.yp = ws.yp.as<double>();
  }
  if (f.zw > 1) {
    const size_t need = (size_t)f.zw * 4 * l * n * sizeof(double);
    if (ws.wp.bytes < need) ws.wp = DeviceBuffer(ctx, need);
    f.wp = ws.wp.as<double>();
  }
}

// One launch of the 8-product engine (+ ordered split-K reductions).
//   Y part: C (M x N) = alpha * A (M x K) * B~ (K x N) + beta * C,
//           A on the fly (4 planes), B~ the 8 combined right planes of B;
//   W part: C (M x N) = alpha * P~ (M x K) * A (K x N) + beta * C,
//           P~ the 8 combined left planes of P (from column col0), A on the fly.
// Either part may be absent.  The sketch launches both (the same A block as
// the Y part's left and the W part's right operand), the 8-product qgemm one.
struct Q8Part {
  QView a;                  // the on-the-fly operand
  const double* comb;       // combined planes (8 x rows x comb_ld)
  int64_t comb_ld, col0;    // leading dimension (even), first column used (even)
  QView c;                  // output
};
void launch8(Ctx& ctx, const Q8Part* y, const Q8Part* w, double alpha, double beta, SketchWork& ws, bool timed) {
  Fused8Args f{};
  f.alpha = alpha;
  f.beta = beta;
  // split simulation extents: rp = Y's M and W's K, n = Y's K and W's N
  const int64_t rp = y ? y->a.rows : w->a.rows, n = y ? y->a.cols : w->a.cols;
  const int64_t s = y ? y->c.cols : 0, l = w ? w->c.rows : 0;
  if (y && w && (w->a.rows != rp || w->a.cols != n)) fail(QLRA_ERR_SHAPE, "launch8: coupled parts differ");
  // (an absent part launches no task, so its operand pointers are never read)
  for (int p = 0; p < 4; ++p) {
    f.yop.l[p] = y ? y->a.p[p] : nullptr;
    f.wop.r[p] = w ? w->a.p[p] : nullptr;
    f.y[p] = y ? y->c.p[p] : nullptr;
    f.w[p] = w ? w->c.p[p] : nullptr;
  }
  for (int i = 0; i < 8; ++i) {
    f.yop.r[i] = y ? y->comb + (size_t)i * n * y->comb_ld : nullptr;
    f.wop.l[i] = w ? w->comb + (size_t)i * l * w->comb_ld + w->col0 : nullptr;
  }
  if (y) {
    f.yop.l_si = y->a.ld; f.yop.r_sk = y->comb_ld;
    f.yop.M = rp; f.yop.N = s;
    f.ldy = y->c.ld;
  }
  if (w) {
    f.wop.l_si = w->comb_ld; f.wop.r_sk = w->a.ld;
    f.wop.M = l; f.wop.N = n;
    f.ldw = w->c.ld;
  }
  f.ky = n;
  f.kw = rp;
  // TMA staging when each on-the-fly operand's planes form one
  // 16-byte-aligned 3D tensor; the maps cover exactly the operands (rows past
  // them, k past K and columns past N come back zero)
  int64_t yps = 0, wps = 0;
  bool tma = sketch_tma_enabled();
  if (tma && y)
    tma = tma_layout(y->a, &yps) && make_map3(&f.ylm, y->a.p[0], n, rp, 4, y->a.ld, yps, qt8::LDK, Y8M, 4) &&
          make_map3(&f.yrm, y->comb, s, n, 8, y->comb_ld, n * y->comb_ld, qt8::Layout<0>::LDX, qt8::BK, 8) &&
          make_map3(&f.ynlm, y->a.p[0], n, rp, 4, y->a.ld, yps, qt8::LDK, YNM, 4) &&
          make_map3(&f.ynrm, y->comb, s, n, 8, y->comb_ld, n * y->comb_ld, qt8::Layout<2>::LDX, qt8::BK, 8);
  if (tma && w)
    tma = tma_layout(w->a, &wps) && (w->col0 % 2) == 0 &&
          make_map3(&f.wlm, w->comb + w->col0, rp, l, 8, w->comb_ld, l * w->comb_ld, qt8::LDK, W8M, 8) &&
          make_map3(&f.wrm, w->a.p[0], n, rp, 4, w->a.ld, wps, qt8::Layout<1>::LDX, qt8::BK, 4) &&
          make_map3(&f.wnlm, w->comb + w->col0, rp, l, 8, w->comb_ld, l * w->comb_ld, qt8::LDK, WNM, 8) &&
          make_map3(&f.wnrm, w->a.p[0], n, rp, 4, w->a.ld, wps, qt8::Layout<3>::LDX, qt8::BK, 4);
  Geom G = kGeom8;
  G.ynarrow = tma && y && narrow_rem(s, Y8N);
  G.wnarrow = tma && w && narrow_rem(l, W8M);
  set_splits(f, G, rp, n, s, l, ctx, ws);
  if (!y) f.y_tm = f.y_tn = f.y_tnf = f.yn_t = 0;
  if (!w) f.w_tm = f.w_tn = f.w_tmf = f.wn_t = 0;
  // Y-only launches with few k-steps (Y R^-1, H = base M: K = s): stream
  // several row tiles per CTA so the TMA pipeline does not drain per tile,
  // keeping >= 2 waves of CTAs
  f.y_rep = 1;
  if (tma && y && !w && f.zy == 1) {
    const int64_t nk = (n + qt8::BK - 1) / qt8::BK;
    const int64_t tiles = (int64_t)f.y_tm * f.y_tn + f.yn_t;
    if (nk <= 32) f.y_rep = (int)std::max<int64_t>(1, std::min<int64_t>({(64 + nk - 1) / nk, 32, tiles / 296}));
  }
  const int64_t ctas = (int64_t)((f.y_tm + f.y_rep - 1) / f.y_rep) * f.y_tn * f.zy +
                       (int64_t)((f.yn_t + f.y_rep - 1) / f.y_rep) * f.zy + (int64_t)f.w_tm * f.w_tn * f.zw +
                       (int64_t)f.wn_t * f.zw;
  if (ctas == 0) return;
  // ring slots sized for the modes present: the narrow tiles need 7424
  // doubles per slot (3 slots), the regular ones 5376 (4 slots)
  static const int ilv = [] {
    const char* e = std::getenv("QLRA_Y_INTERLEAVE");  // (C5 sketch -1%, C2 DRAM reads -5%)
    return e ? std::atoi(e) : 1;
  }();
  f.y_ilv = ilv;
  f.stride = (f.yn_t || f.wn_t) ? qt8::STAGE_TMA : qt8::STAGE;
  // (streamed launches keep a separate 64 KB exchange buffer after the ring)
  const size_t xbytes = f.y_rep > 1 ? (size_t)8 * 32 * 32 * sizeof(double) : 0;
  f.stages = tma_stages(f.stride, xbytes);
  LaunchTimer lt(ctx, timed);
  if (tma)
    sketch8_kernel<true><<<(unsigned)ctas, qt8::NT_TMA, (size_t)f.stages * f.stride * sizeof(double) + xbytes + 128,
                           ctx.stream>>>(f);
  else
    sketch8_kernel<false><<<(unsigned)ctas, qt8::NT, qt8::SMEM_BYTES + 128, ctx.stream>>>(f);
  QLRA_LAUNCH_CHECK();
  count_launch();
  lt.done(rp, n, s, l);
  if (y && f.zy > 1) splitk_reduce(ctx, f.yp, f.zy, y->c, alpha, beta);
  if (w && f.zw > 1) splitk_reduce(ctx, f.wp, f.zw, w->c, alpha, beta);
}

// One fused launch (+ ordered partial reductions) for a row panel `ap` of A
// whose Psi columns are ps[:, pc0 : pc0 + ap.rows].
void sketch_panel(Ctx& ctx, const Emb& e, int64_t pc0, const QView& ap, const QView& yv, const QView& w,
                  SketchWork& ws) {
  const Q8Part yp{ap, e.om8, e.om8_ld, 0, yv};
  const Q8Part wq{ap, e.ps8, e.ps8_ld, pc0, w};
  launch8(ctx, &yp, &wq, 1.0, 1.0, ws, true);
}

// Plane combinations of an embedding for the 8-product engine.
void launch_combine8(Ctx& ctx, const QView& in, double* out, int64_t ld, bool left, bool adj = false) {
  const int64_t total = in.rows * in.cols;
  if (total == 0) return;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((total + threads - 1) / threads, 148 * 16);
  combine8_kernel<<<(unsigned)blocks, threads, 0, ctx.stream>>>(in, out, ld, left ? 1 : 0, adj ? 1 : 0);
  QLRA_LAUNCH_CHECK();
  count_launch();
}

// Fill e.om8 / e.ps8 (when the 8-product engine is on) into the context's
// kept combination buffer.
void prepare_emb(Ctx& ctx, Emb& e, const qlra_spec_t& psi, int64_t row0) {
  ctx.comb_keep.psi_valid = false;
  e.om8_ld = (e.om.cols + 1) / 2 * 2;
  e.ps8_ld = (e.ps.cols + 1) / 2 * 2;
  const size_t no = (size_t)8 * e.om.rows * e.om8_ld, np = (size_t)8 * e.ps.rows * e.ps8_ld;
  const size_t bytes = (no + np) * sizeof(double);
  Ctx::CombKeep& k = ctx.comb_keep;
  if (k.bytes < bytes) {
    if (k.buf) QLRA_CUDA(cudaFreeAsync(k.buf, ctx.stream));
    k.buf = nullptr;
    k.bytes = 0;
    QLRA_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&k.buf), bytes, ctx.stream));
    k.bytes = bytes;
  }
  double* base = k.buf;
  launch_combine8(ctx, e.om, base, e.om8_ld, false);
  launch_combine8(ctx, e.ps, base + no, e.ps8_ld, true);
  e.om8 = base;
  e.ps8 = base + no;
  k.psi_valid = true;
  k.psi = psi;
  k.row0 = row0;
  k.rows = e.ps.cols;
  k.ps8 = e.ps8;
  k.ps8_ld = e.ps8_ld;
}

void set_kernel_attrs() {
  set_func_attr((const void*)sketch8_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                (int)qt8::SMEM_BYTES + 128);
  set_func_attr((const void*)gram8_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDynSmemMax);
  set_func_attr((const void*)gram8_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDynSmemMax);
  set_func_attr((const void*)sketch8_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                (int)kDynSmemMax);
}

// Rows per fused launch.  Device-resident A: panels of up to kPanelBytes --
// the kernel does ~300 flop per byte of A, so an A tile re-read from HBM
// instead of L2 costs nothing measurable, while one long launch balances the
// CTAs over the SMs far better than many short ones (C2: 16.3 ms as one
// launch vs 19.9 ms as 32 L2-sized panels).  Host-streamed A: chunks of
// kStreamBytes so the H2D copy of the next chunk overlaps the sketch of this
// one (about 16 chunks per block, at least kStreamBytes each).  Multiples of
// 64 rows, at least 256.  QLRA_PANEL_BYTES / QLRA_STREAM_BYTES override
// (tuning).
constexpr double kPanelBytes = 2e9;
constexpr double kStreamBytes = 64e6;
double env_or(const char* name, double dflt) {
  const char* e = std::getenv(name);
  return e ? std::atof(e) : dflt;
}
int64_t rows_for(double bytes, int64_t n, int64_t b) {
  int64_t R = (int64_t)(bytes / (32.0 * (double)n));
  R = std::max<int64_t>(256, (R / 64) * 64);
  return std::min<int64_t>(R, ((b + 63) / 64) * 64);
}
int64_t panel_rows(int64_t n, int64_t b) {
  static const double bytes = env_or("QLRA_PANEL_BYTES", kPanelBytes);
  return rows_for(bytes, n, b);
}
int64_t stream_rows(int64_t n, int64_t b) {
  // ~16 chunks per block (each DMA call and chunk boundary costs; measured
  // C2: 16 x 96 MB 28.6 ms vs 32 x 48 MB 29.0 ms, plain copy 27.6 ms), never
  // below kStreamBytes: small chunks of a narrow A (C5: n = 300) make short,
  // inefficient launches
  static const double floor_bytes = env_or("QLRA_STREAM_BYTES", kStreamBytes);
  const double bytes = std::max(floor_bytes, 32.0 * (double)n * (double)b / 16.0);
  return rows_for(bytes, n, b);
}

}  // namespace

namespace {
QView view_of_buf(double* base, int64_t rows, int64_t cols) {
  QView v{};
  for (int p = 0; p < 4; ++p) v.p[p] = base + (size_t)p * rows * cols;
  v.rows = rows;
  v.cols = cols;
  v.ld = cols;
  return v;
}
bool same_spec(const qlra_spec_t& a, const qlra_spec_t& b) {
  return a.kind == b.kind && a.rows == b.rows && a.cols == b.cols && a.seed == b.seed && a.density == b.density;
}
}  // namespace

// C = alpha * A B + beta * C on the 8-product engine when one factor is much
// smaller than the other (the tall products of the rangefinders and the core
// solve: Y R^-1, Q0 C, Psi Q0, ...): the small factor is combined into its 8
// planes (one pass over it), the large one streams through the kernel as
// the sketch's A does.  Returns false (nothing launched) when the shapes do
// not fit that pattern; the caller then runs the 16-product qgemm.
bool q8gemm_try(Ctx& ctx, int op_a, int op_b, double alpha, const QView& A, const QView& B, double beta,
                const QView& C) {
  static const bool enabled = [] {
    const char* e = std::getenv("QLRA_Q8GEMM");
    return !(e && std::atoi(e) == 0);
  }();
  if (!enabled || !sketch_use8()) return false;
  const bool ca = op_a == QLRA_OP_C, cb = op_b == QLRA_OP_C;
  if (ca && cb) return false;
  const int64_t M = ca ? A.cols : A.rows, K = ca ? A.rows : A.cols;
  const int64_t Kb = cb ? B.cols : B.rows, N = cb ? B.rows : B.cols;
  if (Kb != K || C.rows != M || C.cols != N || M == 0 || N == 0 || K == 0) return false;
  const double a_el = (double)M * (double)K, b_el = (double)K * (double)N;
  // the combined (small) factor may be an adjoint -- it is materialised by
  // the combine pass; the streamed (large) factor must be plain
  const bool right = !ca && b_el * 4.0 <= a_el, left = !right && !cb && a_el * 4.0 <= b_el;
  if (!right && !left) return false;
  set_kernel_attrs();
  const QView& small = right ? B : A;
  const bool adj = right ? cb : ca;
  const int64_t srows = adj ? small.cols : small.rows, scols = adj ? small.rows : small.cols;
  const int64_t ld = (scols + 1) / 2 * 2;
  DeviceBuffer comb(ctx, (size_t)8 * srows * ld * sizeof(double));
  launch_combine8(ctx, small, comb.as<double>(), ld, left, adj);
  SketchWork ws;
  if (right) {
    const Q8Part y{A, comb.as<double>(), ld, 0, C};
    launch8(ctx, &y, nullptr, alpha, beta, ws, false);
  } else {
    const Q8Part w{B, comb.as<double>(), ld, 0, C};
    launch8(ctx, nullptr, &w, alpha, beta, ws, false);
  }
  return true;
}


QView psi_for_sketch(Ctx& ctx, const qlra_spec_t& psi, int64_t row0, int64_t rows, DevQMat& tmp) {
  static const double cap = env_or("QLRA_PSI_KEEP_BYTES", 8e9);
  const int64_t l = psi.rows;
  const size_t bytes = (size_t)4 * l * rows * sizeof(double);
  Ctx::PsiKeep& k = ctx.psi_keep;
  k.valid = false;
  if ((double)bytes > cap || bytes == 0) {
    tmp = DevQMat(ctx, l, rows);
    launch_gen(ctx.stream, psi, 0, row0, l, rows, tmp.v, false);
    return tmp.v;
  }
  if (k.bytes < bytes) {
    if (k.buf) QLRA_CUDA(cudaFreeAsync(k.buf, ctx.stream));
    k.buf = nullptr;
    k.bytes = 0;
    QLRA_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&k.buf), bytes, ctx.stream));
    k.bytes = bytes;
  }
  const QView v = view_of_buf(k.buf, l, rows);
  launch_gen(ctx.stream, psi, 0, row0, l, rows, v, false);
  k.valid = true;
  k.spec = psi;
  k.row0 = row0;
  k.rows = rows;
  return v;
}

QView psi_for_solve(Ctx& ctx, const qlra_spec_t& psi, int64_t row0, int64_t rows, DevQMat& tmp) {
  const Ctx::PsiKeep& k = ctx.psi_keep;
  if (k.valid && same_spec(k.spec, psi) && k.row0 == row0 && k.rows == rows) return view_of_buf(k.buf, psi.rows, rows);
  tmp = DevQMat(ctx, psi.rows, rows);
  launch_gen(ctx.stream, psi, 0, row0, psi.rows, rows, tmp.v, false);
  return tmp.v;
}

bool psi8_gemm(Ctx& ctx, const qlra_spec_t& psi, int64_t row0, const QView& B, const QView& C) {
  {
    // long contraction (Psi H over all local rows): the int8 engine on the
    // kept fp64 Psi block
    const Ctx::PsiKeep& pk = ctx.psi_keep;
    if (pk.valid && same_spec(pk.spec, psi) && pk.row0 == row0 && pk.rows == B.rows && C.rows == psi.rows &&
        C.cols == B.cols &&
        oz_gemm_try(ctx, QLRA_OP_N, QLRA_OP_N, 1.0, view_of_buf(pk.buf, psi.rows, B.rows), B, 0.0, C))
      return true;
  }
  const Ctx::CombKeep& k = ctx.comb_keep;
  if (!k.psi_valid || !same_spec(k.psi, psi) || k.row0 != row0 || k.rows != B.rows || C.rows != psi.rows ||
      C.cols != B.cols || B.rows == 0 || B.cols == 0)
    return false;
  set_kernel_attrs();
  SketchWork ws;
  const Q8Part w{B, k.ps8, k.ps8_ld, 0, C};
  launch8(ctx, nullptr, &w, 1.0, 0.0, ws, false);
  return true;
}

bool q8gram(Ctx& ctx, const QView& Y, const QView& G) {
  const int64_t m = Y.rows, s = Y.cols;
  int64_t pstride = 0;
  // s >= 96 (QLRA_Q8GRAM_MIN_S): narrower Grams leave most of the 64 x 32
  // tiles' warps without a block (C5, s = 40: 3.5 -> 4.7 ms); the
  // 16-product 64 x 64 Hermitian path is faster there (C2, s = 100: 8-product
  // one-pass 9.68 ms vs 9.74)
  static const int64_t smin = [] {
    const char* e = std::getenv("QLRA_Q8GRAM_MIN_S");
    return e ? std::atoll(e) : 96;
  }();
  const bool small = s <= qt8::Cfg<5>::TM;  // whole Gram in one tile (mode 5)
  if (!sketch_use8() || !sketch_tma_enabled() || (!small && s < smin) || s > 512 || m < 4 * s || G.rows != s ||
      G.cols != s ||
      !tma_layout(Y, &pstride))
    return false;
  static const bool enabled = [] {
    const char* e = std::getenv("QLRA_Q8GEMM");
    return !(e && std::atoi(e) == 0);
  }();
  if (!enabled) return false;
  using CG = qt8::Cfg<4>;
  Gram8Args f{};
  if (small ? !make_map3(&f.lm, Y.p[0], s, m, 4, Y.ld, pstride, qt8::Layout<5>::LDL, qt8::BK, 4)
            : (!make_map3(&f.lm, Y.p[0], s, m, 4, Y.ld, pstride, qt8::Layout<4>::LDL, qt8::BK, 4) ||
               !make_map3(&f.rm, Y.p[0], s, m, 4, Y.ld, pstride, qt8::Layout<4>::LDX, qt8::BK, 4)))
    return false;
  int nt = 0;
  if (small) {
    f.tm[0] = f.tn[0] = 0;
    nt = 1;
  }
  for (int tn = 0; !small && tn < (int)((s + CG::TN - 1) / CG::TN); ++tn)
    for (int tm = 0; tm < (int)((s + CG::TM - 1) / CG::TM); ++tm)
      if ((int64_t)tm * CG::TM < (int64_t)(tn + 1) * CG::TN) {  // touches the upper triangle
        if (nt == GRAM_MAXT) return false;
        f.tm[nt] = (unsigned short)tm;
        f.tn[nt] = (unsigned short)tn;
        ++nt;
      }
  f.ntiles = nt;
  for (int p = 0; p < 4; ++p) {
    f.op.l[p] = Y.p[p];
    f.op.r[p] = Y.p[p];
    f.g[p] = G.p[p];
  }
  f.op.M = f.op.N = s;
  f.ldg = G.ld;
  f.K = m;
  // split K so that about two waves of CTAs run, >= 16 k-steps each
  int64_t zk = std::max<int64_t>(1, std::min<int64_t>((296 + nt - 1) / nt, m / (16 * qt8::BK)));
  f.kchunk = ((m + zk - 1) / zk + qt8::BK - 1) / qt8::BK * qt8::BK;
  f.zk = (int)((m + f.kchunk - 1) / f.kchunk);
  DeviceBuffer part;
  if (f.zk > 1) {
    part = DeviceBuffer(ctx, (size_t)f.zk * 4 * s * s * sizeof(double));
    f.part = part.as<double>();
  }
  f.stride = qt8::STAGE;
  f.stages = tma_stages(f.stride, 0);
  set_kernel_attrs();
  const size_t smem = (size_t)f.stages * f.stride * sizeof(double) + 128;
  if (small)
    gram8_kernel<5><<<(unsigned)(nt * f.zk), qt8::NT_TMA, smem, ctx.stream>>>(f);
  else
    gram8_kernel<4><<<(unsigned)(nt * f.zk), qt8::NT_TMA, smem, ctx.stream>>>(f);
  QLRA_LAUNCH_CHECK();
  count_launch();
  if (f.zk > 1) splitk_reduce(ctx, f.part, f.zk, G, 1.0, 0.0);
  mirror_upper(ctx, G);
  return true;
}

void psi_keep_release(Ctx& ctx) {
  Ctx::PsiKeep& k = ctx.psi_keep;
  if (k.buf) cudaFreeAsync(k.buf, ctx.stream);
  k = Ctx::PsiKeep{};
  if (ctx.comb_keep.buf) cudaFreeAsync(ctx.comb_keep.buf, ctx.stream);
  ctx.comb_keep = Ctx::CombKeep{};
}

void sketch_update_rows(Ctx& ctx, const qlra_spec_t& omega, const qlra_spec_t& psi, int64_t row0,
                        const QView& block, const QView& y_rows, const QView& w) {
  const int64_t b = block.rows, n = block.cols, s = omega.cols;
  if (b == 0 || n == 0) return;
  if (oz_wanted(ctx, n, s, psi.rows)) {
    // int8 tensor-core engine (ozaki.cu): no TMA alignment needed
    DevQMat om(ctx, n, s), ps_tmp;
    launch_gen(ctx.stream, omega, 0, 0, n, s, om.v, false);
    Emb e;
    e.om = om.v;
    e.ps = psi_for_sketch(ctx, psi, row0, b, ps_tmp);
    prepare_emb(ctx, e, psi, row0);  // keeps the combined Psi block for the core solve (psi8_gemm)
    if (oz_sketch_block(ctx, e.om, e.ps, block, y_rows, w)) return;
    // non-finite entries: the FP64 engine below
  }
  int64_t pstride = 0;
  if (sketch_use8() && sketch_tma_enabled() && !tma_layout(block, &pstride) && n >= 1024) {
    // A's rows are not 16-byte aligned (n odd, e.g. C4's 27125): stream the
    // block through even-pitched staging buffers (device-to-device copies
    // overlapped with the sketch of the previous chunk) so the TMA path
    // applies (C4: the staged copies overlap the previous panel's sketch;
    // sketch 693 ms against 723 ms on the cp.async path)
    sketch_update_rows_host(ctx, omega, psi, row0, block, y_rows, w, 0, true);
    return;
  }
  set_kernel_attrs();
  DevQMat om(ctx, n, s), ps_tmp;
  launch_gen(ctx.stream, omega, 0, 0, n, s, om.v, false);
  Emb e;
  e.om = om.v;
  e.ps = psi_for_sketch(ctx, psi, row0, b, ps_tmp);
  prepare_emb(ctx, e, psi, row0);
  const int64_t R = panel_rows(n, b);
  SketchWork ws;
  for (int64_t r0 = 0; r0 < b; r0 += R) {
    const int64_t rp = std::min(R, b - r0);
    sketch_panel(ctx, e, r0, sub(block, r0, 0, rp, n), sub(y_rows, r0, 0, rp, s), w, ws);
  }
}

// Streaming ingestion (sketch_from_source, sketching.cpp:156-167, with the
// source in host memory): row chunks are copied H2D on a dedicated stream into
// a double buffer while the previous chunk is sketched, so the PCIe transfer
// of A overlaps the FP64 work.  A is still read exactly once.  Sources:
//  * direct: pinned host rows (or, for the relayout of a device-resident A
//    whose rows are not 16-byte aligned, device rows) -- one DMA per plane;
//  * staged: host rows the DMA engine cannot read at full speed or at all
//    (pageable memory, a file): a host-side `fill` writes each chunk into a
//    pinned staging buffer (double-buffered, kept in the context) while the
//    previous chunk's DMA and sketch run.
namespace {

// RAII for the pipeline's copy stream and events: on any exit (including an
// exception thrown by a launch) the copy stream is drained before the device
// and staging buffers it reads or writes are released.
struct CopyPipe {
  cudaStream_t cs = nullptr;
  cudaEvent_t copied[2] = {nullptr, nullptr}, freed[2] = {nullptr, nullptr};
  CopyPipe() {
    QLRA_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      QLRA_CUDA(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
      QLRA_CUDA(cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming));
    }
  }
  ~CopyPipe() {
    if (cs) cudaStreamSynchronize(cs);
    for (int i = 0; i < 2; ++i) {
      if (copied[i]) cudaEventDestroy(copied[i]);
      if (freed[i]) cudaEventDestroy(freed[i]);
    }
    if (cs) cudaStreamDestroy(cs);
  }
  CopyPipe(const CopyPipe&) = delete;
  CopyPipe& operator=(const CopyPipe&) = delete;
};

// Pinned staging of the context (grown on demand, kept: a 2 x 100 MB
// cudaMallocHost per call would cost more than the copies it feeds).
double* staging(Ctx& ctx, size_t doubles) {
  if (ctx.staging_n < doubles) {
    if (ctx.staging) {
      QLRA_CUDA(cudaStreamSynchronize(ctx.stream));
      QLRA_CUDA(cudaFreeHost(ctx.staging));
    }
    ctx.staging = nullptr;
    ctx.staging_n = 0;
    QLRA_CUDA(cudaMallocHost(&ctx.staging, doubles * sizeof(double)));
    ctx.staging_n = doubles;
  }
  return ctx.staging;
}

}  // namespace

void sketch_rows_pipeline(Ctx& ctx, const qlra_spec_t& omega, const qlra_spec_t& psi, int64_t row0, int64_t b,
                          int64_t n, const RowSource& src, const QView& y_rows, const QView& w,
                          int64_t block_rows, bool relayout) {
  const int64_t s = omega.cols;
  if (b == 0 || n == 0) return;
  set_kernel_attrs();
  // (relayout of a device-resident A: panel-sized chunks, no short tail --
  // a device-to-device copy never bounds the pipeline)
  int64_t R = block_rows > 0 ? block_rows : relayout ? panel_rows(n, b) : stream_rows(n, b);
  R = std::min(R, b);
  DevQMat om(ctx, n, s), ps_tmp;
  // Device buffers with an even leading dimension: the copy lands A in the
  // layout the TMA path needs (16-byte rows) even when n is odd (C4's
  // 27125), at the cost of a pitched copy -- fine for wide rows.
  const int64_t ldb = (n % 2 == 0 || n < 1024) ? n : n + 1;
  DeviceBuffer bufmem[2] = {DeviceBuffer(ctx, (size_t)4 * R * ldb * sizeof(double)),
                            DeviceBuffer(ctx, (size_t)4 * R * ldb * sizeof(double))};
  QView buf[2];
  for (int i = 0; i < 2; ++i) {
    for (int p = 0; p < 4; ++p) buf[i].p[p] = bufmem[i].as<double>() + (size_t)p * R * ldb;
    buf[i].rows = R;
    buf[i].cols = n;
    buf[i].ld = ldb;
  }
  const bool staged = src.kind == RowSource::kStaged;
  double* stage[2] = {nullptr, nullptr};
  if (staged) {
    double* sb = staging(ctx, (size_t)8 * R * n);
    stage[0] = sb;
    stage[1] = sb + (size_t)4 * R * n;
  }
  CopyPipe pipe;  // declared after every buffer it touches: drained first
  // the buffers were allocated on ctx.stream: the copy stream waits for
  // that, and only that -- Omega / Psi generation below overlaps the first
  // H2D chunk
  QLRA_CUDA(cudaEventRecord(pipe.freed[0], ctx.stream));
  QLRA_CUDA(cudaEventRecord(pipe.freed[1], ctx.stream));
  launch_gen(ctx.stream, omega, 0, 0, n, s, om.v, false);
  Emb e;
  e.om = om.v;
  e.ps = psi_for_sketch(ctx, psi, row0, b, ps_tmp);
  prepare_emb(ctx, e, psi, row0);
  SketchWork ws;
  // the int8 engine takes the chunks when it is selected for these shapes
  // (max |A| of each chunk is taken on the copy stream right after its DMA,
  // so the host reads it without waiting for the previous chunk's work)
  std::unique_ptr<OzRun> oz;
  if (oz_wanted(ctx, n, s, psi.rows)) oz.reset(new OzRun(ctx, e.om, e.ps, b));
  // The last R rows go in quarter-size chunks: the sketch of the final chunk
  // is the one part of the pipeline nothing overlaps (the copy stream is the
  // bottleneck before it), so it should be short.
  const int64_t tail_start = !relayout && b > 2 * R ? b - R : b;
  const int64_t Rt = std::max<int64_t>(64, ((R / 4 + 63) / 64) * 64);
  // ...and the first chunks ramp up (R/8, R/4, R/2): the copy of the first
  // chunk is the one part nothing overlaps at the start (C4: 1.7 GB at
  // 55 GB/s = 31 ms before the first sketch launch otherwise)
  const bool ramp = !relayout && b > 4 * R;
  int chunk = 0;
  int idx = 0;
  for (int64_t r0 = 0, rp = 0; r0 < b; r0 += rp, idx ^= 1, ++chunk) {
    rp = std::min(r0 >= tail_start ? Rt : std::min(R, tail_start - r0), b - r0);
    if (ramp && chunk < 3)
      rp = std::min(rp, std::max<int64_t>(256, (((R >> (3 - chunk)) + 63) / 64) * 64));
    const QView dst = sub(buf[idx], 0, 0, rp, n);
    const double* from[4];
    int64_t from_ld = n;
    cudaMemcpyKind kind = cudaMemcpyHostToDevice;
    if (staged) {
      // staging buffer idx is free once its previous DMA has completed
      QLRA_CUDA(cudaEventSynchronize(pipe.copied[idx]));
      src.fill(r0, rp, stage[idx]);
      for (int p = 0; p < 4; ++p) from[p] = stage[idx] + (size_t)p * rp * n;
    } else {
      for (int p = 0; p < 4; ++p) from[p] = src.direct.p[p] + r0 * src.direct.ld;
      from_ld = src.direct.ld;
      kind = src.copy_kind;
    }
    QLRA_CUDA(cudaStreamWaitEvent(pipe.cs, pipe.freed[idx], 0));
    for (int p = 0; p < 4; ++p) {
      if (from_ld == n && dst.ld == n) {
        // contiguous rows: one linear DMA (2D copies of narrow rows, e.g.
        // C5's 2400-byte rows, run far below PCIe bandwidth)
        QLRA_CUDA(cudaMemcpyAsync(dst.p[p], from[p], sizeof(double) * (size_t)(rp * n), kind, pipe.cs));
      } else {
        QLRA_CUDA(cudaMemcpy2DAsync(dst.p[p], (size_t)dst.ld * sizeof(double), from[p],
                                    (size_t)from_ld * sizeof(double), (size_t)n * sizeof(double), (size_t)rp,
                                    kind, pipe.cs));
      }
    }
    if (oz) oz->amax_async(dst, pipe.cs, idx);
    QLRA_CUDA(cudaEventRecord(pipe.copied[idx], pipe.cs));
    QLRA_CUDA(cudaStreamWaitEvent(ctx.stream, pipe.copied[idx], 0));
    if (oz) QLRA_CUDA(cudaEventSynchronize(pipe.copied[idx]));
    if (oz && std::isfinite(oz->amax_host(idx))) {
      oz->panel(r0, dst, sub(y_rows, r0, 0, rp, s), w, oz->amax_host(idx), 1);
    } else {
      // (a chunk with NaN / inf takes the FP64 engine: its products add into
      // W directly, beside the int8 engine's pending epoch)
      sketch_panel(ctx, e, r0, dst, sub(y_rows, r0, 0, rp, s), w, ws);
    }
    QLRA_CUDA(cudaEventRecord(pipe.freed[idx], ctx.stream));
  }
  if (oz) oz->finish(w);
}

// Host rows of a (4-plane, ld) host matrix copied into pinned staging by
// several host threads (pageable memcpy runs at ~10 GB/s per thread; PCIe
// takes ~55 GB/s).
void parallel_fill(const QView& host, int64_t r0, int64_t rows, double* dst) {
  const int64_t n = host.cols;
  const size_t bytes = (size_t)(4 * rows * n) * sizeof(double);
  // 8 threads, >= 8 MB each (14 threads measured slower on the 16-thread
  // host: C4 pageable e2e 1.15 s against 0.98 -- they compete with the DMA
  // for host memory bandwidth)
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(8, (int64_t)(bytes >> 23)));
  auto work = [&](int t) {
    for (int p = 0; p < 4; ++p) {
      const int64_t i0 = rows * t / nt, i1 = rows * (t + 1) / nt;
      double* d = dst + (size_t)p * rows * n;
      const double* sp = host.p[p] + (r0 + i0) * host.ld;
      if (host.ld == n) {
        std::memcpy(d + i0 * n, sp, sizeof(double) * (size_t)((i1 - i0) * n));
      } else {
        for (int64_t i = i0; i < i1; ++i) std::memcpy(d + i * n, sp + (i - i0) * host.ld, sizeof(double) * n);
      }
    }
  };
  if (nt == 1) {
    work(0);
    return;
  }
  std::vector<std::thread> ts;
  for (int t = 1; t < nt; ++t) ts.emplace_back(work, t);
  work(0);
  for (auto& t : ts) t.join();
}

void sketch_update_rows_host(Ctx& ctx, const qlra_spec_t& omega, const qlra_spec_t& psi,
                             int64_t row0, const QView& host_block, const QView& y_rows,
                             const QView& w, int64_t block_rows, bool relayout) {
  RowSource src;
  src.kind = RowSource::kDirect;
  src.direct = host_block;
  src.copy_kind = relayout ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (!relayout && host_block.rows > 0 && host_block.cols > 0) {
    // Pageable host memory (a reference QMatrix's std::vector planes): the
    // DMA engine would stage it through a driver bounce buffer synchronously,
    // serialising the pipeline; copy it into pinned staging on host threads
    // instead, overlapped with the previous chunk's DMA and sketch.
    cudaPointerAttributes at{};
    bool pinned = true;
    for (int p = 0; p < 4 && pinned; ++p) {
      if (cudaPointerGetAttributes(&at, host_block.p[p]) != cudaSuccess) {
        cudaGetLastError();
        pinned = false;
      } else {
        pinned = at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeDevice ||
                 at.type == cudaMemoryTypeManaged;
      }
    }
    if (!pinned) {
      src.kind = RowSource::kStaged;
      const QView hb = host_block;
      src.fill = [hb](int64_t r0, int64_t rows, double* dst) { parallel_fill(hb, r0, rows, dst); };
    }
  }
  sketch_rows_pipeline(ctx, omega, psi, row0, host_block.rows, host_block.cols, src, y_rows, w, block_rows,
                       relayout);
}

}  // namespace qlra_dev
