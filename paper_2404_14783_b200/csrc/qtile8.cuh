// qtile8.cuh -- the sketch's tile engine: quaternion products with EIGHT real
// matrix products instead of sixteen.
//
// A quaternion product c = a b (Hamilton table, proj/include/qlra/
// quaternion.hpp:33-38) is a real bilinear map of rank 8 (Howell & Lafon,
// 1975).  With planes (w, x, y, z) = (0, 1, 2, 3):
//
//   m1 = (a0 + a1)(b0 + b1)      m5 = (a1 + a3)(b1 + b2)/2
//   m2 = (a3 - a2)(b2 - b3)      m6 = (a1 - a3)(b1 - b2)/2
//   m3 = (a0 - a1)(b2 + b3)      m7 = (a0 + a2)(b0 - b3)/2
//   m4 = (a2 + a3)(b0 - b1)      m8 = (a0 - a2)(b0 + b3)/2
//
//   c0 = m2 - m5 - m6 + m7 + m8      c1 = m1 - m5 - m6 - m7 - m8
//   c2 = m3 + m5 - m6 + m7 - m8      c3 = m4 + m5 - m6 - m7 + m8
//
// Every m_i keeps a on the left and b on the right, so the identity holds for
// matrix entries as well: a quaternion GEMM is 8 real GEMMs of plane
// combinations, 8 accumulators per output element.  On B200 the FP64 tensor
// op (DMMA.8x8x4) and DFMA share one pipe of 64 FMA/clk/SM, so the DMMA count
// is the cost: half of the 16-product engine (qtile.cuh), plus the pairwise
// sums that form the combinations (DADD, 1/8 of a DMMA each).
//
// The sketch products are Y = A Omega and W = Psi A.  The embedding side is
// combined ONCE in HBM (8 planes, halves folded into combinations 5..8:
// exact, a power of two), the A side in registers from the 4 staged planes
// (A is read once and never rewritten):
//
//   Y task: C 64x32 = A (k-fast, 4 planes) x Omega~ (j-fast, 8 planes);
//   W task: C 32x64 = Psi~ (k-fast, 8 planes) x A (j-fast, 4 planes).
//
// Paired warps.  512 threads = 8 warp-tile positions (16x16 outputs, 2x2
// blocks of 8x8) x 2 product halves: warp w covers position w & 7 and
// products 4*(w >> 3) .. +3, so each warp holds 4 products x 4 blocks x 2 =
// 32 FP64 accumulators (the 128-register cap of 512 threads) and forms only
// its own 4 combinations.  Measured alternatives: 16 warps of 16x8 tiles
// with all 8 products (one sum per DMMA, register-starved schedule) and 8
// warps of 16x16 tiles with all 8 products (2 warps per SM sub-partition
// cannot cover the DADD -> DMMA and LDS -> DMMA latencies) reached 61% / 70%
// of the DMMA pipe.  The halves meet in the epilogue through shared memory.
//
// Rounding: every product and sum is an IEEE operation in a fixed order
// (deterministic); the combination sums add at most a few ulp of |a||b| per
// term, the same order as the 16-product sum (the sketch is compared with the
// oracle at 1e-13 relative).
#pragma once

#include <cuda.h>

#include "qtile.cuh"

namespace qlra_dev {
namespace qt8 {

constexpr int NT = 512, BK = 8, STAGES = 4;
// TMA launches add one producer warp (warp 16) that only issues the stage
// copies, so no compute warp ever waits on a slot's release
constexpr int NT_TMA = NT + 32;
constexpr int LDK = BK + 4;  // k-fast rows, pitch 12 (4 mod 16: conflict-free fragments)

// Tile configurations (MODE): 8 positions of 16x16 outputs as PR x PC.
//   0 Y : 64 x 32, left A on the fly (k-fast), right Omega~ (8 planes)
//   1 W : 32 x 64, left Psi~ (8 planes), right A on the fly (j-fast)
//   2 YN: 128 x 16, as Y -- the last Y column tile when s % 32 <= 16
//   3 WN: 16 x 128, as W -- the last W row tile when l % 32 <= 16
//   4 G : 64 x 32 of a Gram Y^* Y -- both operands on the fly from Y's 4
//         planes, the left one as the adjoint (i-fast in memory, conjugated
//         in registers); warp positions below the diagonal issue no DMMA
//   5 SG: the whole Gram of a narrow Y (s <= 48) in one tile: the 6 upper
//         16x16 blocks of a 3 x 3 grid as 6 positions, both operands read
//         from ONE staged k-slice of Y (one TMA box per stage)
// The narrow modes keep all 16 warps busy on a remainder that would leave
// half of a regular tile's warps without a valid 8x8 block.
template <int MODE>
struct Cfg {
  static constexpr bool GRAM = MODE == 4 || MODE == 5;
  static constexpr bool SMALL = MODE == 5;
  static constexpr bool LPRE = !GRAM && (MODE & 1) != 0;
  static constexpr int PR = MODE == 0 || MODE == 4 ? 4 : MODE == 1 ? 2 : MODE == 2 ? 8 : MODE == 5 ? 3 : 1;
  static constexpr int PC = MODE == 5 ? 3 : 8 / PR;
  static constexpr int TM = 16 * PR, TN = 16 * PC, WRB = 2, WCB = 2;
  static constexpr int LP = LPRE ? 8 : 4, RP = LPRE || GRAM ? 4 : 8;
};
// Warp w issues on SMSP w % 4.  The position index runs fastest along the
// long side of the position grid, so the warps of a tile padded along the
// short side still cover all four SMSPs (two warps each: both product halves).
template <int MODE>
__device__ __forceinline__ int warp_row(int w) {
  using C = Cfg<MODE>;
  if constexpr (C::SMALL) return (0x33211000u >> (4 * (w & 7))) & 0xF;  // upper blocks of 3x3; 6, 7 -> 3 (idle)
  return C::PR >= C::PC ? (w & 7) % C::PR : (w & 7) / C::PC;
}
template <int MODE>
__device__ __forceinline__ int warp_col(int w) {
  using C = Cfg<MODE>;
  if constexpr (C::SMALL) return (0x33221210u >> (4 * (w & 7))) & 0xF;
  return C::PR >= C::PC ? (w & 7) / C::PR : (w & 7) % C::PC;
}
__device__ __forceinline__ int warp_half(int w) { return w >> 3; }

template <int MODE>
struct Layout {
  using C = Cfg<MODE>;
  static constexpr int LDX = C::TN + 4;  // j-fast rows: 36 / 68 / 20 / 132 (4 mod 16)
  static constexpr int LDL = C::TM + 4;  // i-fast left rows (Gram): 68 / 52
  static constexpr int L_ELEMS = C::GRAM ? C::LP * BK * LDL : C::LP * C::TM * LDK;
  static constexpr int R_ELEMS = C::SMALL ? 0 : C::RP * BK * LDX;  // SG: the right operand is the same slice
  static constexpr int ELEMS = L_ELEMS + R_ELEMS;
};
constexpr int cmax(int a, int b) { return a > b ? a : b; }
// stage stride of the cp.async path (regular modes only) and of the TMA path
constexpr int STAGE = cmax(Layout<0>::ELEMS, Layout<1>::ELEMS);
constexpr int STAGE_TMA = cmax(STAGE, cmax(Layout<2>::ELEMS, Layout<3>::ELEMS));
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE * sizeof(double);

// op(L)(i, k) = l[q][i * l_si + k];  op(R)(k, j) = r[q][k * r_sk + j]
struct Operands {
  const double* l[8];
  const double* r[8];
  int64_t l_si, r_sk;
  int64_t M, N;
};

// combination i of a's planes (left side, on the fly: no halves)
__device__ __forceinline__ double lcomb(int i, const double (&a)[4]) {
  switch (i) {
    case 0: return a[0] + a[1];
    case 1: return a[3] - a[2];
    case 2: return a[0] - a[1];
    case 3: return a[2] + a[3];
    case 4: return a[1] + a[3];
    case 5: return a[1] - a[3];
    case 6: return a[0] + a[2];
    default: return a[0] - a[2];
  }
}
// combination i of b's planes (right side, on the fly: no halves)
__device__ __forceinline__ double rcomb(int i, const double (&b)[4]) {
  switch (i) {
    case 0: return b[0] + b[1];
    case 1: return b[2] - b[3];
    case 2: return b[2] + b[3];
    case 3: return b[0] - b[1];
    case 4: return b[1] + b[2];
    case 5: return b[1] - b[2];
    case 6: return b[0] - b[3];
    default: return b[0] + b[3];
  }
}

// Accumulators of one warp: acc[ii][rb][cb][h] = product m_{4*half + ii + 1}
// at row 16*warp_row + 8*rb + lane/4, col 16*warp_col + 8*cb + 2*(lane%4) + h.
using Acc = double[4][2][2][2];

__device__ __forceinline__ void zero_acc(Acc& acc) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int rb = 0; rb < 2; ++rb)
#pragma unroll
      for (int cb = 0; cb < 2; ++cb) acc[i][rb][cb][0] = acc[i][rb][cb][1] = 0.0;
}

// the quaternion planes from the 8 products (fixed summation order)
__device__ __forceinline__ void combine(const double (&m)[8], double (&c)[4]) {
  const double s56 = m[4] + m[5], d78 = m[6] - m[7];
  c[0] = m[1] - s56 + (m[6] + m[7]);
  c[1] = m[0] - s56 - (m[6] + m[7]);
  c[2] = m[2] + (m[4] - m[5]) + d78;
  c[3] = m[3] + (m[4] - m[5]) - d78;
}

template <int MODE>
__device__ __forceinline__ int acc_row(int rb) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  return 16 * warp_row<MODE>(w) + 8 * rb + (lane >> 2);
}
template <int MODE>
__device__ __forceinline__ int acc_col(int cb) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  return 16 * warp_col<MODE>(w) + 8 * cb + 2 * (lane & 3);
}

// Per-thread copy plan of one tile, fixed for the whole k loop: each thread
// copies the same (row, k) / (k, col) position of LP / RP planes every stage,
// so a stage costs a pointer add per operand and the k bound test (the
// general address arithmetic once per tile, not once per element per stage).
template <int MODE>
struct Loader {
  using C = Cfg<MODE>;
  using Lay = Layout<MODE>;
  static constexpr int LPER = C::TM * BK, RPER = BK * C::TN;  // elements per plane per stage
  static constexpr int LSPLIT = NT / LPER, RSPLIT = NT / RPER;   // thread groups per copy round
  static_assert(NT % LPER == 0 && NT % RPER == 0, "copy plan");
  static_assert(C::LP % LSPLIT == 0 && C::RP % RSPLIT == 0, "copy plan");
  static constexpr int LCOPIES = C::LP / LSPLIT, RCOPIES = C::RP / RSPLIT;
  int64_t loff, roff, rstep;
  int lk, rk, lhi, rhi, ldst, rdst;
  bool lrow, rcol;
  __device__ __forceinline__ Loader(const Operands& g, int64_t i0, int64_t j0, int64_t kbeg, int tid) {
    const int lidx = tid % LPER, ridx = tid % RPER;
    lhi = tid / LPER;
    rhi = tid / RPER;
    const int lx = lidx / BK, rx = ridx % C::TN;
    lk = lidx % BK;
    rk = ridx / C::TN;
    lrow = i0 + lx < g.M;
    rcol = j0 + rx < g.N;
    loff = (lrow ? (i0 + lx) * g.l_si : 0) + kbeg + lk;
    roff = (kbeg + rk) * g.r_sk + (rcol ? j0 + rx : 0);
    rstep = (int64_t)BK * g.r_sk;
    ldst = (lhi * C::TM + lx) * LDK + lk;
    rdst = (rhi * BK + rk) * Lay::LDX + rx;
  }
  // copy stage starting at k0 (the offsets are then advanced to k0 + BK)
  __device__ __forceinline__ void stage(const Operands& g, double* Ls, double* Rs, int64_t k0, int64_t kend) {
    const bool lok = lrow && k0 + lk < kend, rok = rcol && k0 + rk < kend;
#pragma unroll
    for (int r = 0; r < LCOPIES; ++r) {
      const double* base = LSPLIT == 1 ? g.l[r] : (lhi ? g.l[LSPLIT * r + 1] : g.l[LSPLIT * r]);
      qt::cp_async8(Ls + ldst + r * LSPLIT * C::TM * LDK, lok ? base + loff : base, lok);
    }
#pragma unroll
    for (int r = 0; r < RCOPIES; ++r) {
      const double* base = RSPLIT == 1 ? g.r[r] : (rhi ? g.r[RSPLIT * r + 1] : g.r[RSPLIT * r]);
      qt::cp_async8(Rs + rdst + r * RSPLIT * BK * Lay::LDX, rok ? base + roff : base, rok);
    }
    loff += BK;
    roff += rstep;
  }
};

// One BK slice: products 4*HALF .. 4*HALF+3 for the warp's first NRB row and
// NCB column blocks.  Per k4 step all fragments are loaded and the warp's 4
// combinations formed before its 4*NRB*NCB DMMAs.
template <int MODE, int HALF, int NRB, int NCB>
__device__ __forceinline__ void kstep(const double* Ls, const double* Rs, int wr, int wc, int gid, int tig, Acc& acc) {
  using C = Cfg<MODE>;
  constexpr int LDX = Layout<MODE>::LDX;
#pragma unroll
  for (int kk = 0; kk < BK / 4; ++kk) {
    const int k = 4 * kk + tig;
    double lv[4][NRB], rv[4][NCB];
    if constexpr (C::GRAM) {
      // left = Y^* (i-fast, conjugated), right = Y (j-fast): both combined here
      constexpr int LDL = Layout<MODE>::LDL;
      const double* Rt = C::SMALL ? Ls : Rs;
      constexpr int LDR = C::SMALL ? LDL : LDX;
      double a[NRB][4], b[NCB][4];
#pragma unroll
      for (int rb = 0; rb < NRB; ++rb) {
        const int x = 16 * wr + 8 * rb + gid;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double v = Ls[(q * BK + k) * LDL + x];
          a[rb][q] = q == 0 ? v : -v;
        }
      }
#pragma unroll
      for (int cb = 0; cb < NCB; ++cb) {
        const int x = 16 * wc + 8 * cb + gid;
#pragma unroll
        for (int q = 0; q < 4; ++q) b[cb][q] = Rt[(q * BK + k) * LDR + x];
      }
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) {
#pragma unroll
        for (int rb = 0; rb < NRB; ++rb) lv[ii][rb] = lcomb(4 * HALF + ii, a[rb]);
#pragma unroll
        for (int cb = 0; cb < NCB; ++cb) rv[ii][cb] = rcomb(4 * HALF + ii, b[cb]);
      }
    } else if (!C::LPRE) {
      // left = A: 4 planes per row block, combined in registers
      double a[NRB][4];
#pragma unroll
      for (int rb = 0; rb < NRB; ++rb) {
        const int x = 16 * wr + 8 * rb + gid;
#pragma unroll
        for (int q = 0; q < 4; ++q) a[rb][q] = Ls[(q * C::TM + x) * LDK + k];
      }
#pragma unroll
      for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int cb = 0; cb < NCB; ++cb) rv[ii][cb] = Rs[((4 * HALF + ii) * BK + k) * LDX + 16 * wc + 8 * cb + gid];
#pragma unroll
      for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int rb = 0; rb < NRB; ++rb) lv[ii][rb] = lcomb(4 * HALF + ii, a[rb]);
    } else {
      // right = A: 4 planes per column block, combined in registers
      double b[NCB][4];
#pragma unroll
      for (int cb = 0; cb < NCB; ++cb) {
        const int x = 16 * wc + 8 * cb + gid;
#pragma unroll
        for (int q = 0; q < 4; ++q) b[cb][q] = Rs[(q * BK + k) * LDX + x];
      }
#pragma unroll
      for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int rb = 0; rb < NRB; ++rb) lv[ii][rb] = Ls[((4 * HALF + ii) * C::TM + 16 * wr + 8 * rb + gid) * LDK + k];
#pragma unroll
      for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int cb = 0; cb < NCB; ++cb) rv[ii][cb] = rcomb(4 * HALF + ii, b[cb]);
    }
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
      for (int rb = 0; rb < NRB; ++rb)
#pragma unroll
        for (int cb = 0; cb < NCB; ++cb) qt::dmma(acc[ii][rb][cb], lv[ii][rb], rv[ii][cb]);
  }
}

// The cp.async ring with mbarrier stage handoff (as qtile.cuh's mma_loop).
template <int MODE, int HALF, int NRB, int NCB>
__device__ __forceinline__ void mma_loop(const Operands& g, double* smem, int64_t i0, int64_t j0, int64_t kbeg,
                                         int64_t kend, Acc& acc, uint64_t* full, uint64_t* empty) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wr = warp_row<MODE>(w), wc = warp_col<MODE>(w);
  const int gid = lane >> 2, tig = lane & 3;
  const int nk = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;
  constexpr int LOFF = Layout<MODE>::L_ELEMS;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      qt::mbar_init(&full[s], NT);
      qt::mbar_init(&empty[s], NT / 32);
    }
  }
  __syncthreads();
  Loader<MODE> ld(g, i0, j0, kbeg, tid);
  if (nk > 0) {
    ld.stage(g, smem, smem + LOFF, kbeg, kend);
    qt::cp_async_arrive(&full[0]);
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % STAGES;
    const int nxt = kt + 1;
    if (nxt < nk) {
      const int sn = nxt % STAGES;
      if (nxt >= STAGES) qt::mbar_wait_parity(&empty[sn], (unsigned)((nxt / STAGES - 1) & 1));
      ld.stage(g, smem + sn * STAGE, smem + sn * STAGE + LOFF, kbeg + (int64_t)nxt * BK, kend);
      qt::cp_async_arrive(&full[sn]);
    }
    qt::mbar_wait_parity(&full[s], (unsigned)((kt / STAGES) & 1));
    const double* Ls = smem + s * STAGE;
    if (NRB > 0 && NCB > 0)
      kstep<MODE, HALF, (NRB > 0 ? NRB : 1), (NCB > 0 ? NCB : 1)>(Ls, Ls + LOFF, wr, wc, gid, tig, acc);
    __syncwarp();
    if (lane == 0) qt::mbar_arrive(&empty[s]);
  }
  qt::cp_async_wait<0>();
  __syncthreads();
}

// ---- TMA staging ------------------------------------------------------------
// With 3D tensor maps (inner, rows, planes) over each operand, one elected
// thread stages a whole operand tile per stage with one
// cp.async.bulk.tensor: no per-thread address arithmetic, and the edges
// (rows / columns / k past the extents) come back zero-filled.  Boxes are
// the padded smem rows themselves -- left {LDK, TM, LP}, right {LDX, BK, RP}
// -- so the pitches stay 12 / 36 / 68 (conflict-free fragment reads); the
// over-fetched columns are never read.  The caller creates the maps so that
// k past the chunk end is out of bounds in at least one operand, or chunks
// end on BK boundaries (split-K).
constexpr int MAX_STAGES = 6;
struct TmaOps {
  const CUtensorMap* lm;  // left map
  const CUtensorMap* rm;  // right map
  int lk_off;             // inner coordinate offset of the left map's k (Psi~ panel column)
  int stages;             // ring slots (<= MAX_STAGES, smem sized by the launch)
  int stride;             // doubles per slot (STAGE, or STAGE_TMA when the launch has narrow tiles)
};

__device__ __forceinline__ void tma_load3(double* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(qt::smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(0), "r"(qt::smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(qt::smem_u32(bar)), "r"(bytes) : "memory");
}

template <int MODE>
__device__ __forceinline__ void tma_stage(const TmaOps& t, double* Ls, double* Rs, int64_t i0, int64_t j0, int64_t k0,
                                          uint64_t* bar) {
  constexpr unsigned BYTES = (unsigned)((Layout<MODE>::L_ELEMS + Layout<MODE>::R_ELEMS) * sizeof(double));
  mbar_expect_tx(bar, BYTES);
  if constexpr (Cfg<MODE>::GRAM)
    tma_load3(Ls, t.lm, (int)i0, (int)k0, bar);  // Y rows k, columns i (the adjoint's rows)
  else
    tma_load3(Ls, t.lm, (int)(t.lk_off + k0), (int)i0, bar);
  if constexpr (!Cfg<MODE>::SMALL) tma_load3(Rs, t.rm, (int)j0, (int)k0, bar);
}

// The ring fed by a dedicated producer warp (warp 16, one elected lane):
// it issues stage k as soon as every compute warp has released the slot's
// previous stage; the 16 compute warps only wait for data.
template <int MODE>
__device__ __forceinline__ void tma_init(const TmaOps& t, uint64_t* full, uint64_t* empty) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < t.stages; ++s) {
      qt::mbar_init(&full[s], 1);
      qt::mbar_init(&empty[s], NT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

template <int MODE>
__device__ __forceinline__ void tma_producer(const TmaOps& t, double* smem, int64_t i0, int64_t j0, int64_t kbeg,
                                             int64_t kend, uint64_t* full, uint64_t* empty) {
  constexpr int LOFF = Layout<MODE>::L_ELEMS;
  const int nk = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;
  if ((threadIdx.x & 31) == 0) {
    const int S = t.stages;
    int s = 0, ph = 0;
    for (int kt = 0; kt < nk; ++kt) {
      if (kt >= S) qt::mbar_wait_parity(&empty[s], (unsigned)((ph - 1) & 1));
      tma_stage<MODE>(t, smem + s * t.stride, smem + s * t.stride + LOFF, i0, j0, kbeg + (int64_t)kt * BK, &full[s]);
      if (++s == S) { s = 0; ++ph; }
    }
  }
  __syncwarp();
  __syncthreads();  // pairs with the compute warps' closing barrier
}

template <int MODE, int HALF, int NRB, int NCB>
__device__ __forceinline__ void mma_loop_tma(const TmaOps& t, double* smem, int64_t i0, int64_t j0, int64_t kbeg,
                                             int64_t kend, Acc& acc, uint64_t* full, uint64_t* empty) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wr = warp_row<MODE>(w), wc = warp_col<MODE>(w);
  const int gid = lane >> 2, tig = lane & 3;
  const int nk = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;
  constexpr int LOFF = Layout<MODE>::L_ELEMS;
  const int S = t.stages;
  int s = 0, ph = 0;
  for (int kt = 0; kt < nk; ++kt) {
    qt::mbar_wait_parity(&full[s], (unsigned)(ph & 1));
    const double* Ls = smem + s * t.stride;
    if (NRB > 0 && NCB > 0)
      kstep<MODE, HALF, (NRB > 0 ? NRB : 1), (NCB > 0 ? NCB : 1)>(Ls, Ls + LOFF, wr, wc, gid, tig, acc);
    __syncwarp();
    if (lane == 0) qt::mbar_arrive(&empty[s]);
    if (++s == S) { s = 0; ++ph; }
  }
  // every issued stage was consumed (waited on full) before the loop ended
  __syncthreads();
}

// The warp's loop instance: product half, and the count of its 8x8 row /
// column blocks inside M x N (blocks past the edge issue no DMMA).
template <int MODE>
__device__ __forceinline__ int instance(const Operands& g, int64_t i0, int64_t j0) {
  const int w = threadIdx.x >> 5;
  const int64_t r0w = i0 + 16 * warp_row<MODE>(w), c0w = j0 + 16 * warp_col<MODE>(w);
  const int nrb = r0w >= g.M ? 0 : (int)min((int64_t)2, (g.M - r0w + 7) / 8);
  const int ncb = c0w >= g.N ? 0 : (int)min((int64_t)2, (g.N - c0w + 7) / 8);
  if (Cfg<MODE>::GRAM && r0w >= c0w + 16) return 0;  // strictly below the diagonal: mirrored later
  return (nrb == 0 || ncb == 0) ? 0 : warp_half(w) * 16 + nrb * 4 + ncb;
}

#define QT8_DISPATCH(LOOP, ...)                                             \
  switch (instance<MODE>(g, i0, j0)) {                                      \
    case 0 * 16 + 2 * 4 + 2: LOOP<MODE, 0, 2, 2>(__VA_ARGS__); break;       \
    case 0 * 16 + 2 * 4 + 1: LOOP<MODE, 0, 2, 1>(__VA_ARGS__); break;       \
    case 0 * 16 + 1 * 4 + 2: LOOP<MODE, 0, 1, 2>(__VA_ARGS__); break;       \
    case 0 * 16 + 1 * 4 + 1: LOOP<MODE, 0, 1, 1>(__VA_ARGS__); break;       \
    case 1 * 16 + 2 * 4 + 2: LOOP<MODE, 1, 2, 2>(__VA_ARGS__); break;       \
    case 1 * 16 + 2 * 4 + 1: LOOP<MODE, 1, 2, 1>(__VA_ARGS__); break;       \
    case 1 * 16 + 1 * 4 + 2: LOOP<MODE, 1, 1, 2>(__VA_ARGS__); break;       \
    case 1 * 16 + 1 * 4 + 1: LOOP<MODE, 1, 1, 1>(__VA_ARGS__); break;       \
    default: LOOP<MODE, 0, 0, 0>(__VA_ARGS__); break; /* loads + barriers */ \
  }

// acc (the warp's 4 products) over k in [kbeg, kend) for the tile at (i0, j0).
template <int MODE>
__device__ __forceinline__ void mma_tile(const Operands& g, double* smem, int64_t i0, int64_t j0, int64_t kbeg,
                                         int64_t kend, Acc& acc) {
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  QT8_DISPATCH(mma_loop, g, smem, i0, j0, kbeg, kend, acc, full, empty)
}
template <int MODE>
__device__ __forceinline__ void mma_tile_tma(const TmaOps& t, const Operands& g, double* smem, int64_t i0, int64_t j0,
                                             int64_t kbeg, int64_t kend, Acc& acc) {
  __shared__ __align__(8) uint64_t full[MAX_STAGES], empty[MAX_STAGES];
  tma_init<MODE>(t, full, empty);
  if ((threadIdx.x >> 5) == NT / 32) {
    tma_producer<MODE>(t, smem, i0, j0, kbeg, kend, full, empty);
    return;
  }
  QT8_DISPATCH(mma_loop_tma, t, smem, i0, j0, kbeg, kend, acc, full, empty)
}
#undef QT8_DISPATCH

// Epilogue exchange: the product-half-1 warps hand their accumulators to the
// half-0 warp of the same position through shared memory (lane-major,
// conflict-free).  `xbuf` needs 8 * 32 * 32 doubles; call after the k loop
// (which ends with a CTA barrier).  Returns the lane's slot for the half-0
// warps (read with other_product), nullptr for the half-1 warps.
__device__ __forceinline__ const double* exchange_products(const Acc& acc, double* xbuf) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w >= NT / 32) {  // the TMA producer warp holds no products
    __syncthreads();
    return nullptr;
  }
  double* slot = xbuf + (w & 7) * 32 * 32 + lane;
  if (warp_half(w) == 1) {
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
      for (int rb = 0; rb < 2; ++rb)
#pragma unroll
        for (int cb = 0; cb < 2; ++cb)
#pragma unroll
          for (int h = 0; h < 2; ++h) slot[32 * (((ii * 2 + rb) * 2 + cb) * 2 + h)] = acc[ii][rb][cb][h];
  }
  __syncthreads();
  return warp_half(w) == 1 ? nullptr : slot;
}
// product m_{5 + ii} of element (rb, cb, h) from the exchange slot
__device__ __forceinline__ double other_product(const double* slot, int ii, int rb, int cb, int h) {
  return slot[32 * (((ii * 2 + rb) * 2 + cb) * 2 + h)];
}

// ---- multi-tile streaming (small K) ---------------------------------------
// For products whose K spans only a few stages (Y R^-1: K = s), a CTA runs
// `ntiles` consecutive row tiles of one column tile with ONE continuous
// stage stream: the producer warp keeps loading the next tile's stages
// while the compute warps finish a tile and store it, so the TMA pipeline
// never drains and the per-CTA set-up is paid once.  The half exchange uses
// its own buffer (xbuf, outside the ring) and a named barrier of the 16
// compute warps (the producer warp never joins it).
__device__ __forceinline__ void compute_bar() { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); }

template <int MODE, int HALF, int NRB, int NCB>
__device__ __forceinline__ void consume_tile(const TmaOps& t, const double* smem, int nk, int& s, int& ph, Acc& acc,
                                             uint64_t* full, uint64_t* empty) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wr = warp_row<MODE>(w), wc = warp_col<MODE>(w);
  const int gid = lane >> 2, tig = lane & 3;
  constexpr int LOFF = Layout<MODE>::L_ELEMS;
  for (int kt = 0; kt < nk; ++kt) {
    qt::mbar_wait_parity(&full[s], (unsigned)(ph & 1));
    const double* Ls = smem + s * t.stride;
    if (NRB > 0 && NCB > 0)
      kstep<MODE, HALF, (NRB > 0 ? NRB : 1), (NCB > 0 ? NCB : 1)>(Ls, Ls + LOFF, wr, wc, gid, tig, acc);
    __syncwarp();
    if (lane == 0) qt::mbar_arrive(&empty[s]);
    if (++s == t.stages) { s = 0; ++ph; }
  }
}

// Row tiles i0 = i00 + r * TM (r < ntiles) at column j0 over k in [kbeg,
// kend); `store(acc, slot, i0)` runs on the compute warps after each tile
// (slot: exchange slot for half 0, nullptr for half 1).  xbuf: 8*32*32
// doubles outside the ring.
template <int MODE, class Store>
__device__ __forceinline__ void stream_tiles(const TmaOps& t, const Operands& g, double* smem, double* xbuf,
                                             int64_t i00, int ntiles, int64_t j0, int64_t kbeg, int64_t kend,
                                             Store store) {
  using C = Cfg<MODE>;
  __shared__ __align__(8) uint64_t full[MAX_STAGES], empty[MAX_STAGES];
  tma_init<MODE>(t, full, empty);
  const int nk = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w == NT / 32) {
    constexpr int LOFF = Layout<MODE>::L_ELEMS;
    if (lane == 0) {
      int s = 0, ph = 0, issued = 0;
      for (int r = 0; r < ntiles; ++r)
        for (int kt = 0; kt < nk; ++kt, ++issued) {
          if (issued >= t.stages) qt::mbar_wait_parity(&empty[s], (unsigned)((ph - 1) & 1));
          tma_stage<MODE>(t, smem + s * t.stride, smem + s * t.stride + LOFF, i00 + (int64_t)r * C::TM, j0,
                          kbeg + (int64_t)kt * BK, &full[s]);
          if (++s == t.stages) { s = 0; ++ph; }
        }
    }
    __syncwarp();
    __syncthreads();
    return;
  }
  int s = 0, ph = 0;
  for (int r = 0; r < ntiles; ++r) {
    const int64_t i0 = i00 + (int64_t)r * C::TM;
    Acc acc;
    zero_acc(acc);
    // the warp's instance for this tile (the last row tile may be partial)
    const int64_t r0w = i0 + 16 * warp_row<MODE>(w), c0w = j0 + 16 * warp_col<MODE>(w);
    const int nrb = r0w >= g.M ? 0 : (int)min((int64_t)2, (g.M - r0w + 7) / 8);
    const int ncb = c0w >= g.N ? 0 : (int)min((int64_t)2, (g.N - c0w + 7) / 8);
    const int inst = (nrb == 0 || ncb == 0) ? 0 : warp_half(w) * 16 + nrb * 4 + ncb;
    switch (inst) {
      case 0 * 16 + 2 * 4 + 2: consume_tile<MODE, 0, 2, 2>(t, smem, nk, s, ph, acc, full, empty); break;
      case 0 * 16 + 2 * 4 + 1: consume_tile<MODE, 0, 2, 1>(t, smem, nk, s, ph, acc, full, empty); break;
      case 0 * 16 + 1 * 4 + 2: consume_tile<MODE, 0, 1, 2>(t, smem, nk, s, ph, acc, full, empty); break;
      case 0 * 16 + 1 * 4 + 1: consume_tile<MODE, 0, 1, 1>(t, smem, nk, s, ph, acc, full, empty); break;
      case 1 * 16 + 2 * 4 + 2: consume_tile<MODE, 1, 2, 2>(t, smem, nk, s, ph, acc, full, empty); break;
      case 1 * 16 + 2 * 4 + 1: consume_tile<MODE, 1, 2, 1>(t, smem, nk, s, ph, acc, full, empty); break;
      case 1 * 16 + 1 * 4 + 2: consume_tile<MODE, 1, 1, 2>(t, smem, nk, s, ph, acc, full, empty); break;
      case 1 * 16 + 1 * 4 + 1: consume_tile<MODE, 1, 1, 1>(t, smem, nk, s, ph, acc, full, empty); break;
      default: consume_tile<MODE, 0, 0, 0>(t, smem, nk, s, ph, acc, full, empty); break;
    }
    // exchange the product halves (compute warps only), then store
    double* slot = xbuf + (w & 7) * 32 * 32 + lane;
    if (warp_half(w) == 1) {
#pragma unroll
      for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int rb = 0; rb < 2; ++rb)
#pragma unroll
          for (int cb = 0; cb < 2; ++cb)
#pragma unroll
            for (int h = 0; h < 2; ++h) slot[32 * (((ii * 2 + rb) * 2 + cb) * 2 + h)] = acc[ii][rb][cb][h];
    }
    compute_bar();
    store(acc, warp_half(w) == 1 ? nullptr : slot, i0);
    compute_bar();  // the slots are free for the next tile's exchange
  }
  __syncthreads();
}

}  // namespace qt8
}  // namespace qlra_dev
