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
//   YT (Y task): C 64x32 = A (k-fast, 4 planes) x Omega~ (j-fast, 8 planes),
//                warp tile 16x8 (2x1 blocks of 8x8);
//   WT (W task): C 32x64 = Psi~ (k-fast, 8 planes) x A (j-fast, 4 planes),
//                warp tile 8x16 (1x2 blocks).
//
// 512 threads as 4x4 warps, 8 products x 2 blocks x 2 = 32 FP64 accumulators
// per thread, as in qtile.cuh.  Rounding: every product and sum is an IEEE
// operation in a fixed order (deterministic); the combination sums add at
// most a few ulp of |a||b| per term, the same order as the 16-product sum
// (the sketch is compared with the oracle at 1e-13 relative).
#pragma once

#include <cuda.h>

#include "qtile.cuh"

namespace qlra_dev {
namespace qt8 {

constexpr int NT = 256, BK = 8, STAGES = 4;
constexpr int LDK = BK + 4;  // k-fast rows, pitch 12 (4 mod 16: conflict-free fragments)

// 8 warps of 16x16 output tiles (2x2 blocks of 8x8): 8 products x 4 blocks x 2
// = 64 FP64 accumulators per thread, up to 255 registers at 256 threads (one
// CTA per SM).  Against 16 warps of 16x8 tiles: half the plane sums and 3/4
// of the fragment loads per DMMA, and room for the sums' registers (at the
// 128-register cap of 512 threads the scheduler reused one register for
// every sum, serialising each DADD behind the previous DMMA's operand read).
template <bool LPRE>
struct Cfg;
template <>
struct Cfg<false> {  // Y task: left operand A (on the fly), right Omega~ (combined); 4 x 2 warps
  static constexpr int TM = 64, TN = 32, WRB = 2, WCB = 2, LP = 4, RP = 8;
};
template <>
struct Cfg<true> {  // W task: left Psi~ (combined), right operand A (on the fly); 2 x 4 warps
  static constexpr int TM = 32, TN = 64, WRB = 2, WCB = 2, LP = 8, RP = 4;
};
// Warp w issues on SMSP w % 4.  The warp index runs fastest along the long
// side of the warp grid, so the warps of a tile padded along the short side
// (Y: s % 32, W: l % 32 valid columns / rows) still cover all four SMSPs.
template <bool LPRE>
__device__ __forceinline__ int warp_row(int w) { return LPRE ? w >> 2 : w & 3; }
template <bool LPRE>
__device__ __forceinline__ int warp_col(int w) { return LPRE ? w & 3 : w >> 2; }
template <bool LPRE>
struct Layout {
  using C = Cfg<LPRE>;
  static constexpr int LDX = C::TN + 4;  // j-fast rows: 36 / 68 (4 mod 16)
  static constexpr int L_ELEMS = C::LP * C::TM * LDK;
  static constexpr int R_ELEMS = C::RP * BK * LDX;
};
constexpr int STAGE = (Layout<false>::L_ELEMS + Layout<false>::R_ELEMS) > (Layout<true>::L_ELEMS + Layout<true>::R_ELEMS)
                          ? (Layout<false>::L_ELEMS + Layout<false>::R_ELEMS)
                          : (Layout<true>::L_ELEMS + Layout<true>::R_ELEMS);
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

// Accumulators: acc[i][rb][cb][h] = product m_{i+1} at row
// 8*WRB*warp_row + 8*rb + lane/4, col 8*WCB*warp_col + 8*cb + 2*(lane%4) + h.
template <bool LPRE>
using Acc = double[8][Cfg<LPRE>::WRB][Cfg<LPRE>::WCB][2];

template <bool LPRE>
__device__ __forceinline__ void zero_acc(Acc<LPRE>& acc) {
  using C = Cfg<LPRE>;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int rb = 0; rb < C::WRB; ++rb)
#pragma unroll
      for (int cb = 0; cb < C::WCB; ++cb) acc[i][rb][cb][0] = acc[i][rb][cb][1] = 0.0;
}

// the quaternion planes of one accumulator element (fixed summation order)
__device__ __forceinline__ void combine(const double (&m)[8], double (&c)[4]) {
  const double s56 = m[4] + m[5], d78 = m[6] - m[7];
  c[0] = m[1] - s56 + (m[6] + m[7]);
  c[1] = m[0] - s56 - (m[6] + m[7]);
  c[2] = m[2] + (m[4] - m[5]) + d78;
  c[3] = m[3] + (m[4] - m[5]) - d78;
}

template <bool LPRE>
__device__ __forceinline__ int acc_row(int rb) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  return 8 * Cfg<LPRE>::WRB * warp_row<LPRE>(w) + 8 * rb + (lane >> 2);
}
template <bool LPRE>
__device__ __forceinline__ int acc_col(int cb) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  return 8 * Cfg<LPRE>::WCB * warp_col<LPRE>(w) + 8 * cb + 2 * (lane & 3);
}

// Per-thread copy plan of one tile, fixed for the whole k loop: each thread
// copies the same (row, k) / (k, col) position of LP / RP planes every stage,
// so a stage costs a pointer add per operand and the k bound test (the
// general address arithmetic once per tile, not once per element per stage).
template <bool LPRE>
struct Loader {
  using C = Cfg<LPRE>;
  using Lay = Layout<LPRE>;
  static constexpr int LPER = C::TM * BK, RPER = BK * C::TN;  // elements per plane per stage
  // NT >= PER: thread groups take different planes (SPLIT groups, one
  // position each); NT < PER: every thread takes POS positions of each plane
  static constexpr int LSPLIT = NT >= LPER ? NT / LPER : 1, RSPLIT = NT >= RPER ? NT / RPER : 1;
  static constexpr int LPOS = NT >= LPER ? 1 : LPER / NT, RPOS = NT >= RPER ? 1 : RPER / NT;
  static_assert((NT % LPER == 0 || LPER % NT == 0) && (NT % RPER == 0 || RPER % NT == 0), "copy plan");
  static_assert(C::LP % LSPLIT == 0 && C::RP % RSPLIT == 0, "copy plan");
  static constexpr int LCOPIES = C::LP / LSPLIT, RCOPIES = C::RP / RSPLIT;
  int64_t loff, roff, rstep, ldelta, rdelta;
  int lk, rk, lhi, rhi, ldst, rdst;
  unsigned lrow, rcol;  // validity bit per position
  __device__ __forceinline__ Loader(const Operands& g, int64_t i0, int64_t j0, int64_t kbeg, int tid) {
    const int lidx = tid % LPER, ridx = tid % RPER;
    lhi = tid / LPER;
    rhi = tid / RPER;
    const int lx = lidx / BK, rx = ridx % C::TN;
    lk = lidx % BK;
    rk = ridx / C::TN;
    lrow = rcol = 0;
#pragma unroll
    for (int p = 0; p < LPOS; ++p) lrow |= (i0 + lx + p * (NT / BK) < g.M ? 1u : 0u) << p;
#pragma unroll
    for (int p = 0; p < RPOS; ++p) rcol |= (j0 + rx < g.N ? 1u : 0u) << p;
    loff = (i0 + lx) * g.l_si + kbeg + lk;
    ldelta = (int64_t)(NT / BK) * g.l_si;     // next position: NT / BK rows further
    roff = (kbeg + rk) * g.r_sk + j0 + rx;
    rdelta = (int64_t)(NT / C::TN) * g.r_sk;  // next position: NT / TN k-rows further
    rstep = (int64_t)BK * g.r_sk;
    ldst = (lhi * C::TM + lx) * LDK + lk;
    rdst = (rhi * BK + rk) * Lay::LDX + rx;
  }
  // copy stage starting at k0 (the offsets are then advanced to k0 + BK)
  __device__ __forceinline__ void stage(const Operands& g, double* Ls, double* Rs, int64_t k0, int64_t kend) {
#pragma unroll
    for (int p = 0; p < LPOS; ++p) {
      const bool ok = ((lrow >> p) & 1u) && k0 + lk < kend;
#pragma unroll
      for (int r = 0; r < LCOPIES; ++r) {
        const double* base = LSPLIT == 1 ? g.l[r] : (lhi ? g.l[LSPLIT * r + 1] : g.l[LSPLIT * r]);
        qt::cp_async8(Ls + ldst + (r * LSPLIT * C::TM + p * (NT / BK)) * LDK, ok ? base + loff + p * ldelta : base,
                      ok);
      }
    }
#pragma unroll
    for (int p = 0; p < RPOS; ++p) {
      const bool ok = ((rcol >> p) & 1u) && k0 + rk + p * (NT / C::TN) < kend;
#pragma unroll
      for (int r = 0; r < RCOPIES; ++r) {
        const double* base = RSPLIT == 1 ? g.r[r] : (rhi ? g.r[RSPLIT * r + 1] : g.r[RSPLIT * r]);
        qt::cp_async8(Rs + rdst + (r * RSPLIT * BK + p * (NT / C::TN)) * Lay::LDX,
                      ok ? base + roff + p * rdelta : base, ok);
      }
    }
    loff += BK;
    roff += rstep;
  }
};

// One BK slice for the first NRB row blocks and NCB column blocks of the warp.
template <bool LPRE, int NRB, int NCB>
__device__ __forceinline__ void kstep(const double* Ls, const double* Rs, int wr, int wc, int gid, int tig,
                                      Acc<LPRE>& acc) {
  using C = Cfg<LPRE>;
  constexpr int LDX = Layout<LPRE>::LDX;
#pragma unroll
  for (int kk = 0; kk < BK / 4; ++kk) {
    const int k = 4 * kk + tig;
    if (!LPRE) {
      // left = A: 4 planes per row block, combined in registers
      double a[NRB][4];
#pragma unroll
      for (int rb = 0; rb < NRB; ++rb) {
        const int x = 8 * C::WRB * wr + 8 * rb + gid;
#pragma unroll
        for (int q = 0; q < 4; ++q) a[rb][q] = Ls[(q * C::TM + x) * LDK + k];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double bv[NCB];
#pragma unroll
        for (int cb = 0; cb < NCB; ++cb) bv[cb] = Rs[(i * BK + k) * LDX + 8 * C::WCB * wc + 8 * cb + gid];
#pragma unroll
        for (int rb = 0; rb < NRB; ++rb) {
          const double av = lcomb(i, a[rb]);
#pragma unroll
          for (int cb = 0; cb < NCB; ++cb) qt::dmma(acc[i][rb][cb], av, bv[cb]);
        }
      }
    } else {
      // right = A: 4 planes per column block, combined in registers
      double b[NCB][4];
#pragma unroll
      for (int cb = 0; cb < NCB; ++cb) {
        const int x = 8 * C::WCB * wc + 8 * cb + gid;
#pragma unroll
        for (int q = 0; q < 4; ++q) b[cb][q] = Rs[(q * BK + k) * LDX + x];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double av[NRB];
#pragma unroll
        for (int rb = 0; rb < NRB; ++rb) av[rb] = Ls[(i * C::TM + 8 * C::WRB * wr + 8 * rb + gid) * LDK + k];
#pragma unroll
        for (int cb = 0; cb < NCB; ++cb) {
          const double bv = rcomb(i, b[cb]);
#pragma unroll
          for (int rb = 0; rb < NRB; ++rb) qt::dmma(acc[i][rb][cb], av[rb], bv);
        }
      }
    }
  }
}

// The cp.async ring with mbarrier stage handoff (as qtile.cuh's mma_loop).
template <bool LPRE, int NRB, int NCB>
__device__ __forceinline__ void mma_loop(const Operands& g, double* smem, int64_t i0, int64_t j0, int64_t kbeg,
                                         int64_t kend, Acc<LPRE>& acc, uint64_t* full, uint64_t* empty) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wr = warp_row<LPRE>(w), wc = warp_col<LPRE>(w);
  const int gid = lane >> 2, tig = lane & 3;
  const int nk = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;
  constexpr int LOFF = Layout<LPRE>::L_ELEMS;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      qt::mbar_init(&full[s], NT);
      qt::mbar_init(&empty[s], NT / 32);
    }
  }
  __syncthreads();
  Loader<LPRE> ld(g, i0, j0, kbeg, tid);
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
      kstep<LPRE, (NRB > 0 ? NRB : 1), (NCB > 0 ? NCB : 1)>(Ls, Ls + LOFF, wr, wc, gid, tig, acc);
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
struct TmaOps {
  const CUtensorMap* lm;  // left map
  const CUtensorMap* rm;  // right map
  int lk_off;             // inner coordinate offset of the left map's k (Psi~ panel column)
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

template <bool LPRE>
__device__ __forceinline__ void tma_stage(const TmaOps& t, double* Ls, double* Rs, int64_t i0, int64_t j0, int64_t k0,
                                          uint64_t* bar) {
  using C = Cfg<LPRE>;
  constexpr unsigned BYTES = (unsigned)((Layout<LPRE>::L_ELEMS + Layout<LPRE>::R_ELEMS) * sizeof(double));
  mbar_expect_tx(bar, BYTES);
  tma_load3(Ls, t.lm, (int)(t.lk_off + k0), (int)i0, bar);
  tma_load3(Rs, t.rm, (int)j0, (int)k0, bar);
}

// The ring with a single producer thread (thread 0) issuing each stage PF
// stages ahead; a refill waits for every warp's release of that slot.
template <bool LPRE, int NRB, int NCB>
__device__ __forceinline__ void mma_loop_tma(const TmaOps& t, double* smem, int64_t i0, int64_t j0, int64_t kbeg,
                                             int64_t kend, Acc<LPRE>& acc, uint64_t* full, uint64_t* empty) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wr = warp_row<LPRE>(w), wc = warp_col<LPRE>(w);
  const int gid = lane >> 2, tig = lane & 3;
  const int nk = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;
  constexpr int LOFF = Layout<LPRE>::L_ELEMS;
  constexpr int PF = 2;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      qt::mbar_init(&full[s], 1);
      qt::mbar_init(&empty[s], NT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int p = 0; p < PF && p < nk; ++p)
      tma_stage<LPRE>(t, smem + p * STAGE, smem + p * STAGE + LOFF, i0, j0, kbeg + (int64_t)p * BK, &full[p]);
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % STAGES;
    if (tid == 0) {
      const int nxt = kt + PF;
      if (nxt < nk) {
        const int sn = nxt % STAGES;
        if (nxt >= STAGES) qt::mbar_wait_parity(&empty[sn], (unsigned)((nxt / STAGES - 1) & 1));
        tma_stage<LPRE>(t, smem + sn * STAGE, smem + sn * STAGE + LOFF, i0, j0, kbeg + (int64_t)nxt * BK, &full[sn]);
      }
    }
    __syncwarp();  // warp 0 reconverges before its DMMAs (mma.sync is .aligned)
    qt::mbar_wait_parity(&full[s], (unsigned)((kt / STAGES) & 1));
    const double* Ls = smem + s * STAGE;
    if (NRB > 0 && NCB > 0)
      kstep<LPRE, (NRB > 0 ? NRB : 1), (NCB > 0 ? NCB : 1)>(Ls, Ls + LOFF, wr, wc, gid, tig, acc);
    __syncwarp();
    if (lane == 0) qt::mbar_arrive(&empty[s]);
  }
  // every issued stage was consumed (waited on full) before the loop ended
  __syncthreads();
}

template <bool LPRE>
__device__ __forceinline__ void mma_tile_tma(const TmaOps& t, const Operands& g, double* smem, int64_t i0, int64_t j0,
                                             int64_t kbeg, int64_t kend, Acc<LPRE>& acc) {
  using C = Cfg<LPRE>;
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int w = threadIdx.x >> 5;
  const int64_t r0w = i0 + 8 * C::WRB * warp_row<LPRE>(w), c0w = j0 + 8 * C::WCB * warp_col<LPRE>(w);
  const int nrb = r0w >= g.M ? 0 : (int)min((int64_t)C::WRB, (g.M - r0w + 7) / 8);
  const int ncb = c0w >= g.N ? 0 : (int)min((int64_t)C::WCB, (g.N - c0w + 7) / 8);
  switch (nrb * 4 + ncb) {
    case 2 * 4 + 2: mma_loop_tma<LPRE, 2, 2>(t, smem, i0, j0, kbeg, kend, acc, full, empty); break;
    case 2 * 4 + 1: mma_loop_tma<LPRE, 2, 1>(t, smem, i0, j0, kbeg, kend, acc, full, empty); break;
    case 1 * 4 + 2: mma_loop_tma<LPRE, 1, 2>(t, smem, i0, j0, kbeg, kend, acc, full, empty); break;
    case 1 * 4 + 1: mma_loop_tma<LPRE, 1, 1>(t, smem, i0, j0, kbeg, kend, acc, full, empty); break;
    default: mma_loop_tma<LPRE, 0, 0>(t, smem, i0, j0, kbeg, kend, acc, full, empty); break;
  }
}

// acc (8 products) over k in [kbeg, kend) for the tile at (i0, j0).  Warp
// blocks past M or N issue no DMMA (the loop instance is chosen per warp).
template <bool LPRE>
__device__ __forceinline__ void mma_tile(const Operands& g, double* smem, int64_t i0, int64_t j0, int64_t kbeg,
                                         int64_t kend, Acc<LPRE>& acc) {
  using C = Cfg<LPRE>;
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int w = threadIdx.x >> 5;
  const int64_t r0w = i0 + 8 * C::WRB * warp_row<LPRE>(w), c0w = j0 + 8 * C::WCB * warp_col<LPRE>(w);
  const int nrb = r0w >= g.M ? 0 : (int)min((int64_t)C::WRB, (g.M - r0w + 7) / 8);
  const int ncb = c0w >= g.N ? 0 : (int)min((int64_t)C::WCB, (g.N - c0w + 7) / 8);
  switch (nrb * 4 + ncb) {
    case 2 * 4 + 2: mma_loop<LPRE, 2, 2>(g, smem, i0, j0, kbeg, kend, acc, full, empty); break;
    case 2 * 4 + 1: mma_loop<LPRE, 2, 1>(g, smem, i0, j0, kbeg, kend, acc, full, empty); break;
    case 1 * 4 + 2: mma_loop<LPRE, 1, 2>(g, smem, i0, j0, kbeg, kend, acc, full, empty); break;
    case 1 * 4 + 1: mma_loop<LPRE, 1, 1>(g, smem, i0, j0, kbeg, kend, acc, full, empty); break;
    default: mma_loop<LPRE, 0, 0>(g, smem, i0, j0, kbeg, kend, acc, full, empty); break;
  }
}

}  // namespace qt8
}  // namespace qlra_dev
