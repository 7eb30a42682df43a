// qtile.cuh -- the quaternion tile engine on the FP64 tensor pipe (DMMA).
//
// One CTA (512 threads, 16 warps) computes a 64x64 quaternion tile
//   acc += op(A)[i0:i0+64, kbeg:kend] * op(B)[kbeg:kend, j0:j0+64]
// with `mma.sync.aligned.m8n8k4.row.col.f64` (SASS DMMA.8x8x4; tcgen05 has
// no f64 kind).  A quaternion MAC is 16 real products
// (proj/include/qlra/quaternion.hpp:33-38); output plane p is
// sum_q sign(p,q) * A_q * B_perm(p,q).  Each warp keeps + and - copies of the
// B fragments it needs, so every one of the 16 products is a plain DMMA and
// conjugation of either operand (op = adjoint) only changes which copy is
// selected -- no extra instructions.
//
// Warp layout: 4 (rows) x 4 (cols) warps, each owning a 16x16 quaternion
// sub-tile = 2x2 blocks of 8x8 per plane: 32 FP64 accumulators per thread
// (16 warps per SM keep the DMMA pipe fed).
// Operands are staged by cp.async into a 4-stage shared-memory ring in the
// layout of their contiguous global dimension.  Row pitches are 4 mod 16
// doubles (k-fast rows padded to 12, i/j-fast rows to 68): a half-warp's
// fragment read covers 4 rows x 4 consecutive elements, which then land in
// 16 distinct 8-byte bank pairs -- every LDS.64 is 2 wavefronts, the minimum
// (measured: C2 sketch 16.4 -> 16.1 ms against pitches 10 / 72).
#pragma once

#include "common.cuh"

namespace qlra_dev {
namespace qt {

constexpr int BM = 64, BN = 64, BK = 8, NT = 512, STAGES = 4;
constexpr int WRB = 2, WCB = 2;  // 8x8 blocks per warp (warp tile 16x16, 4x4 warps)
constexpr int LDK = BK + 4;    // k-fast rows: [x][k]
constexpr int LDX = BM + 4;    // i/j-fast rows: [k][x]
constexpr int OP_STAGE = 4 * BM * LDK > 4 * BK * LDX ? 4 * BM * LDK : 4 * BK * LDX;  // doubles
constexpr int STAGE = 2 * OP_STAGE;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE * sizeof(double);

// op(A)(i, k) = a[q][i * a_si + k * a_sk];  op(B)(k, j) = b[q][k * b_sk + j * b_sj]
struct Operands {
  const double* a[4];
  const double* b[4];
  int64_t a_si, a_sk, b_sk, b_sj;
  int64_t M, N;
  // Hermitian product (C = A^* A): warp tiles strictly below the diagonal
  // issue no DMMA (the caller mirrors the upper triangle)
  int herm = 0;
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// AK: op(A) is k-fast in memory (a_sk == 1), smem [q][i][k]; else [q][k][i].
// BJ: op(B) is j-fast (b_sj == 1), smem [q][k][j]; else [q][j][k].
template <bool AK, bool BJ>
__device__ __forceinline__ void load_stage(const Operands& g, double* As, double* Bs, int64_t i0,
                                           int64_t j0, int64_t k0, int64_t kend, int tid) {
  constexpr int PER = BM * BK;  // elements per plane per stage
#pragma unroll
  for (int r = 0; r < 4 * PER / NT; ++r) {
    const int e = tid + NT * r;  // 4 planes x 64 x BK
    const int q = e / PER, idx = e % PER;
    int x, k;
    if (AK) { x = idx / BK; k = idx % BK; } else { x = idx % BM; k = idx / BM; }
    const int64_t gi = i0 + x, gk = k0 + k;
    const bool ok = gi < g.M && gk < kend;
    const double* src = ok ? g.a[q] + gi * g.a_si + gk * g.a_sk : g.a[q];
    double* dst = AK ? As + (q * BM + x) * LDK + k : As + (q * BK + k) * LDX + x;
    cp_async8(dst, src, ok);
  }
#pragma unroll
  for (int r = 0; r < 4 * PER / NT; ++r) {
    const int e = tid + NT * r;
    const int q = e / PER, idx = e % PER;
    int x, k;
    if (BJ) { x = idx % BN; k = idx / BN; } else { x = idx / BK; k = idx % BK; }
    const int64_t gj = j0 + x, gk = k0 + k;
    const bool ok = gj < g.N && gk < kend;
    const double* src = ok ? g.b[q] + gk * g.b_sk + gj * g.b_sj : g.b[q];
    double* dst = BJ ? Bs + (q * BK + k) * LDX + x : Bs + (q * BN + x) * LDK + k;
    cp_async8(dst, src, ok);
  }
}

// Accumulator fragment: acc[rb][cb][p][0..1] = C_p[row][col..col+1] with
// row = i0 + 16*wr + 8*rb + lane/4, col = j0 + 16*wc + 8*cb + 2*(lane%4).
using Acc = double[WRB][WCB][4][2];

__device__ __forceinline__ void zero_acc(Acc& acc) {
#pragma unroll
  for (int rb = 0; rb < WRB; ++rb)
#pragma unroll
    for (int cb = 0; cb < WCB; ++cb)
#pragma unroll
      for (int p = 0; p < 4; ++p) acc[rb][cb][p][0] = acc[rb][cb][p][1] = 0.0;
}

// Warp w owns the 16x16 sub-tile (warp_row(w), warp_col(w)).  Warps issue on
// SMSP w % 4 = (row + col) % 4: this anti-diagonal assignment gives every
// SMSP one warp of each row band AND each column band, so the 8x8 blocks
// skipped in tiles padded along either M or N take work off all four tensor
// pipes evenly (with wc = w % 4, a tile padded along N left one SMSP idle and
// the CTA waited on the other three), and it also spreads the upper triangle
// of a Hermitian product's diagonal tile (4 x 4 warp tiles: 3/2/3/2 per SMSP;
// the (col - row) % 4 assignment put all four diagonal warp tiles on SMSP 0).
__device__ __forceinline__ int warp_row(int w) { return w >> 2; }
__device__ __forceinline__ int warp_col(int w) { return ((w & 3) - (w >> 2)) & 3; }

__device__ __forceinline__ int acc_row(int rb) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  return 16 * warp_row(w) + 8 * rb + (lane >> 2);
}
__device__ __forceinline__ int acc_col(int cb) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  return 16 * warp_col(w) + 8 * cb + 2 * (lane & 3);
}

// Hamilton table in (term q, output plane p) -> (B plane, sign):
//   q=0 (a_w): +bw +bx +by +bz      q=1 (a_x): -bx +bw -bz +by
//   q=2 (a_y): -by +bz +bw -bx      q=3 (a_z): -bz -by +bx +bw
__device__ __forceinline__ constexpr int hplane(int q, int p) {
  return q == 0 ? p : q == 1 ? (p == 0 ? 1 : p == 1 ? 0 : p == 2 ? 3 : 2)
                    : q == 2 ? (p == 0 ? 2 : p == 1 ? 3 : p == 2 ? 0 : 1)
                             : (p == 0 ? 3 : p == 1 ? 2 : p == 2 ? 1 : 0);
}
__device__ __forceinline__ constexpr int hsign(int q, int p) {
  return q == 0 ? 1 : q == 1 ? (p == 0 || p == 2 ? -1 : 1)
                    : q == 2 ? (p == 0 || p == 3 ? -1 : 1)
                             : (p == 0 || p == 1 ? -1 : 1);
}

// One BK slice of the tile product from shared memory for the first NRB
// row blocks and NCB column blocks of the warp (the valid ones are always a
// prefix).  Instantiated per (NRB, NCB) so the DMMA stream carries no
// predicates -- predicated-off DMMAs still occupy the tensor pipe.
template <bool CA, bool CB, bool AK, bool BJ, int NRB, int NCB>
__device__ __forceinline__ void kstep(const double* As, const double* Bs, int wr, int wc, int gid, int tig,
                                      Acc& acc) {
#pragma unroll
  for (int kk = 0; kk < BK / 4; ++kk) {
    const int k = 4 * kk + tig;
    double a[NRB][4];  // [rb][q]
#pragma unroll
    for (int rb = 0; rb < NRB; ++rb) {
      const int x = 16 * wr + 8 * rb + gid;
#pragma unroll
      for (int q = 0; q < 4; ++q) a[rb][q] = AK ? As[(q * BM + x) * LDK + k] : As[(q * BK + k) * LDX + x];
    }
    double bp[NCB][4], bn[NCB][4];  // + and - copies, [cb][plane]
#pragma unroll
    for (int cb = 0; cb < NCB; ++cb) {
      const int x = 16 * wc + 8 * cb + gid;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        bp[cb][q] = BJ ? Bs[(q * BK + k) * LDX + x] : Bs[(q * BN + x) * LDK + k];
        bn[cb][q] = -bp[cb][q];
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int rb = 0; rb < NRB; ++rb)
#pragma unroll
        for (int cb = 0; cb < NCB; ++cb)
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const int bq = hplane(q, p);
            // conj(A): a_x,y,z negated -> flip terms q >= 1;
            // conj(B): b_x,y,z negated -> flip when the B plane is not w.
            int sg = hsign(q, p);
            if (CA && q > 0) sg = -sg;
            if (CB && bq > 0) sg = -sg;
            dmma(acc[rb][cb][p], a[rb][q], sg > 0 ? bp[cb][bq] : bn[cb][bq]);
          }
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "QT_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra QT_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// arrive on `bar` once all of this thread's earlier cp.async copies landed
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// The cp.async ring and the k loop for one (NRB, NCB) instance.  Stage
// handoff by mbarriers instead of a CTA barrier per stage: each thread's
// copies of stage k arrive on full[k % S] when they land; each warp arrives
// on empty[k % S] when it has read stage k.  Prefetch distance 1 over S = 4
// slots: refilling a slot waits only for the consumption three stages back,
// so warps drift up to three stages apart instead of meeting every stage.
template <bool CA, bool CB, int NRB, int NCB>
__device__ __forceinline__ void mma_loop(const Operands& g, double* smem, int64_t i0, int64_t j0,
                                         int64_t kbeg, int64_t kend, Acc& acc, uint64_t* full, uint64_t* empty) {
  constexpr bool AK = !CA, BJ = !CB;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wr = warp_row(w), wc = warp_col(w);
  const int gid = lane >> 2, tig = lane & 3;
  const int nk = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], NT);
      mbar_init(&empty[s], NT / 32);
    }
  }
  __syncthreads();
  // prefetch distance 1: a refill waits only for the consumption STAGES - 1
  // stages back (measured: distance 2 is slower -- the waits are on slow
  // warps, not on data)
  constexpr int PF = 1;
#pragma unroll
  for (int p = 0; p < PF; ++p)
    if (p < nk) {
      load_stage<AK, BJ>(g, smem + p * STAGE, smem + p * STAGE + OP_STAGE, i0, j0, kbeg + (int64_t)p * BK, kend,
                         tid);
      cp_async_arrive(&full[p]);
    }
  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % STAGES;
    const int nxt = kt + PF;
    if (nxt < nk) {
      const int sn = nxt % STAGES;
      if (nxt >= STAGES) mbar_wait_parity(&empty[sn], (unsigned)((nxt / STAGES - 1) & 1));
      load_stage<AK, BJ>(g, smem + sn * STAGE, smem + sn * STAGE + OP_STAGE, i0, j0,
                         kbeg + (int64_t)nxt * BK, kend, tid);
      cp_async_arrive(&full[sn]);
    }
    mbar_wait_parity(&full[s], (unsigned)((kt / STAGES) & 1));
    const double* As = smem + s * STAGE;
    const double* Bs = As + OP_STAGE;
    if (NRB > 0 && NCB > 0) kstep<CA, CB, AK, BJ, (NRB > 0 ? NRB : 1), (NCB > 0 ? NCB : 1)>(As, Bs, wr, wc, gid, tig, acc);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  cp_async_wait<0>();
  __syncthreads();  // the ring (and the barriers) may be reused by the caller
}

// acc += op(A) op(B) over k in [kbeg, kend).  CA/CB: op = adjoint, which
// requires the i-fast / k-fast layouts (AK = !CA, BJ = !CB).  The caller must
// __syncthreads() between successive calls that reuse `smem`.  8x8 blocks
// entirely past M or N (l, s not multiples of 64) issue no DMMA: each warp
// runs the loop instance for its count of valid row/column blocks (a warp-
// uniform choice made once), so edge tiles finish early and free the SM.
template <bool CA, bool CB>
__device__ __forceinline__ void mma_tile(const Operands& g, double* smem, int64_t i0, int64_t j0,
                                         int64_t kbeg, int64_t kend, Acc& acc) {
  // stage barriers shared by every warp of the CTA, whichever loop instance
  // it runs
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int w = threadIdx.x >> 5;
  const int64_t r0w = i0 + 16 * warp_row(w), c0w = j0 + 16 * warp_col(w);
  const int nrb = r0w >= g.M || (g.herm && r0w >= c0w + 16) ? 0 : r0w + 8 >= g.M ? 1 : 2;
  const int ncb = c0w >= g.N ? 0 : c0w + 8 >= g.N ? 1 : 2;
  switch (nrb * 4 + ncb) {
    case 2 * 4 + 2: mma_loop<CA, CB, 2, 2>(g, smem, i0, j0, kbeg, kend, acc, full, empty); break;
    case 2 * 4 + 1: mma_loop<CA, CB, 2, 1>(g, smem, i0, j0, kbeg, kend, acc, full, empty); break;
    case 1 * 4 + 2: mma_loop<CA, CB, 1, 2>(g, smem, i0, j0, kbeg, kend, acc, full, empty); break;
    case 1 * 4 + 1: mma_loop<CA, CB, 1, 1>(g, smem, i0, j0, kbeg, kend, acc, full, empty); break;
    default: mma_loop<CA, CB, 0, 0>(g, smem, i0, j0, kbeg, kend, acc, full, empty); break;  // loads + barriers only
    // (nrb = 0 with ncb > 0 -- a Hermitian product's lower warp tiles -- lands here too)
  }
}

}  // namespace qt
}  // namespace qlra_dev
