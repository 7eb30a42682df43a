// i8gemm.cu -- the int8 engine's batched residue GEMMs on tcgen05 (sm_100a).
//
// The hot contraction of the int8 sketch engine (ozaki.cu): for every batch
// b = (plane combination, modulus) an exact int8 x int8 -> int32 product,
//   mode 0 (Y side):   C[b][m][n]  = sum_k A[b][m][k] B[b][n][k]      (A, B K-major)
//   mode 1 (W^* side): C[b][n][m] (+)= sum_k A[b][k][m] B[b][n][k]    (A MN-major, B K-major)
// i.e. the residue images of Y = A Omega and W^* = A^* Psi^* (the reference's
// two ordered products of sketch_update_rows, proj/src/sketching.cpp:125-139)
// straight from the row-major residue panel k_res_a writes: mode 0 contracts
// over its columns, mode 1 over its rows, so the panel is never transposed.
//
// One persistent CTA per SM, 256 threads in four roles:
//   warp 0 (one lane)  TMA producer: cp.async.bulk.tensor (128B-swizzled
//                      boxes of 128 bytes x 128 / 256 rows) into a 4-slot
//                      shared-memory ring (48 KB per slot);
//   warp 1 (one lane)  MMA issuer: tcgen05.mma.cta_group::1.kind::i8,
//                      128 x N x 32 per instruction (N <= 256, the tile's
//                      valid columns), operands by shared-memory descriptors,
//                      int32 accumulators in TMEM (two 256-column stages);
//                      tcgen05.commit hands ring slots back to the producer
//                      and finished accumulators to the epilogue;
//   warp 2             allocates / frees the 512 TMEM columns;
//   warps 4-7          epilogue: tcgen05.ld (32 lanes x 32 columns per
//                      instruction) into per-warp double-buffered 4 KB staging
//                      blocks, written out by TMA: cp.async.bulk.tensor stores,
//                      or cp.reduce.async.bulk.tensor .add when beta = 1 (W^*'s
//                      products accumulate over panels in L2, no loads in the
//                      SM); TMA clips the ragged edges.  Overlapped with the
//                      next tile's MMAs through the second TMEM stage.
// Tiles are ordered (batch, m, n) with n fastest so that the CTAs running
// together share an A tile row in L2 and the batch's B operand stays
// resident; the producers of a row's n-tile siblings meet at every tile start
// (sibling_rendezvous) so that they stay within the L2's residency of each
// other.  The CTA-pair form below (tcgen05.mma.cta_group::2) is the one the
// engine uses; this 1-CTA form serves M <= 128 and QLRA_I8_CTAS=1.
//
// Integer arithmetic: the result is exact and independent of the tiling, so
// it is bitwise equal to cuBLASLt's on the same residues (tests/test_gpu_i8gemm.py).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "i8gemm.cuh"
#include "kernels.cuh"

namespace qlra_dev {

namespace {

constexpr int BM = 128;      // accumulator rows (TMEM lanes)
constexpr int BN = 256;      // accumulator columns per TMEM stage
constexpr int BK = 128;      // bytes of K per ring slot (one 128B swizzle row)
constexpr int UK = 32;       // K per tcgen05.mma kind::i8
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK;  // 16 KB
constexpr int B_BYTES = BN * BK;  // 32 KB
constexpr int SLOT = A_BYTES + B_BYTES;
constexpr int NTHREADS = 256;
constexpr int TMEM_COLS = 512;
constexpr int EPI_COLS = 32;                  // accumulator columns per staged chunk
constexpr int EPI_WARP = 32 * EPI_COLS * 4;   // one warp's staged block: 4 KB
constexpr int EPI_BYTES = 4 * EPI_WARP;       // 16 KB per buffer set
constexpr size_t SMEM_BYTES = 1024 /* alignment slack */ + (size_t)STAGES * SLOT + 2 * EPI_BYTES + 256 /* barriers */;

struct Args {
  int64_t M, N, K;
  int batch, beta, mode;
  // tile-row rendezvous of the n-tile siblings (0: off): sync[row] counts the
  // producers that reached the row, sib of them per row
  unsigned* sync;
  unsigned sib;
  int tiles_m, tiles_n, num_k;
  int64_t total_tiles;
};

__device__ __forceinline__ uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "I8_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra I8_WAIT_%=;\n}" ::"r"(s32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          s32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(s32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
// arrives on `b` once every tcgen05.mma issued so far by this thread is done
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(b)) : "memory");
}
__device__ __forceinline__ void tc_mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor (tcgen05, version 1), 128B swizzle, 8-row
// groups 1024 bytes apart (SBO).  K-major: rows of 128 bytes of K; MN-major:
// rows of 128 bytes of M, one row per k (8 k per group).  LBO is unused by
// both layouts at these tile widths (one swizzle row per line).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  return (uint64_t)((addr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// Instruction descriptor: D = S32 (2 at bit 4), A / B = signed 8 bit (1 at
// bits 7 / 10), A MN-major flag at bit 15, N >> 3 at bit 17, M >> 4 at bit 24.
__device__ __forceinline__ uint32_t instr_desc(int n, int a_mn_major) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn_major << 15) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}

// The n-tile siblings of a tile row (2 or 4 CTAs, or CTA pairs, running the
// row together) read the same A k-blocks and share them through L2, which
// holds ~45 us of the operand stream.  Nothing else ties them together: a
// sibling that falls behind by more than that re-reads A from DRAM (measured:
// 2x the DRAM reads on C3's W* product and on long-K tiles), which slows all
// of them and it never catches up.  So the siblings' producers meet at every
// tile start on a counter in global memory (all CTAs of the persistent grid
// are resident, so the wait is bounded by one tile).
__device__ __forceinline__ void sibling_rendezvous(unsigned* cnt, unsigned sib) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
  unsigned v;
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
    if (v < sib) __nanosleep(64);
  } while (v < sib);
}

__global__ void __launch_bounds__(NTHREADS, 1)
    i8gemm_tc05_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                       const __grid_constant__ CUtensorMap map_c, const Args g) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* ring = smem;
  uint8_t* epi = smem + (size_t)STAGES * SLOT;  // 2 x 16 KB, 1024-aligned (128B-swizzled in mode 0)
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + 2 * EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // accumulator stage ready for the epilogue
  uint64_t* tempty = tfull + 2;       // accumulator stage drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      bar_init(&tfull[s], 1);
      bar_init(&tempty[s], 4);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int64_t per_batch = (int64_t)g.tiles_m * g.tiles_n;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer ----
      unsigned it = 0;
      for (int64_t t = blockIdx.x; t < g.total_tiles; t += gridDim.x) {
        const int b = (int)(t / per_batch);
        const int r = (int)(t - (int64_t)b * per_batch);
        const int m0 = (r / g.tiles_n) * BM, n0 = (r % g.tiles_n) * BN;
        if (g.sib) sibling_rendezvous(g.sync + t / g.tiles_n, g.sib);
        for (int kb = 0; kb < g.num_k; ++kb, ++it) {
          const int s = it % STAGES;
          bar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          bar_expect_tx(&full[s], SLOT);
          uint8_t* as = ring + (size_t)s * SLOT;
          if (g.mode == 0)
            tma3(as, &map_a, kb * BK, m0, b, &full[s]);
          else
            tma3(as, &map_a, m0, kb * BK, b, &full[s]);
          tma3(as + A_BYTES, &map_b, kb * BK, n0, b, &full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer ----
      unsigned it = 0, lt = 0;
      for (int64_t t = blockIdx.x; t < g.total_tiles; t += gridDim.x, ++lt) {
        const int r = (int)(t % per_batch);
        const int n0 = (r % g.tiles_n) * BN;
        const int nt = g.N - n0 < BN ? (int)(g.N - n0) : BN;  // multiple of 16
        const uint32_t idesc = instr_desc(nt, g.mode);
        const unsigned as = lt & 1;
        bar_wait(&tempty[as], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + as * BN;
        for (int kb = 0; kb < g.num_k; ++kb, ++it) {
          const int s = it % STAGES;
          bar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint32_t a0 = s32(ring + (size_t)s * SLOT), b0 = a0 + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / UK; ++k) {
            // K-major: 32 bytes along the swizzled row; MN-major: 32 rows of 128 bytes
            const uint64_t ad = smem_desc(a0 + (g.mode == 0 ? k * UK : k * UK * BM));
            const uint64_t bd = smem_desc(b0 + k * UK);
            tc_mma_i8(d, ad, bd, idesc, (kb | k) != 0);
          }
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[as]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ---- epilogue: TMEM lanes 32 q .. 32 q + 31 belong to warp q = warp % 4; each
    // warp stages and stores its own 32 x 32 blocks (4 KB, double-buffered), so the
    // four warps never meet ----
    const int q = warp & 3;
    uint8_t* wbuf = epi + q * (2 * EPI_WARP);
    unsigned lt = 0, ch = 0;
    for (int64_t t = blockIdx.x; t < g.total_tiles; t += gridDim.x, ++lt) {
      const int b = (int)(t / per_batch);
      const int r = (int)(t - (int64_t)b * per_batch);
      const int m0 = (r / g.tiles_n) * BM + q * 32, n0 = (r % g.tiles_n) * BN;
      const int nt = g.N - n0 < BN ? (int)(g.N - n0) : BN;
      const unsigned as = lt & 1;
      bar_wait(&tfull[as], (lt >> 1) & 1);
      tc_fence_after();
      for (int c0 = 0; c0 < nt; c0 += EPI_COLS, ++ch) {
        uint32_t v[32];
        tc_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + as * BN + c0, v);
        if (c0 + EPI_COLS >= nt) {
          // the tile's last TMEM read: hand the accumulator stage back
          tc_fence_before();
          __syncwarp();
          if (lane == 0) bar_arrive(&tempty[as]);
        }
        if (m0 >= g.M) continue;  // rows past M: nothing to store (warp-uniform)
        uint8_t* sb = wbuf + (ch & 1) * EPI_WARP;
        // the store issued two chunks ago has finished reading this buffer
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
        if (g.mode == 0) {
          // [32 m][32 n], 128-byte rows, 16-byte chunks swizzled by the row (TMA SWIZZLE_128B)
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<uint4*>(sb + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        } else {
          // [32 n][32 m]: the lanes are contiguous in m
#pragma unroll
          for (int j = 0; j < 32; ++j) reinterpret_cast<uint32_t*>(sb)[j * 32 + lane] = v[j];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          const int x = g.mode == 0 ? n0 + c0 : m0, y = g.mode == 0 ? m0 : n0 + c0;
          if (g.beta)
            asm volatile(
                "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                    &map_c),
                "r"(x), "r"(y), "r"(b), "r"(s32(sb))
                : "memory");
          else
            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                             &map_c),
                         "r"(x), "r"(y), "r"(b), "r"(s32(sb))
                         : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS) : "memory");
  }
}

// ---------------------------------------------------------------------------
// The same product on CTA pairs: tcgen05.mma.cta_group::2, one 256 x N tile per
// pair of SMs (a 2-CTA cluster).  Each CTA stages its own 128 rows of A and
// its own half of the tile's B rows (32 KB per ring slot, 6 slots); the
// leader CTA's elected thread issues the MMAs for both SMs, whose tensor
// cores read the two B halves from both CTAs' shared memory; each CTA's TMEM
// holds its 128 accumulator rows and its own epilogue warps drain them.
// Against the 1-CTA kernel: a third less L2 -> SM operand traffic and a
// third fewer shared-memory operand reads per MMA -- energy, which is what
// the power-capped clock of a long int8 run is made of.
//   full[s]    leader only, 2 arrivals (each CTA's producer: expect_tx of its
//              own 32 KB; both CTAs' TMA loads complete_tx on the leader's);
//   empty[s]   per CTA, tcgen05.commit multicast to both;
//   tfull[a]   per CTA, commit multicast; tempty[a] leader only, 8 arrivals
//              (the epilogue warps of both CTAs).
constexpr int STAGES2 = 6;
constexpr int B2_BYTES = (BN / 2) * BK;  // 16 KB: this CTA's half of the B rows
constexpr int SLOT2 = A_BYTES + B2_BYTES;
static_assert(STAGES2 * SLOT2 == STAGES * SLOT, "both kernels use the same ring bytes");

__device__ __forceinline__ uint32_t leader_addr(uint32_t a) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ void tma3_2sm(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(s32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_commit2(uint64_t* b) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(s32(b)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tc_mma_i8_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
    i8gemm_tc05_2sm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                           const __grid_constant__ CUtensorMap map_c, const Args g) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* ring = smem;
  uint8_t* epi = smem + (size_t)STAGES2 * SLOT2;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + 2 * EPI_BYTES);
  uint64_t* empty = full + STAGES2;
  uint64_t* tfull = empty + STAGES2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      bar_init(&full[s], 2);
      bar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      bar_init(&tfull[s], 1);
      bar_init(&tempty[s], 8);  // the epilogue warps of both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's barriers are initialised and its TMEM allocated
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int64_t per_batch = (int64_t)g.tiles_m * g.tiles_n;
  const int64_t pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer (both CTAs): own A rows, own half of the B rows ----
      unsigned it = 0;
      for (int64_t t = pair; t < g.total_tiles; t += npairs) {
        const int b = (int)(t / per_batch);
        const int r = (int)(t - (int64_t)b * per_batch);
        const int m0 = (r / g.tiles_n) * (2 * BM) + (int)rank * BM, n0 = (r % g.tiles_n) * BN;
        const int nt = g.N - n0 < BN ? (int)(g.N - n0) : BN;
        const int nb0 = n0 + (int)rank * (nt >> 1);  // the MMA reads nt / 2 B rows from each CTA
        if (g.sib) sibling_rendezvous(g.sync + t / g.tiles_n, g.sib);
        for (int kb = 0; kb < g.num_k; ++kb, ++it) {
          const int s = it % STAGES2;
          bar_wait(&empty[s], ((it / STAGES2) & 1) ^ 1);
          const uint32_t fb = leader_addr(s32(&full[s]));
          asm volatile("mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;" ::"r"(fb), "r"(SLOT2) : "memory");
          uint8_t* as = ring + (size_t)s * SLOT2;
          if (g.mode == 0)
            tma3_2sm(as, &map_a, kb * BK, m0, b, fb);
          else
            tma3_2sm(as, &map_a, m0, kb * BK, b, fb);
          tma3_2sm(as + A_BYTES, &map_b, kb * BK, nb0, b, fb);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---- MMA issuer (leader CTA) ----
      unsigned it = 0, lt = 0;
      for (int64_t t = pair; t < g.total_tiles; t += npairs, ++lt) {
        const int r = (int)(t % per_batch);
        const int n0 = (r % g.tiles_n) * BN;
        const int nt = g.N - n0 < BN ? (int)(g.N - n0) : BN;  // multiple of 16
        // M = 256: M >> 4 = 16 at bit 24
        const uint32_t idesc = (instr_desc(nt, g.mode) & ~(0x1Fu << 24)) | (16u << 24);
        const unsigned as = lt & 1;
        bar_wait(&tempty[as], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + as * BN;
        for (int kb = 0; kb < g.num_k; ++kb, ++it) {
          const int s = it % STAGES2;
          bar_wait(&full[s], (it / STAGES2) & 1);
          tc_fence_after();
          const uint32_t a0 = s32(ring + (size_t)s * SLOT2), b0 = a0 + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / UK; ++k) {
            const uint64_t ad = smem_desc(a0 + (g.mode == 0 ? k * UK : k * UK * BM));
            const uint64_t bd = smem_desc(b0 + k * UK);
            tc_mma_i8_2sm(d, ad, bd, idesc, (kb | k) != 0);
          }
          tc_commit2(&empty[s]);
        }
        tc_commit2(&tfull[as]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ---- epilogue (both CTAs): this CTA's 128 accumulator rows ----
    const int q = warp & 3;
    uint8_t* wbuf = epi + q * (2 * EPI_WARP);
    unsigned lt = 0, ch = 0;
    for (int64_t t = pair; t < g.total_tiles; t += npairs, ++lt) {
      const int b = (int)(t / per_batch);
      const int r = (int)(t - (int64_t)b * per_batch);
      const int m0 = (r / g.tiles_n) * (2 * BM) + (int)rank * BM + q * 32, n0 = (r % g.tiles_n) * BN;
      const int nt = g.N - n0 < BN ? (int)(g.N - n0) : BN;
      const unsigned as = lt & 1;
      bar_wait(&tfull[as], (lt >> 1) & 1);
      tc_fence_after();
      for (int c0 = 0; c0 < nt; c0 += EPI_COLS, ++ch) {
        uint32_t v[32];
        tc_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + as * BN + c0, v);
        if (c0 + EPI_COLS >= nt) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            const uint32_t tb = leader_addr(s32(&tempty[as]));
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tb) : "memory");
          }
        }
        if (m0 >= g.M) continue;
        uint8_t* sb = wbuf + (ch & 1) * EPI_WARP;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
        if (g.mode == 0) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<uint4*>(sb + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) reinterpret_cast<uint32_t*>(sb)[j * 32 + lane] = v[j];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          const int x = g.mode == 0 ? n0 + c0 : m0, y = g.mode == 0 ? m0 : n0 + c0;
          if (g.beta)
            asm volatile(
                "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                    &map_c),
                "r"(x), "r"(y), "r"(b), "r"(s32(sb))
                : "memory");
          else
            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                             &map_c),
                         "r"(x), "r"(y), "r"(b), "r"(s32(sb))
                         : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // neither CTA leaves while the other may still signal its barriers or read its operands
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS) : "memory");
  }
}

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

// 3D map over int8 (inner bytes, rows, batch), boxes of 128 bytes x box_rows,
// 128B swizzle; out-of-range bytes read as zero
void make_map(CUtensorMap* m, const int8_t* base, int64_t inner, int64_t rows, int64_t batch, int64_t ld,
              int64_t stride, int box_rows) {
  auto fn = encode_fn();
  if (!fn) fail(QLRA_ERR_CUDA, "i8gemm: cuTensorMapEncodeTiled is not available");
  const cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)ld, (cuuint64_t)stride};
  const cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  static const CUtensorMapL2promotion promo = [] {
    const char* e = std::getenv("QLRA_I8_L2PROMO");  // 0 none, 1 64B, 2 128B, 3 256B
    const int v = e ? std::atoi(e) : 3;
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
           : v == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }();
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(QLRA_ERR_CUDA, "i8gemm: cuTensorMapEncodeTiled failed (operand layout)");
}
// the int32 output (inner, rows, batch): boxes of one staged chunk, stores
// clipped at the extents; boxes of one warp's staged block (32 x 32 int32)
void make_map_c(CUtensorMap* m, int32_t* base, int64_t inner, int64_t rows, int64_t batch, int64_t ld, int64_t stride,
                int box_inner, int box_rows, bool swizzle) {
  auto fn = encode_fn();
  if (!fn) fail(QLRA_ERR_CUDA, "i8gemm: cuTensorMapEncodeTiled is not available");
  const cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)stride * 4};
  const cuuint32_t box[3] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_INT32, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(QLRA_ERR_CUDA, "i8gemm: cuTensorMapEncodeTiled failed (output layout)");
}

}  // namespace

const char* i8gemm_kernel_name() {
  return "i8gemm_tc05_2sm_kernel (tcgen05.mma.cta_group::2 kind::i8 256xNx32 on CTA pairs, TMA 128B-swizzled 6-slot "
         "ring, 2 TMEM accumulator stages, TMA store / reduce-add epilogue, persistent; i8gemm_tc05_kernel: the "
         "1-CTA 128xNx32 form for M <= 128)";
}

void i8gemm_batched(Ctx& c, int mode, int64_t M, int64_t N, int64_t K, const int8_t* A, int64_t lda, int64_t stride_a,
                    const int8_t* B, int64_t ldb, int64_t stride_b, int32_t* C, int64_t ldc, int64_t stride_c,
                    int batch, int beta, cudaStream_t stream, int ctas) {
  if (M <= 0 || N <= 0 || batch <= 0) return;
  if (mode != 0 && mode != 1) fail(QLRA_ERR_PARAMETER, "i8gemm: mode must be 0 or 1");
  if (N % 16 || lda % 16 || ldb % 16 || stride_a % 16 || stride_b % 16 || ldc % 4 || stride_c % 4 ||
      (reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(C)) % 16)
    fail(QLRA_ERR_PARAMETER, "i8gemm: N, leading dimensions and batch strides must be multiples of 16 (ldc of 4)");
  // TMA stores move whole 16-byte units: the contiguous extent of C must be one
  if (mode == 1 && M % 4) fail(QLRA_ERR_PARAMETER, "i8gemm: mode 1 needs M to be a multiple of 4");
  if (K <= 0) {
    if (!beta)
      for (int b = 0; b < batch; ++b)
        QLRA_CUDA(cudaMemset2DAsync(C + (int64_t)b * stride_c, (size_t)ldc * 4, 0,
                                    (size_t)(mode == 0 ? N : M) * 4, (size_t)(mode == 0 ? M : N), stream));
    return;
  }
  // per device (one process may drive several): the kernels' shared-memory
  // opt-in and the SM count
  struct DevInfo {
    std::atomic<int> sms{0};
  };
  static DevInfo devs[64];
  DevInfo& di = devs[c.device & 63];
  int sms = di.sms.load(std::memory_order_acquire);
  if (sms == 0) {
    if (cudaFuncSetAttribute(i8gemm_tc05_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES) !=
            cudaSuccess ||
        cudaFuncSetAttribute(i8gemm_tc05_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES) !=
            cudaSuccess)
      fail(QLRA_ERR_CUDA, "i8gemm: cannot reserve the shared-memory ring");
    QLRA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
    di.sms.store(sms, std::memory_order_release);
  }
  CUtensorMap ma, mb, mc;
  if (mode == 0)
    make_map_c(&mc, C, N, M, batch, ldc, stride_c, EPI_COLS, 32, true);  // [m][n], swizzled staging
  else
    make_map_c(&mc, C, M, N, batch, ldc, stride_c, 32, EPI_COLS, false);  // [n][m]
  if (mode == 0)
    make_map(&ma, A, K, M, batch, lda, stride_a, BM);  // rows m, K inner
  else
    make_map(&ma, A, M, K, batch, lda, stride_a, BM);  // rows k, M inner (box: 128 m x 128 k)
  Args g{};
  g.M = M, g.N = N, g.K = K;
  g.batch = batch, g.beta = beta, g.mode = mode;
  // CTA pairs (256-row tiles) unless M fits one CTA's rows; QLRA_I8_CTAS=1|2 overrides
  bool two = ctas == 0 ? M > BM : ctas == 2;
  if (const char* e = std::getenv("QLRA_I8_CTAS")) two = std::atoi(e) == 2;
  const int tm = two ? 2 * BM : BM;
  make_map(&mb, B, K, N, batch, ldb, stride_b, two ? BN / 2 : BN);
  g.tiles_m = (int)((M + tm - 1) / tm);
  g.tiles_n = (int)((N + BN - 1) / BN);
  g.num_k = (int)((K + BK - 1) / BK);
  g.total_tiles = (int64_t)batch * g.tiles_m * g.tiles_n;
  // CTAs (or pairs) in flight, and the sibling rendezvous: persistent grids
  // whose size is a multiple of the row's 2 or 4 n-tiles (so that a row's
  // siblings always run in the same sweep), tiles long enough to drift
  int64_t units = two ? sms / 2 : sms;
  bool rendezvous = (g.tiles_n == 2 || g.tiles_n == 4) && g.num_k >= 16;
  if (const char* e = std::getenv("QLRA_I8_SIBSYNC")) rendezvous = rendezvous && std::atoi(e) != 0;
  if (rendezvous) units = units / g.tiles_n * g.tiles_n;
  if (g.total_tiles < units) rendezvous = false, units = g.total_tiles;
  unsigned* sync = nullptr;
  g.sync = nullptr;
  g.sib = 0;
  if (rendezvous) {
    const size_t bytes = sizeof(unsigned) * (size_t)(g.total_tiles / g.tiles_n);
    QLRA_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&sync), bytes, stream));
    QLRA_CUDA(cudaMemsetAsync(sync, 0, bytes, stream));
    g.sync = sync;
    g.sib = (unsigned)g.tiles_n * (two ? 2u : 1u);  // every CTA's producer arrives
  }
  if (two)
    i8gemm_tc05_2sm_kernel<<<2 * (unsigned)units, NTHREADS, SMEM_BYTES, stream>>>(ma, mb, mc, g);
  else
    i8gemm_tc05_kernel<<<(unsigned)units, NTHREADS, SMEM_BYTES, stream>>>(ma, mb, mc, g);
  const cudaError_t le = cudaGetLastError();
  if (sync) cudaFreeAsync(sync, stream);
  cuda_check(le, "kernel launch");
  count_launch();
}

}  // namespace qlra_dev
