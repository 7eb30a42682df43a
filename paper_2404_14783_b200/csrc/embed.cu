// embed.cu -- K1: on-device generation of the sketching test matrices.
//
// Replaces gen_block / entry_value (proj/src/sketching.cpp:25-71) and the
// CounterRng draws they make (proj/include/qlra/rng.hpp:32-47).  Entry (i, j)
// of plane p of a spec uses stream CounterRng(seed).substream(p) with counter
// base 4*(i*cols + j): Gaussian draws base+0/+1, the sparse keep test base+2,
// the Rademacher sign base+3.  Every block regenerates bit-identically in its
// integer draws, which is what lets each rank build its own Psi column slice
// with no broadcast.
#include "common.cuh"
#include "kernels.cuh"

namespace qlra_dev {

namespace {

struct GenArgs {
  QView out;
  int kind;
  double density;
  uint64_t key[4];
  int64_t spec_cols, r0, c0, nrows, ncols;
  int transposed;  // write out(j, i) instead of out(i, j)
};

template <int KIND>
__device__ __forceinline__ double entry_value(uint64_t key, double density, uint64_t idx) {
  constexpr int kind = KIND;
  const uint64_t base = 4 * idx;
  switch (kind) {
    case QLRA_GAUSSIAN:
      return box_muller(rng_uniform_at(key, base), rng_uniform_at(key, base + 1));
    case QLRA_RADEMACHER:
      return (rng_u64_at(key, base + 3) & 1u) ? 1.0 : -1.0;
    case QLRA_SPARSE_GAUSSIAN:
      if (rng_uniform_at(key, base + 2) >= density) return 0.0;
      return box_muller(rng_uniform_at(key, base), rng_uniform_at(key, base + 1)) /
             sqrt(density);
    default:  // QLRA_SPARSE_RADEMACHER
      if (rng_uniform_at(key, base + 2) >= density) return 0.0;
      return ((rng_u64_at(key, base + 3) & 1u) ? 1.0 : -1.0) / sqrt(density);
  }
}

// one instantiation per kind: the four planes' draws of an entry are
// independent and interleave (no runtime switch between them)
template <int KIND>
__global__ void gen_kernel(GenArgs a) {
  const int64_t cols = a.ncols;
  const int64_t total = a.nrows * a.ncols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / cols, j = e % cols;
    const uint64_t idx = (uint64_t)(a.r0 + i) * (uint64_t)a.spec_cols + (uint64_t)(a.c0 + j);
    const int64_t off = a.transposed ? j * a.out.ld + i : i * a.out.ld + j;
#pragma unroll
    for (int p = 0; p < 4; ++p)
      a.out.p[p][off] = entry_value<KIND>(a.key[p], a.density, idx);
  }
}

}  // namespace

void launch_gen(cudaStream_t st, const qlra_spec_t& spec, int64_t r0, int64_t c0, int64_t nrows,
                int64_t ncols, const QView& out, bool transposed) {
  GenArgs a;
  a.out = out;
  a.kind = spec.kind;
  a.density = spec.density;
  const uint64_t root = rng_key(spec.seed);
  for (int p = 0; p < 4; ++p) a.key[p] = rng_substream(root, (uint64_t)p);
  a.spec_cols = spec.cols;
  a.r0 = r0;
  a.c0 = c0;
  a.nrows = nrows;
  a.ncols = ncols;
  a.transposed = transposed ? 1 : 0;
  const int64_t total = nrows * ncols;
  if (total == 0) return;
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  switch (spec.kind) {
    case QLRA_GAUSSIAN: gen_kernel<QLRA_GAUSSIAN><<<(unsigned)blocks, threads, 0, st>>>(a); break;
    case QLRA_RADEMACHER: gen_kernel<QLRA_RADEMACHER><<<(unsigned)blocks, threads, 0, st>>>(a); break;
    case QLRA_SPARSE_GAUSSIAN: gen_kernel<QLRA_SPARSE_GAUSSIAN><<<(unsigned)blocks, threads, 0, st>>>(a); break;
    default: gen_kernel<QLRA_SPARSE_RADEMACHER><<<(unsigned)blocks, threads, 0, st>>>(a); break;
  }
  QLRA_LAUNCH_CHECK();
  count_launch();
}

}  // namespace qlra_dev
