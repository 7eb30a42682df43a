// i8gemm.cuh -- batched int8 x int8 -> int32 GEMMs on tcgen05 (i8gemm.cu).
#pragma once

#include <cstdint>

#include "kernels.cuh"

namespace qlra_dev {

// C[b] = (beta ? C[b] : 0) + A[b] B[b]^T for b < batch, exact in int32.
//   mode 0: A is M x K (K contiguous, lda), B is N x K (ldb), C[m * ldc + n];
//   mode 1: A is K x M (M contiguous, lda), B is N x K (ldb), C[n * ldc + m].
// N, lda, ldb and the operand batch strides are multiples of 16, ldc and
// stride_c of 4 (mode 1: M too), pointers 16-byte aligned; reads past M / N / K are zero
// filled by TMA, stores are clipped to M x N.  ctas: 2 = CTA pairs (256-row
// tiles, tcgen05.mma.cta_group::2), 1 = single CTAs, 0 = pairs when M > 128.
void i8gemm_batched(Ctx& c, int mode, int64_t M, int64_t N, int64_t K, const int8_t* A, int64_t lda, int64_t stride_a,
                    const int8_t* B, int64_t ldb, int64_t stride_b, int32_t* C, int64_t ldc, int64_t stride_c,
                    int batch, int beta, cudaStream_t stream, int ctas = 0);
const char* i8gemm_kernel_name();

}  // namespace qlra_dev
