// Probe: cuBLASLt int8 x int8 -> int32 batched GEMM on this B200: which
// operand layouts have an algorithm, and their throughput at the Ozaki
// sketch shapes.  nvcc -O2 -arch=sm_100a tools/probe_lt.cu -lcublasLt -o /tmp/probe_lt
#include <cublasLt.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#define CK(x) do { auto e = (x); if ((int)e) { printf("err %d at %s:%d\n", (int)e, __FILE__, __LINE__); return -1; } } while (0)
static cublasLtHandle_t H;
static void* ws; static size_t wsz = 64 << 20;
// column-major C (m x n) = op(A) (m x k) * op(B) (k x n), batch b
double run(cublasOperation_t ta, cublasOperation_t tb, int64_t m, int64_t n, int64_t k, int batch, bool time_it) {
  int64_t lda = ta == CUBLAS_OP_N ? m : k, ldb = tb == CUBLAS_OP_N ? k : n, ldc = m;
  lda = (lda + 15) / 16 * 16; ldb = (ldb + 15) / 16 * 16; ldc = (ldc + 3) / 4 * 4;
  int64_t sa = lda * (ta == CUBLAS_OP_N ? k : m), sb = ldb * (tb == CUBLAS_OP_N ? n : k), sc = ldc * n;
  int8_t *A, *B; int32_t* C;
  if (cudaMalloc(&A, sa * batch) || cudaMalloc(&B, sb * batch) || cudaMalloc(&C, sc * 4 * batch)) { printf("oom\n"); cudaGetLastError(); return -2; }
  cudaMemset(A, 1, sa * batch); cudaMemset(B, 1, sb * batch);
  cublasLtMatmulDesc_t d; cublasLtMatrixLayout_t la, lb, lc;
  cublasLtMatmulDescCreate(&d, CUBLAS_COMPUTE_32I, CUDA_R_32I);
  cublasLtMatmulDescSetAttribute(d, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta));
  cublasLtMatmulDescSetAttribute(d, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb));
  cublasLtMatrixLayoutCreate(&la, CUDA_R_8I, ta == CUBLAS_OP_N ? m : k, ta == CUBLAS_OP_N ? k : m, lda);
  cublasLtMatrixLayoutCreate(&lb, CUDA_R_8I, tb == CUBLAS_OP_N ? k : n, tb == CUBLAS_OP_N ? n : k, ldb);
  cublasLtMatrixLayoutCreate(&lc, CUDA_R_32I, m, n, ldc);
  for (auto [l, s] : {std::pair{la, sa}, std::pair{lb, sb}, std::pair{lc, sc}}) {
    cublasLtMatrixLayoutSetAttribute(l, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &batch, sizeof(batch));
    cublasLtMatrixLayoutSetAttribute(l, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &s, sizeof(s));
  }
  cublasLtMatmulPreference_t pref; cublasLtMatmulPreferenceCreate(&pref);
  cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsz, sizeof(wsz));
  cublasLtMatmulHeuristicResult_t res[4]; int nres = 0;
  auto st = cublasLtMatmulAlgoGetHeuristic(H, d, la, lb, lc, lc, pref, 4, res, &nres);
  double tops = -1;
  if (st || nres == 0) {
    printf("  %c%c m=%ld n=%ld k=%ld b=%d: no algorithm (status %d)\n", ta == CUBLAS_OP_N ? 'N' : 'T', tb == CUBLAS_OP_N ? 'N' : 'T', (long)m, (long)n, (long)k, batch, (int)st);
  } else {
    int32_t alpha = 1, beta = 1;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int reps = time_it ? 5 : 1;
    for (int w = 0; w < 2; ++w) cublasLtMatmul(H, d, &alpha, A, la, B, lb, &beta, C, lc, C, lc, &res[0].algo, ws, wsz, 0);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) cublasLtMatmul(H, d, &alpha, A, la, B, lb, &beta, C, lc, C, lc, &res[0].algo, ws, wsz, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    auto err = cudaGetLastError();
    tops = 2.0 * m * n * k * batch / (ms * 1e9);
    printf("  %c%c m=%ld n=%ld k=%ld b=%d: %.3f ms %.0f TOPS (err %d, beta=1)\n", ta == CUBLAS_OP_N ? 'N' : 'T', tb == CUBLAS_OP_N ? 'N' : 'T', (long)m, (long)n, (long)k, batch, ms, tops, (int)err);
  }
  cudaFree(A); cudaFree(B); cudaFree(C);
  return tops;
}
int main() {
  cublasLtCreate(&H); cudaMalloc(&ws, wsz);
  auto N = CUBLAS_OP_N, T = CUBLAS_OP_T;
  printf("layouts (8192^3, batch 1):\n");
  for (auto ta : {N, T}) for (auto tb : {N, T}) run(ta, tb, 8192, 8192, 8192, 1, true);
  printf("Y side (col-major C = s x R): m=s=500, n=R, k=n=27136, batch 128:\n");
  run(T, N, 500, 2048, 27136, 128, true);
  run(T, N, 512, 2048, 27136, 128, true);
  run(T, N, 500, 8192, 27136, 32, true);
  printf("W side (col-major C = n x l): m=27136, n=l=1000, k=R, batch 128:\n");
  run(T, N, 27136, 1000, 2048, 128, true);
  run(N, N, 27136, 1000, 2048, 128, true);
  run(T, N, 27136, 1024, 2048, 64, true);
  printf("C2 shapes: Y m=100 n=8000 k=6000; W m=6000 n=200 k=8000 (batch 128)\n");
  run(T, N, 100, 8000, 6000, 128, true);
  run(T, N, 6000, 200, 8000, 128, true);
  run(N, N, 6000, 200, 8000, 128, true);
  printf("C5 shapes: Y m=40 n=131072 k=300; W m=300 n=80 k=131072 (batch 128)\n");
  run(T, N, 40, 131072, 304, 128, true);
  run(T, N, 304, 80, 131072, 128, true);
  return 0;
}
