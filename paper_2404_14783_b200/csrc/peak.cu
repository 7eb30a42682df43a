// peak.cu -- measured FP64 throughput of the device (roofline denominator).
//
// BASELINE.md has no FP64 entry in MEASURED_PEAKS.json, so the sketch's
// compute roofline uses the peak measured here, on the same box, in the same
// bench run: mode 0 = DFMA (SIMT FP64 pipe), mode 1 = DMMA
// m8n8k4 (the only f64 tensor shape on sm_100; tcgen05 has no f64 kind).
#include "common.cuh"
#include "kernels.cuh"

namespace qlra_dev {

namespace {

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = fma(x[j], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_dmma(double* out, int iters, double a, double b) {
  double c[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) { c[j][0] = 0.0; c[j][1] = 0.0; }
  const double av = a + threadIdx.x * 1e-9, bv = b;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1])
                   : "d"(av), "d"(bv));
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// mode 2: half the warps DMMA, half DFMA (4x the iterations, equal flops):
// a combined rate above the DMMA peak would mean the two pipes issue
// concurrently.
__global__ void __launch_bounds__(256) k_mixed(double* out, int iters, double a, double b) {
  const int w = threadIdx.x >> 5;
  double s = 0.0;
  if (w & 1) {
    double x[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < 4 * iters; ++i) {
#pragma unroll
      for (int j = 0; j < 16; ++j) x[j] = fma(x[j], a, b);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) s += x[j];
  } else {
    double c[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) { c[j][0] = 0.0; c[j][1] = 0.0; }
    const double av = a + threadIdx.x * 1e-9, bv = b;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[j][0]), "+d"(c[j][1])
                     : "d"(av), "d"(bv));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace

double measure_fp64_peak(Ctx& ctx, int mode, double ms) {
  int sms = 148;
  QLRA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx.device));
  const int blocks = sms * 4, threads = 256;
  DeviceBuffer out(ctx, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1;
  QLRA_CUDA(cudaEventCreate(&e0));
  QLRA_CUDA(cudaEventCreate(&e1));
  auto run = [&](int iters) {
    QLRA_CUDA(cudaEventRecord(e0, ctx.stream));
    if (mode == 0)
      k_dfma<<<blocks, threads, 0, ctx.stream>>>(out.as<double>(), iters, 0.999999, 1e-7);
    else if (mode == 1)
      k_dmma<<<blocks, threads, 0, ctx.stream>>>(out.as<double>(), iters, 0.999999, 1e-7);
    else
      k_mixed<<<blocks, threads, 0, ctx.stream>>>(out.as<double>(), iters, 0.999999, 1e-7);
    QLRA_LAUNCH_CHECK();
    count_launch();
    QLRA_CUDA(cudaEventRecord(e1, ctx.stream));
    QLRA_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    QLRA_CUDA(cudaEventElapsedTime(&t, e0, e1));
    return (double)t;
  };
  int iters = 1000;
  run(iters);  // warm-up
  double t = run(iters);
  while (t < ms * 0.5 && iters < (1 << 26)) {
    iters *= 2;
    t = run(iters);
  }
  double best = 1e300;
  for (int r = 0; r < 3; ++r) best = std::min(best, run(iters));
  QLRA_CUDA(cudaEventDestroy(e0));
  QLRA_CUDA(cudaEventDestroy(e1));
  const double warps = (double)blocks * threads / 32.0;
  const double flops = mode == 0   ? 2.0 * 16.0 * iters * blocks * threads
                       : mode == 1 ? 512.0 * 8.0 * iters * warps
                                   : 0.5 * warps * (512.0 * 8.0 * iters + 32.0 * 2.0 * 16.0 * 4.0 * iters);
  return flops / (best * 1e-3) / 1e12;
}

}  // namespace qlra_dev
