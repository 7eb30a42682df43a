// common.cuh -- shared device helpers for the qlra B200 kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "qlra_cuda.h"

namespace qlra_dev {

// ------------------------------------------------------------ status ---
struct Status : std::runtime_error {
  int code;
  double cond;
  Status(int c, const std::string& m, double k = 0.0) : std::runtime_error(m), code(c), cond(k) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg, double cond = 0.0) {
  throw Status(code, msg, cond);
}
inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    fail(QLRA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define QLRA_CUDA(x) ::qlra_dev::cuda_check((x), #x)
#define QLRA_LAUNCH_CHECK() ::qlra_dev::cuda_check(cudaGetLastError(), "kernel launch")

// ----------------------------------------------------- matrix views ---
// Device view of one quaternion matrix (4 row-major planes, leading dim ld).
struct QView {
  double* p[4];
  int64_t rows, cols, ld;
};
// Device view of a complex matrix: column-major, interleaved (re, im).
struct CView {
  double* data;
  int64_t rows, cols, ld;
};
inline CView cview_of(const qlra_cmat_t* m) { return CView{m->data, m->rows, m->cols, m->ld}; }

inline QView view_of(const qlra_qmat_t* m) {
  QView v;
  for (int i = 0; i < 4; ++i) v.p[i] = m->p[i];
  v.rows = m->rows;
  v.cols = m->cols;
  v.ld = m->ld;
  return v;
}

// ------------------------------------------------------------- RNG ---
// Counter-based splitmix64 stream (proj/include/qlra/rng.hpp:10-55).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kSalt = 0xD1B54A32D192ED03ULL;
__host__ __device__ __forceinline__ uint64_t rng_key(uint64_t seed) { return mix64(seed ^ kSalt); }
__host__ __device__ __forceinline__ uint64_t rng_substream(uint64_t key, uint64_t index) {
  return mix64(key ^ mix64(index + kSalt));
}
__host__ __device__ __forceinline__ uint64_t rng_u64_at(uint64_t key, uint64_t c) {
  return mix64(key + kGolden * (c + 1));
}
__host__ __device__ __forceinline__ double rng_uniform_at(uint64_t key, uint64_t c) {
  return static_cast<double>(rng_u64_at(key, c) >> 11) * 0x1.0p-53;
}
// Box-Muller exactly as rng.hpp:42-47 / sketching.cpp:32-34 (2*M_PI folded
// to the same double constant).  The device log1p/cos may differ from glibc
// by an ulp on some draws; the integer streams are bit-identical.
__device__ __forceinline__ double box_muller(double u1, double u2) {
  const double kTwoPi = 6.283185307179586476925286766559;
  return sqrt(-2.0 * log1p(-u1)) * cos(kTwoPi * u2);
}

}  // namespace qlra_dev
