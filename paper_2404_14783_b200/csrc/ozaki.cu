// ozaki.cu -- the fused dual sketch on the INT8 tensor cores.
//
// Replaces the same reference step as sketch8_kernel (sketch_update_rows,
// proj/src/sketching.cpp:125-139: Y += A Omega, W += Psi A through
// qmat_mul_accumulate_ordered, qmatrix.cpp:203-242), for the shapes where it
// is faster (oz_wanted).  FP64 has no tcgen05 kind on sm_100 (DMMA.8x8x4 at
// 37 TFLOP/s is the FP64 tensor ceiling), but INT8 does (tcgen05.mma
// kind::i8, 2.6-3 POPS sustained at the board's power cap).  So every
// real product of the sketch is computed EXACTLY in integers (the Ozaki
// scheme, CRT form) and rounded once at the end:
//
//  * scaling: A' = rint(A 2^sigma) with one power-of-two scale per epoch
//    (|A'| <= 2^beta, beta = 49 with 15 moduli or 52 with 16), Omega' per
//    column (2^tau_j), Psi' per row (2^rho_k): the only rounding of the
//    operands, 2^-(beta+1) relative to their maxima;
//  * the 8-product identity (qtile8.cuh): each quaternion GEMM is 8 real
//    GEMMs of plane combinations (exact integers < 2^53 after scaling);
//  * residues: each combination reduced modulo 16 pairwise-coprime moduli
//    p <= 256 (symmetric int8); the 8 x 16 = 128 residue products are ONE
//    batched int8 x int8 -> int32 GEMM per sketch side (exact while K 128^2
//    < 2^31, i.e. K < 2^17 rows or columns per int32 accumulation), run by
//    the engine's own tcgen05 kernel (i8gemm.cu; cuBLASLt's IMMA kernel is
//    kept as the A/B reference, QLRA_OZ_GEMM=lt, and for the general
//    long-K product oz_gemm_try);
//  * recovery: the CRT in 128-bit integers (P = prod p = 2^124.7 > 2 K
//    2^106 for 16 moduli; 15 moduli and 49-bit scales when K <= 2^15), the 8 products combined into the quaternion planes exactly in
//    int128, one rounding to double, scaled back by powers of two.
//
// One residue set serves both sketches: Y = A Omega takes lcomb(A) as its
// left operand, and W is formed as its adjoint W^* = A^* Psi^*, whose left
// combinations lcomb(conj A) are a signed permutation of lcomb(A) (below),
// so the A residues are written once per panel (row-major: the K-major left
// operand of Y's GEMM and, read as a column-major n x R matrix, the left
// operand of W^*'s).  W's int32 products accumulate over panels (beta = 1)
// within an epoch (rows < 2^17 and one A scale) and are recovered once.
//
// Determinism: integer products are exact, so the result does not depend on
// cuBLASLt's algorithm, split-K or batch order: bitwise reproducible.
#include <cublasLt.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "i8gemm.cuh"
#include "kernels.cuh"
#include "ozaki.cuh"
#include "qtile8.cuh"

namespace qlra_dev {

namespace {

constexpr int NMOD = 16;                // moduli available; a call uses the first nmod (15 or 16)
constexpr int NB = 8 * NMOD;            // batch: (combination t, modulus mu), b = t * nmod + mu
constexpr int64_t KMAX = 131056;        // K per int32 accumulation: K * 128^2 < 2^31 (multiple of 16)
constexpr int NTAB = 2;                 // CRT tables: [0] the 16 moduli, [1] the first 15
// odd moduli <= 253: a residue off the symmetric range by one (below) still
// fits int8; 256 wraps in int8 congruently.  P = 2^124.7 > 2 * 2^17 * 2^106.
constexpr int kModuli[NMOD] = {256, 253, 251, 247, 241, 239, 233, 229, 227, 223, 211, 199, 197, 193, 191, 181};

__constant__ int c_p[NMOD];
__constant__ double c_pinv[NMOD];
__constant__ float c_pinvf[NMOD];
__constant__ int c_yinv[NTAB][NMOD];                   // (P / p)^-1 mod p
__constant__ unsigned long long c_M[NTAB][NMOD][2];    // P / p as (lo, hi)
__constant__ unsigned long long c_P[NTAB][2], c_H[NTAB][2];  // P, floor(P / 2)
__constant__ unsigned long long c_m64[NMOD];             // ceil(2^64 / p)
__constant__ unsigned c_m32[NMOD];                       // ceil(2^32 / p)
__constant__ long long c_off[NMOD];                      // p 2^24 >= 2^31: makes an int32 non-negative

// Moduli in use: the first nmod, CRT table tab, operands scaled to < 2^beta
// per plane (combinations < 2^(beta+1)): P > 2 K 2^(2 beta + 2) bounds the
// products of an int32 accumulation of K terms.
struct ModCfg {
  int nmod, tab, beta;
};

// lcomb(conj a)_t = kConjSign[t] * lcomb(a)_{kConjPerm[t]}: conj(a) = (a0,
// -a1, -a2, -a3) in qtile8's lcomb list (a0+a1, a3-a2, a0-a1, a2+a3, a1+a3,
// a1-a3, a0+a2, a0-a2) gives (L2, -L1, L0, -L3, -L4, -L5, L7, L6).
//   kConjPerm = {2, 1, 0, 3, 4, 5, 7, 6}, kConjSign = {1, -1, 1, -1, -1, -1, 1, 1}

typedef unsigned __int128 u128;
typedef __int128 i128;

struct ModTables {
  int p[NMOD], yinv[NMOD];
  double pinv[NMOD];
  float pinvf[NMOD];
  unsigned long long M[NMOD][2], P[2], H[2];
  unsigned long long m64[NMOD];
  unsigned m32[NMOD];
  long long off[NMOD];
  double log2P = 0.0;
};

ModTables make_tables(int nmod) {
  ModTables t{};
  u128 P = 1;
  for (int i = 0; i < nmod; ++i) {
    for (int j = 0; j < i; ++j) {
      int a = kModuli[i], b = kModuli[j];
      while (b) { const int r = a % b; a = b; b = r; }
      if (a != 1) fail(QLRA_ERR_CUDA, "ozaki: moduli not pairwise coprime");
    }
    P *= (u128)kModuli[i];
    t.log2P += std::log2((double)kModuli[i]);
  }
  for (int i = 0; i < nmod; ++i) {
    const int p = kModuli[i];
    const u128 M = P / (u128)p;
    const int mr = (int)(M % (u128)p);
    int inv = -1;
    for (int x = 1; x < p; ++x)
      if ((mr * x) % p == 1) { inv = x; break; }
    if (inv < 0) fail(QLRA_ERR_CUDA, "ozaki: no CRT inverse");
    t.p[i] = p;
    t.yinv[i] = inv;
    t.pinv[i] = 1.0 / p;
    t.pinvf[i] = 1.0f / (float)p;
    // ceil(2^64 / p) (2^56 for p = 256, exact) and ceil(2^32 / p)
    t.m64[i] = (unsigned long long)((((u128)1 << 64) + (u128)(p - 1)) / (u128)p);
    t.m32[i] = (unsigned)((((unsigned long long)1 << 32) + (unsigned long long)(p - 1)) / (unsigned long long)p);
    t.off[i] = (long long)p << 24;
    t.M[i][0] = (unsigned long long)M;
    t.M[i][1] = (unsigned long long)(M >> 64);
  }
  t.P[0] = (unsigned long long)P;
  t.P[1] = (unsigned long long)(P >> 64);
  const u128 H = P >> 1;
  t.H[0] = (unsigned long long)H;
  t.H[1] = (unsigned long long)(H >> 64);
  return t;
}

const ModTables& tables(int tab) {
  static const ModTables t[NTAB] = {make_tables(16), make_tables(15)};
  return t[tab];
}

void upload_tables(int device) {
  static std::mutex mu;
  static bool done[64] = {};
  std::lock_guard<std::mutex> g(mu);
  if (device >= 0 && device < 64 && done[device]) return;
  const ModTables& t = tables(0);
  QLRA_CUDA(cudaMemcpyToSymbol(c_p, t.p, sizeof(t.p)));
  QLRA_CUDA(cudaMemcpyToSymbol(c_pinv, t.pinv, sizeof(t.pinv)));
  QLRA_CUDA(cudaMemcpyToSymbol(c_pinvf, t.pinvf, sizeof(t.pinvf)));
  QLRA_CUDA(cudaMemcpyToSymbol(c_m64, t.m64, sizeof(t.m64)));
  QLRA_CUDA(cudaMemcpyToSymbol(c_m32, t.m32, sizeof(t.m32)));
  QLRA_CUDA(cudaMemcpyToSymbol(c_off, t.off, sizeof(t.off)));
  for (int k = 0; k < NTAB; ++k) {
    const ModTables& u = tables(k);
    QLRA_CUDA(cudaMemcpyToSymbol(c_yinv, u.yinv, sizeof(u.yinv), k * sizeof(u.yinv)));
    QLRA_CUDA(cudaMemcpyToSymbol(c_M, u.M, sizeof(u.M), k * sizeof(u.M)));
    QLRA_CUDA(cudaMemcpyToSymbol(c_P, u.P, sizeof(u.P), k * sizeof(u.P)));
    QLRA_CUDA(cudaMemcpyToSymbol(c_H, u.H, sizeof(u.H), k * sizeof(u.H)));
  }
  if (device >= 0 && device < 64) done[device] = true;
}

// ---------------------------------------------------------------- device --
// |x| < 2^53 exact integer (x_lo: its low 32 bits) -> a residue mod p_mu
// that fits int8, with ONE FP64 op: the quotient q = x / p rounded to the
// nearest integer through the 1.5 * 2^52 shifter (its double then carries
// q mod 2^32 in the low word: the shifter's low 32 bits are zero), and
// r = x - p q computed in wrapping 32-bit integers -- exact, since the true
// r is small.  x * (1/p) is off by < 0.0015 for |x| < 2^53, so for odd p
// (x / p never within 1 / (2p) > 0.0015 of a half) q = round(x / p) and
// |r| <= (p - 1) / 2 <= 126; for p = 256 (r = +-128 at exact halves) the
// int8 wrap is congruent mod 256.  (The CRT takes any representative.)
__device__ __forceinline__ int sres(double x, int x_lo, int mu) {
  constexpr double kShift = 6755399441055744.0;  // 1.5 * 2^52
  const int q_lo = __double2loint(fma(x, c_pinv[mu], kShift));
  return x_lo - c_p[mu] * q_lo;
}
__device__ __forceinline__ unsigned pack4(int a, int b, int c, int d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

// the 8 x 16 residue words of 4 consecutive elements: word (t, mu) at
// o[(t * nmod + mu) * ws] (ws: words per batch matrix)
__device__ __forceinline__ void store_res(unsigned* o, int64_t ws, const double (&c)[8][4], int nmod) {
  const int64_t ts = nmod * ws;
  int lo[8][4];  // low 32 bits of the exact integers (one conversion each, shared by all moduli)
#pragma unroll
  for (int t = 0; t < 8; ++t)
#pragma unroll
    for (int q = 0; q < 4; ++q) lo[t][q] = (int)(unsigned long long)__double2ll_rn(c[t][q]);
#pragma unroll 1
  for (int mu = 0; mu < nmod; ++mu, o += ws)
#pragma unroll
    for (int t = 0; t < 8; ++t)
      o[t * ts] = pack4(sres(c[t][0], lo[t][0], mu), sres(c[t][1], lo[t][1], mu), sres(c[t][2], lo[t][2], mu),
                        sres(c[t][3], lo[t][3], mu));
}

// max |x| over the four planes of a view -> atomicMax on the bit pattern
// (non-negative doubles order like their unsigned bits)
__global__ void k_absmax(QView a, unsigned long long* out) {
  double m = 0.0;
  const int64_t total = a.rows * a.cols;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / a.cols, j = e - i * a.cols;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const double v = a.p[p][i * a.ld + j];
      m = fmax(m, isfinite(v) ? fabs(v) : INFINITY);  // NaN / inf report inf (fmax would drop a NaN)
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double sm[32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0 && m > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
  }
}

// per-column max |x| of a (rows x cols) view: out[j] (bits, atomicMax)
__global__ void k_colmax(QView a, unsigned long long* out) {
  const int64_t j = blockIdx.x * (int64_t)32 + (threadIdx.x & 31);
  if (j >= a.cols) return;
  double m = 0.0;
  for (int64_t i = blockIdx.y * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < a.rows;
       i += (int64_t)gridDim.y * (blockDim.x >> 5))
#pragma unroll
    for (int p = 0; p < 4; ++p) m = fmax(m, fabs(a.p[p][i * a.ld + j]));
  if (m > 0.0) atomicMax(out + j, (unsigned long long)__double_as_longlong(m));
}

// per-row max |x|: one block per row
__global__ void k_rowmax(QView a, unsigned long long* out) {
  const int64_t i = blockIdx.x;
  double m = 0.0;
  for (int64_t j = threadIdx.x; j < a.cols; j += blockDim.x)
#pragma unroll
    for (int p = 0; p < 4; ++p) m = fmax(m, fabs(a.p[p][i * a.ld + j]));
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double sm[32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? sm[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) out[i] = (unsigned long long)__double_as_longlong(m);
  }
}

// 2^e with max * 2^e in [2^(beta-1), 2^beta) (0 for an all-zero line)
__device__ __forceinline__ int scale_exp(unsigned long long maxbits, int beta) {
  const double m = __longlong_as_double((long long)maxbits);
  return m > 0.0 ? beta - 1 - ilogb(m) : 0;
}

// A panel (R x n) -> Ares[t*16+mu][i][k] (Rpad x npad, zero padded):
// residues of lcomb_t(rint(A 2^sigma)).  Thread: one row, 4 columns.
__global__ void k_res_a(QView a, int64_t npad, int64_t rpad, int sigma, int8_t* out, int64_t pitch, int64_t bstride,
                        int nmod) {
  const int64_t nw = npad >> 2;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= rpad * nw) return;
  const int64_t i = e / nw, k0 = (e - i * nw) * 4;
  const double s1 = ldexp(1.0, sigma / 2), s2 = ldexp(1.0, sigma - sigma / 2);  // 2^sigma, exact in two steps
  double c[8][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    if (i < a.rows && k0 + q < a.cols) {
#pragma unroll
      for (int p = 0; p < 4; ++p) v[p] = rint(a.p[p][i * a.ld + k0 + q] * s1 * s2);
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t][q] = qt8::lcomb(t, v);
  }
  store_res(reinterpret_cast<unsigned*>(out + i * pitch + k0), bstride >> 2, c, nmod);
}

// Omega (n x s) -> Ores[t*16+mu][j][k] (s x npad): residues of
// rcomb_t(rint(Omega(k, j) 2^tau_j)).  Thread: one column j, 4 rows k.
__global__ void k_res_om(QView om, const unsigned long long* colmax, int64_t npad, int64_t spad, int8_t* out, int64_t pitch,
                         int64_t bstride, ModCfg mc) {
  const int64_t nw = npad >> 2;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= spad * nw) return;
  const int64_t j = e / nw, k0 = (e - j * nw) * 4;
  const int tau = j < om.cols ? scale_exp(colmax[j], mc.beta) : 0;
  const double s1 = ldexp(1.0, tau / 2), s2 = ldexp(1.0, tau - tau / 2);
  double c[8][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    if (k0 + q < om.rows && j < om.cols) {
#pragma unroll
      for (int p = 0; p < 4; ++p) v[p] = rint(om.p[p][(k0 + q) * om.ld + j] * s1 * s2);
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t][q] = qt8::rcomb(t, v);
  }
  store_res(reinterpret_cast<unsigned*>(out + j * pitch + k0), bstride >> 2, c, mc.nmod);
}

// Psi columns [c0, c0 + R) (l x R) -> Pres[u*16+mu][k][i] (l x Rpad): the
// right operand of W^* = A^* Psi^*, rcomb_t(rint(conj(Psi(k, i)) 2^rho_k)),
// stored at the batch u = kConjPerm[t] of the A residues it multiplies.
__global__ void k_res_psi(QView ps, int64_t c0, int64_t R, int64_t rpad, int64_t lpad,
                          const unsigned long long* rowmax, int8_t* out, int64_t pitch, int64_t bstride, ModCfg mc) {
  const int64_t nw = rpad >> 2;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= lpad * nw) return;
  const int64_t k = e / nw, i0 = (e - k * nw) * 4;
  const int rho = k < ps.rows ? scale_exp(rowmax[k], mc.beta) : 0;
  const double s1 = ldexp(1.0, rho / 2), s2 = ldexp(1.0, rho - rho / 2);
  double c[8][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    if (i0 + q < R && k < ps.rows) {
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const double x = rint(ps.p[p][k * ps.ld + c0 + i0 + q] * s1 * s2);
        v[p] = p == 0 ? x : -x;
      }
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t][q] = qt8::rcomb(t, v);
  }
  // rcomb_t goes to batch kConjPerm[t] = {2, 1, 0, 3, 4, 5, 7, 6}
  double d[8][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    d[0][q] = c[2][q];
    d[1][q] = c[1][q];
    d[2][q] = c[0][q];
    d[3][q] = c[3][q];
    d[4][q] = c[4][q];
    d[5][q] = c[5][q];
    d[6][q] = c[7][q];
    d[7][q] = c[6][q];
  }
  store_res(reinterpret_cast<unsigned*>(out + k * pitch + i0), bstride >> 2, d, mc.nmod);
}

// the signed integer whose residues mod the 16 moduli are c[mu * bstride]
// (any int32 representatives), |X| < P / 2
__device__ __forceinline__ i128 crt(const int32_t* c, int64_t bstride, ModCfg mc) {
  const int tb = mc.tab;
  const u128 P = ((u128)c_P[tb][1] << 64) | c_P[tb][0];
  u128 acc = 0;
#pragma unroll 4
  for (int mu = 0; mu < mc.nmod; ++mu) {
    // v mod p and (r y) mod p by multiply-high with ceil(2^64 / p) and
    // ceil(2^32 / p): exact at these ranges, no conversion instructions
    const unsigned p = (unsigned)c_p[mu];
    const unsigned long long xv = (unsigned long long)((long long)c[mu * bstride] + c_off[mu]);  // >= 0, < 2^33
    const unsigned r = (unsigned)(xv - __umul64hi(xv, c_m64[mu]) * p);
    const unsigned t = r * (unsigned)c_yinv[tb][mu];  // < 2^16
    const unsigned u = t - __umulhi(t, c_m32[mu]) * p;
    acc += (u128)u * (((u128)c_M[tb][mu][1] << 64) | c_M[tb][mu][0]);
    if (acc >= P) acc -= P;
  }
  const u128 H = ((u128)c_H[tb][1] << 64) | c_H[tb][0];
  return acc > H ? -(i128)(P - acc) : (i128)acc;
}
__device__ __forceinline__ double i128_to_double(i128 x) {
  const bool neg = x < 0;
  const u128 m = neg ? (u128)(-x) : (u128)x;
  const double d = (double)(unsigned long long)(m >> 64) * 0x1p64 + (double)(unsigned long long)m;
  return neg ? -d : d;
}
// the quaternion planes of 2 x (product) from the 8 raw integer products
// (m_t without the Howell-Lafon halves of t >= 4): exact in int128
__device__ __forceinline__ void combine2(const i128 (&x)[8], i128 (&z)[4]) {
  const i128 s56 = x[4] + x[5], d56 = x[4] - x[5], s78 = x[6] + x[7], d78 = x[6] - x[7];
  z[0] = 2 * x[1] - s56 + s78;
  z[1] = 2 * x[0] - s56 - s78;
  z[2] = 2 * x[2] + d56 + d78;
  z[3] = 2 * x[3] + d56 - d78;
}

// Y rows of a panel += the recovered products.  cy[t*16+mu][i][j] (ld
// spad, batch stride bs).  Thread: one (i, j).
__global__ void k_crt_y(const int32_t* cy, int64_t bs, int64_t spad, QView y, const unsigned long long* om_colmax,
                        int sigma, ModCfg mc) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= y.rows * y.cols) return;
  const int64_t i = e / y.cols, j = e - i * y.cols;
  i128 x[8];
#pragma unroll 1
  for (int t = 0; t < 8; ++t) x[t] = crt(cy + (int64_t)t * mc.nmod * bs + i * spad + j, bs, mc);
  i128 z[4];
  combine2(x, z);
  const int sh = -(sigma + scale_exp(om_colmax[j], mc.beta)) - 1;  // the 2 of combine2
#pragma unroll
  for (int p = 0; p < 4; ++p) y.p[p][i * y.ld + j] += ldexp(i128_to_double(z[p]), sh);
}

// W += conj of the recovered W^* products.  cw[u*16+mu][k][j] (ld npad,
// batch stride bs), u = kConjPerm[t] holding sign kConjSign[t] * m_t.
__global__ void k_crt_w(const int32_t* cw, int64_t bs, int64_t npad, QView w, const unsigned long long* ps_rowmax,
                        int sigma, ModCfg mc) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= w.rows * w.cols) return;
  const int64_t k = e / w.cols, j = e - k * w.cols;
  i128 xu[8], x[8];
#pragma unroll 1
  for (int u = 0; u < 8; ++u) xu[u] = crt(cw + (int64_t)u * mc.nmod * bs + k * npad + j, bs, mc);
  // x[t] = kConjSign[t] * xu[kConjPerm[t]]
  x[0] = xu[2];
  x[1] = -xu[1];
  x[2] = xu[0];
  x[3] = -xu[3];
  x[4] = -xu[4];
  x[5] = -xu[5];
  x[6] = xu[7];
  x[7] = xu[6];
  i128 z[4];
  combine2(x, z);
  const int sh = -(sigma + scale_exp(ps_rowmax[k], mc.beta)) - 1;
  w.p[0][k * w.ld + j] += ldexp(i128_to_double(z[0]), sh);
#pragma unroll
  for (int p = 1; p < 4; ++p) w.p[p][k * w.ld + j] -= ldexp(i128_to_double(z[p]), sh);
}


// Rows of a K-major operand (rows x K) -> residues [t*16+mu][r][kpad] of
// lcomb_t (LEFT) or rcomb_t of rint(x 2^e_r), x = src or conj(src), with a
// per-row scale from rowmax (the general product's left rows / right
// columns).  Rows past src.rows and k past src.cols are zero.
template <bool LEFT>
__global__ void k_res_rows(QView src, int conj, const unsigned long long* rowmax, int64_t k0, int64_t kc,
                           int64_t kpad, int64_t rpad, int8_t* out, int64_t bstride) {
  const int64_t nw = kpad >> 2;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= rpad * nw) return;
  const int64_t r = e / nw, kk = (e - r * nw) * 4;
  const int ex = r < src.rows ? scale_exp(rowmax[r], 52) : 0;
  const double s1 = ldexp(1.0, ex / 2), s2 = ldexp(1.0, ex - ex / 2);
  double c[8][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    if (r < src.rows && kk + q < kc) {
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const double x = rint(src.p[p][r * src.ld + k0 + kk + q] * s1 * s2);
        v[p] = conj && p > 0 ? -x : x;
      }
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t][q] = LEFT ? qt8::lcomb(t, v) : qt8::rcomb(t, v);
  }
  store_res(reinterpret_cast<unsigned*>(out + r * kpad + kk), bstride >> 2, c, NMOD);
}

// dst (cols x rows, 4 planes, ld rows) = src^T (32 x 32 smem tiles)
__global__ void k_transpose(QView src, QView dst) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int p = 0; p < 4; ++p) {
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
      const int64_t r = r0 + i, c = c0 + threadIdx.x;
      tile[i][threadIdx.x] = r < src.rows && c < src.cols ? src.p[p][r * src.ld + c] : 0.0;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
      const int64_t c = c0 + i, r = r0 + threadIdx.x;
      if (c < src.cols && r < src.rows) dst.p[p][c * dst.ld + r] = tile[threadIdx.x][i];
    }
    __syncthreads();
  }
}

// C = alpha * (recovered product) + beta * C; ci[t*16+mu][i][j] (ld npad)
__global__ void k_crt_gen(const int32_t* ci, int64_t bs, int64_t npad, QView c, const unsigned long long* lmax,
                          const unsigned long long* rmax, double alpha, double beta) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= c.rows * c.cols) return;
  const int64_t i = e / c.cols, j = e - i * c.cols;
  i128 x[8];
#pragma unroll 1
  for (int t = 0; t < 8; ++t) x[t] = crt(ci + (int64_t)t * NMOD * bs + i * npad + j, bs, ModCfg{NMOD, 0, 52});
  i128 z[4];
  combine2(x, z);
  const int sh = -(scale_exp(lmax[i], 52) + scale_exp(rmax[j], 52)) - 1;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    double* d = c.p[p] + i * c.ld + j;
    const double v = alpha * ldexp(i128_to_double(z[p]), sh);
    *d = beta == 0.0 ? v : fma(beta, *d, v);
  }
}

inline unsigned blocks_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }
inline int64_t up16(int64_t x) { return (x + 15) / 16 * 16; }
inline int64_t up128(int64_t x) { return (x + 127) / 128 * 128; }

void lt_check(cublasStatus_t s, const char* what) {
  if (s != CUBLAS_STATUS_SUCCESS) fail(QLRA_ERR_CUDA, std::string("cuBLASLt ") + what + " failed (status " +
                                                        std::to_string((int)s) + ")");
}

}  // namespace

// ------------------------------------------------------------ host state --
// Per-context engine state: cuBLASLt handle, cached plans, grown buffers.
struct OzState {
  cublasLtHandle_t lt = nullptr;
  void* lt_ws = nullptr;
  size_t lt_ws_bytes = 0;
  struct Plan {
    cublasLtMatmulDesc_t d = nullptr;
    cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
    cublasLtMatmulAlgo_t algo{};
  };
  std::map<std::tuple<int, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, int>, Plan> plans;
  struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
  };
  Buf ares[2], pres[2], ores, cy[2], cw, stat;
  cudaStream_t aux = nullptr;  // residues / recovery beside the GEMMs (oz_sketch_block)
  unsigned long long* amax_dev = nullptr;   // 4 slots of max |A| (row pipeline: 0, 1; block: 2)
  unsigned long long* amax_host = nullptr;  // their pinned host copies
};

namespace {

void* grow(Ctx& c, OzState::Buf& b, size_t bytes) {
  if (b.bytes < bytes) {
    if (b.p) QLRA_CUDA(cudaFreeAsync(b.p, c.stream));
    b.p = nullptr;
    b.bytes = 0;
    QLRA_CUDA(cudaMallocAsync(&b.p, bytes, c.stream));
    b.bytes = bytes;
  }
  return b.p;
}

OzState& state(Ctx& c) {
  if (!c.oz) {
    upload_tables(c.device);
    auto* s = new OzState();
    c.oz = s;
    lt_check(cublasLtCreate(&s->lt), "create");
    s->lt_ws_bytes = 64u << 20;
    QLRA_CUDA(cudaMalloc(&s->lt_ws, s->lt_ws_bytes));
    QLRA_CUDA(cudaMallocHost(&s->amax_host, 4 * sizeof(unsigned long long)));
    QLRA_CUDA(cudaMalloc(&s->amax_dev, 4 * sizeof(unsigned long long)));
  }
  return *c.oz;
}

// col-major C (m x n, ldc) = op(A) (m x k) * op(B) (k x n) + beta C, int8 ->
// int32, `batch` matrices at the given strides (elements)
OzState::Plan& plan(OzState& s, bool ta, int64_t m, int64_t n, int64_t k, int64_t lda, int64_t ldb, int64_t ldc,
                    int64_t sa, int64_t sb, int64_t sc, int batch) {
  const auto key = std::make_tuple((int)ta, m, n, k, lda, ldb, ldc, batch);
  auto it = s.plans.find(key);
  if (it != s.plans.end()) return it->second;
  if (s.plans.size() >= 256) {  // many distinct panel heights (streamed blocks): start over
    for (auto& kv : s.plans) {
      cublasLtMatrixLayoutDestroy(kv.second.la);
      cublasLtMatrixLayoutDestroy(kv.second.lb);
      cublasLtMatrixLayoutDestroy(kv.second.lc);
      cublasLtMatmulDescDestroy(kv.second.d);
    }
    s.plans.clear();
  }
  OzState::Plan p;
  const cublasOperation_t opa = ta ? CUBLAS_OP_T : CUBLAS_OP_N, opb = CUBLAS_OP_N;
  lt_check(cublasLtMatmulDescCreate(&p.d, CUBLAS_COMPUTE_32I, CUDA_R_32I), "desc");
  lt_check(cublasLtMatmulDescSetAttribute(p.d, CUBLASLT_MATMUL_DESC_TRANSA, &opa, sizeof(opa)), "transa");
  lt_check(cublasLtMatmulDescSetAttribute(p.d, CUBLASLT_MATMUL_DESC_TRANSB, &opb, sizeof(opb)), "transb");
  lt_check(cublasLtMatrixLayoutCreate(&p.la, CUDA_R_8I, ta ? k : m, ta ? m : k, lda), "layout a");
  lt_check(cublasLtMatrixLayoutCreate(&p.lb, CUDA_R_8I, k, n, ldb), "layout b");
  lt_check(cublasLtMatrixLayoutCreate(&p.lc, CUDA_R_32I, m, n, ldc), "layout c");
  const std::pair<cublasLtMatrixLayout_t, int64_t> ls[3] = {{p.la, sa}, {p.lb, sb}, {p.lc, sc}};
  for (const auto& l : ls) {
    lt_check(cublasLtMatrixLayoutSetAttribute(l.first, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &batch, sizeof(batch)),
             "batch");
    lt_check(cublasLtMatrixLayoutSetAttribute(l.first, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &l.second,
                                              sizeof(l.second)),
             "stride");
  }
  cublasLtMatmulPreference_t pref;
  lt_check(cublasLtMatmulPreferenceCreate(&pref), "pref");
  lt_check(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &s.lt_ws_bytes,
                                                sizeof(s.lt_ws_bytes)),
           "pref ws");
  cublasLtMatmulHeuristicResult_t res{};
  int nres = 0;
  const cublasStatus_t st = cublasLtMatmulAlgoGetHeuristic(s.lt, p.d, p.la, p.lb, p.lc, p.lc, pref, 1, &res, &nres);
  cublasLtMatmulPreferenceDestroy(pref);
  if (st != CUBLAS_STATUS_SUCCESS || nres == 0)
    fail(QLRA_ERR_CUDA, "ozaki: no cuBLASLt int8 algorithm for " + std::to_string(m) + "x" + std::to_string(n) +
                            "x" + std::to_string(k));
  p.algo = res.algo;
  return s.plans.emplace(key, p).first->second;
}

void run_gemm(Ctx& c, OzState& s, OzState::Plan& p, const void* A, const void* B, void* C, int beta,
              void* ws = nullptr) {
  // ws: a caller-owned workspace of lt_ws_bytes (products issued on a side
  // stream must not share the context's)
  const int32_t alpha = 1;
  lt_check(cublasLtMatmul(s.lt, p.d, &alpha, A, p.la, B, p.lb, &beta, C, p.lc, C, p.lc, &p.algo,
                          ws ? ws : s.lt_ws, s.lt_ws_bytes, c.stream),
           "matmul");
  count_launch();
}

}  // namespace

void oz_release(Ctx& c) {
  OzState* s = c.oz;
  if (!s) return;
  for (auto& kv : s->plans) {
    cublasLtMatrixLayoutDestroy(kv.second.la);
    cublasLtMatrixLayoutDestroy(kv.second.lb);
    cublasLtMatrixLayoutDestroy(kv.second.lc);
    cublasLtMatmulDescDestroy(kv.second.d);
  }
  for (OzState::Buf* b : {&s->ares[0], &s->ares[1], &s->pres[0], &s->pres[1], &s->ores, &s->cy[0], &s->cy[1], &s->cw,
                          &s->stat})
    if (b->p) cudaFreeAsync(b->p, c.stream);
  cudaStreamSynchronize(c.stream);
  if (s->aux) {
    cudaStreamSynchronize(s->aux);
    cudaStreamDestroy(s->aux);
  }
  if (s->lt_ws) cudaFree(s->lt_ws);
  if (s->amax_host) cudaFreeHost(s->amax_host);
  if (s->amax_dev) cudaFree(s->amax_dev);
  if (s->lt) cublasLtDestroy(s->lt);
  delete s;
  c.oz = nullptr;
}

int64_t oz_kmax() { return KMAX; }

// which kernel runs the batched residue GEMMs of the sketch: the engine's own
// tcgen05 kernel (i8gemm.cu, the default) or cuBLASLt's IMMA kernel, kept as
// the A/B reference (QLRA_OZ_GEMM=lt; bitwise the same sketch)
bool oz_gemm_tcgen05() {
  const char* e = std::getenv("QLRA_OZ_GEMM");  // read per call: tests switch it between sketches
  if (e && std::string(e) == "lt") return false;
  return true;
}

bool oz_wanted(const Ctx& c, int64_t n, int64_t s, int64_t l) {
  if (up16(n) > KMAX || n == 0 || s == 0 || l == 0) return false;
  int engine = c.sketch_engine;
  if (engine == QLRA_SKETCH_AUTO) {
    const char* e = std::getenv("QLRA_SKETCH_ENGINE");
    if (e && std::string(e) == "int8") engine = QLRA_SKETCH_INT8;
    if (e && std::string(e) == "dmma") engine = QLRA_SKETCH_DMMA;
  }
  if (engine == QLRA_SKETCH_INT8) return true;
  if (engine == QLRA_SKETCH_DMMA) return false;
  // auto: the int8 GEMMs pay off once the products are wide (measured:
  // cuBLASLt int8 2.5-3.5 POPS at C2-C4 shapes, ~0.1 POPS at C5's n = 300)
  return n >= 2048 && s >= 64 && l >= 64;
}

ModCfg mcfg_of(const OzRun& r) { return ModCfg{r.nmod, r.tab, r.beta}; }

OzRun::OzRun(Ctx& c, const QView& om, const QView& ps, int64_t rows) : ctx(c), omega(om), psi(ps) {
  OzState& s = state(c);
  n = om.rows;
  npad = up16(n);
  npitch = up128(npad);
  // moduli: 15 (P = 2^117.2) carry every product exactly at 49-bit operand
  // scales while each int32 accumulation has K <= 2^15 terms (|X| <= K
  // 2^50 2^50 = 2^115 < P / 2): the block's rows (W^*'s K, one epoch) and n
  // (Y's K) both within 32768; else 16 (P = 2^124.7) at 52 bits with K < 2^17
  // (2^123 < P / 2).  15 moduli: 1/16 less residue traffic and int8 work,
  // operands rounded at 2^-50 of their maxima instead of 2^-53.
  static const bool force16 = [] {
    const char* e = std::getenv("QLRA_OZ_MODULI");
    return e && std::atoi(e) == 16;
  }();
  if (!force16 && npad <= 32768 && rows <= 32768) {
    nmod = 15;
    tab = 1;
    beta = 49;
    kcap = 32768;
  } else {
    nmod = 16;
    tab = 0;
    beta = 52;
    kcap = KMAX;
  }
  nb = 8 * nmod;
  scols = om.cols;
  spad = up16(scols);  // cuBLASLt's IMMA kernels want 16-aligned m and n
  l = ps.rows;
  lpad = up16(l);
  // maxima: Omega columns, then Psi rows
  auto* st = static_cast<unsigned long long*>(grow(c, s.stat, sizeof(unsigned long long) * (size_t)(scols + l + 1)));
  QLRA_CUDA(cudaMemsetAsync(st, 0, sizeof(unsigned long long) * (size_t)(scols + l + 1), c.stream));
  om_colmax = st;
  ps_rowmax = st + scols;
  {
    dim3 grid((unsigned)((scols + 31) / 32), (unsigned)std::min<int64_t>(64, (n + 7) / 8));
    k_colmax<<<grid, 256, 0, c.stream>>>(om, om_colmax);
    QLRA_LAUNCH_CHECK();
    count_launch();
  }
  if (l > 0 && ps.cols > 0) {
    k_rowmax<<<(unsigned)l, 256, 0, c.stream>>>(ps, ps_rowmax);
    QLRA_LAUNCH_CHECK();
    count_launch();
  }
  ores = static_cast<int8_t*>(grow(c, s.ores, (size_t)nb * spad * npitch));
  k_res_om<<<blocks_for(spad * (npad / 4), 256), 256, 0, c.stream>>>(om, om_colmax, npad, spad, ores, npitch, spad * npitch,
                                                                      mcfg_of(*this));
  QLRA_LAUNCH_CHECK();
  count_launch();
  cw = static_cast<int32_t*>(grow(c, s.cw, sizeof(int32_t) * (size_t)nb * npad * lpad));
}

// max |A| of a view on `stream`, into panel slot `slot` (device) and its
// pinned host copy
void OzRun::amax_async(const QView& a, cudaStream_t stream, int slot) {
  OzState& s = *ctx.oz;
  unsigned long long* d = s.amax_dev + slot;
  QLRA_CUDA(cudaMemsetAsync(d, 0, sizeof(*d), stream));
  const int64_t total = a.rows * a.cols;
  if (total > 0) {
    k_absmax<<<(unsigned)std::min<int64_t>(148 * 8, (total + 255) / 256), 256, 0, stream>>>(a, d);
    QLRA_LAUNCH_CHECK();
    count_launch();
  }
  QLRA_CUDA(cudaMemcpyAsync(s.amax_host + slot, d, sizeof(*d), cudaMemcpyDeviceToHost, stream));
}
double OzRun::amax_host(int slot) const {
  const unsigned long long b = ctx.oz->amax_host[slot];
  double d;
  std::memcpy(&d, &b, sizeof(d));
  return d;
}

void OzRun::flush(const QView& w) {
  if (!epoch_open) return;
  if (epoch_rows > 0 && w.rows > 0 && w.cols > 0) {
    k_crt_w<<<blocks_for(w.rows * w.cols, 128), 128, 0, ctx.stream>>>(cw, npad * lpad, npad, w, ps_rowmax, sigma,
                                                                       mcfg_of(*this));
    QLRA_LAUNCH_CHECK();
    count_launch();
  }
  epoch_open = false;
  epoch_rows = 0;
}

// Epoch bookkeeping for a panel of rpad rows whose max |A| is amax: flush
// W^*'s products first when the panel would leave the open epoch's range.
void OzRun::open_for(int64_t rpad, double amax, int headroom, const QView& w) {
  if (rpad > kcap) fail(QLRA_ERR_PARAMETER, "ozaki: panel taller than the int32 accumulation bound");
  const int e = std::ilogb(amax);
  if (epoch_open && (e + sigma > beta - 1 || epoch_rows + rpad > kcap)) flush(w);
  if (!epoch_open) {
    sigma = beta - 1 - e - headroom;
    epoch_open = true;
    epoch_rows = 0;
  }
}

// Residues of a panel (A rows [pc0, pc0 + R), Psi columns likewise) into
// residue buffer `buf`, on `st`.
void OzRun::prep(int64_t pc0, const QView& ap, int buf, cudaStream_t st) {
  OzState& s = *ctx.oz;
  const int64_t R = ap.rows, rpad = up16(R);
  auto* ares = static_cast<int8_t*>(s.ares[buf].p);
  k_res_a<<<blocks_for(rpad * (npad / 4), 128), 128, 0, st>>>(ap, npad, rpad, sigma, ares, npitch, rpad * npitch, nmod);
  QLRA_LAUNCH_CHECK();
  count_launch();
  if (l > 0) {
    k_res_psi<<<blocks_for(lpad * (rpad / 4), 128), 128, 0, st>>>(
        psi, pc0, R, rpad, lpad, ps_rowmax, static_cast<int8_t*>(s.pres[buf].p), up128(rpad), lpad * up128(rpad),
        mcfg_of(*this));
    QLRA_LAUNCH_CHECK();
    count_launch();
  }
}

// Grow the panel buffers of slot `buf` for panels of up to rpad rows (on
// the context stream: before any other stream touches them).
void OzRun::reserve(int64_t rpad, int buf) {
  OzState& s = *ctx.oz;
  grow(ctx, s.ares[buf], (size_t)nb * rpad * npitch);
  if (l > 0) grow(ctx, s.pres[buf], (size_t)nb * lpad * up128(rpad));
  if (scols > 0) grow(ctx, s.cy[buf], sizeof(int32_t) * (size_t)nb * rpad * spad);
}

// The two batched GEMMs of a prepared panel (context stream; bench timed).
void OzRun::gemms(int64_t R, int buf) {
  OzState& s = *ctx.oz;
  const int64_t rpad = up16(R), rpitch = up128(rpad);
  LaunchTimer lt(ctx);
  if (oz_gemm_tcgen05()) {
    // the engine's own tcgen05 kernel (i8gemm.cu): both products straight
    // from the row-major residue panel
    const auto* ar = static_cast<const int8_t*>(s.ares[buf].p);
    // CTA pairs (tcgen05.mma.cta_group::2) at every size: with the siblings'
    // tile-row rendezvous they beat the 1-CTA form on C2-C4 (DESIGN 3)
    const int ctas = 2;
    // Y panel: cy[b][i][j] = sum_k Ares[b][i][k] Ores[b][j][k]
    if (scols > 0)
      i8gemm_batched(ctx, 0, rpad, spad, npad, ar, npitch, rpad * npitch, ores, npitch, spad * npitch,
                     static_cast<int32_t*>(s.cy[buf].p), spad, rpad * spad, nb, 0, ctx.stream, ctas);
    // W^*: cw[b][k][j] += sum_i Ares[b][i][j] Pres[b][k][i]
    if (l > 0)
      i8gemm_batched(ctx, 1, npad, lpad, rpad, ar, npitch, rpad * npitch, static_cast<const int8_t*>(s.pres[buf].p),
                     rpitch, lpad * rpitch, cw, npad, npad * lpad, nb, epoch_rows > 0 ? 1 : 0, ctx.stream, ctas);
  } else {
    // Y panel: col-major C (s x Rpad, ldc spad) = Ores^T (s x npad) * Ares (npad x Rpad)
    if (scols > 0) {
      OzState::Plan& py = plan(s, true, spad, rpad, npad, npitch, npitch, spad, spad * npitch, rpad * npitch, rpad * spad, nb);
      run_gemm(ctx, s, py, ores, s.ares[buf].p, s.cy[buf].p, 0);
    }
    // W^* (npad x l, ldc npad) += Ares (npad x Rpad) * Pres (Rpad x l)
    if (l > 0) {
      OzState::Plan& pw = plan(s, false, npad, lpad, rpad, npitch, rpitch, npad, rpad * npitch, lpad * rpitch, npad * lpad, nb);
      run_gemm(ctx, s, pw, s.ares[buf].p, s.pres[buf].p, cw, epoch_rows > 0 ? 1 : 0);
    }
  }
  lt.close(32.0 * (double)R * (double)n * (double)(scols + l), 32.0 * (double)R * (double)n,
           2.0 * nb * (double)rpad * (double)npad * (double)(scols + l), 2);
  epoch_rows += rpad;
}

// Y rows of a panel += its recovered products (on `st`).
void OzRun::recover_y(const QView& yr, int buf, cudaStream_t st) {
  if (scols == 0 || yr.rows == 0) return;
  OzState& s = *ctx.oz;
  const int64_t rpad = up16(yr.rows);
  k_crt_y<<<blocks_for(yr.rows * scols, 128), 128, 0, st>>>(static_cast<const int32_t*>(s.cy[buf].p), rpad * spad,
                                                            spad, yr, om_colmax, sigma, mcfg_of(*this));
  QLRA_LAUNCH_CHECK();
  count_launch();
}

// One row panel, all on the context stream (the row pipeline's chunks):
// A rows [pc0, pc0 + R) of the block, Y rows of the panel, W of the block;
// amax = max |A| over the panel (or an upper bound).
void OzRun::panel(int64_t pc0, const QView& ap, const QView& yr, const QView& w, double amax, int headroom) {
  const int64_t R = ap.rows;
  if (R == 0 || amax == 0.0) return;  // an all-zero panel adds nothing
  const int64_t rpad = up16(R);
  open_for(rpad, amax, headroom, w);
  reserve(rpad, 0);
  prep(pc0, ap, 0, ctx.stream);
  gemms(R, 0);
  recover_y(yr, 0, ctx.stream);
}

void OzRun::finish(const QView& w) { flush(w); }

// Whole device-resident block: one scan for max |A| (a single epoch unless
// the block is taller than one int32 accumulation), then panels sized for
// the residue buffers, software-pipelined over two streams: the residues of
// panel p+1 (k_res_a, k_res_psi: HBM / FP64-pipe work) and the recovery of
// panel p-1's Y rows run on an auxiliary stream while panel p's GEMMs hold
// the tensor cores; two residue / product buffers alternate.
bool oz_sketch_block(Ctx& c, const QView& om, const QView& ps, const QView& block, const QView& y_rows,
                     const QView& w) {
  OzRun run(c, om, ps, block.rows);
  run.amax_async(block, c.stream, 2);
  QLRA_CUDA(cudaStreamSynchronize(c.stream));
  const double amax = run.amax_host(2);
  // NaN / inf in A: no fixed-point image -- the caller runs the FP64 engine,
  // which propagates them as the reference's products do
  if (!std::isfinite(amax)) return false;
  if (amax == 0.0 || block.rows == 0) return true;
  // residue panels: as tall as memory allows (each panel re-reads and
  // re-writes W^*'s int32 products inside its GEMM), capped by
  // QLRA_OZ_PANEL_BYTES (default 28 GB) and 45% of the free memory (22% per
  // buffer when pipelined: two of them)
  static const bool pipelined = [] {
    const char* e = std::getenv("QLRA_OZ_PIPELINE");
    return e && std::atoi(e) != 0;
  }();
  static const double cap = [] {
    const char* e = std::getenv("QLRA_OZ_PANEL_BYTES");
    return e ? std::atof(e) : 28e9;
  }();
  size_t free_b = 0, total_b = 0;
  QLRA_CUDA(cudaMemGetInfo(&free_b, &total_b));
  {
    // memory the context's stream-ordered pool holds but no allocation uses
    // (its release threshold keeps freed blocks reserved) is available too
    cudaMemPool_t pool = nullptr;
    cuuint64_t reserved = 0, used = 0;
    if (cudaDeviceGetDefaultMemPool(&pool, c.device) == cudaSuccess &&
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && reserved > used)
      free_b += (size_t)(reserved - used);
    cudaGetLastError();
  }
  const double budget = std::max(0.5e9, std::min(cap, (pipelined ? 0.22 : 0.45) * (double)free_b));
  int64_t R = (int64_t)(budget / (run.nb * (double)run.npitch));
  R = std::max<int64_t>(256, std::min<int64_t>(R / 16 * 16, run.kcap));
  const int64_t np = (block.rows + R - 1) / R;  // equal panels (no short tail)
  R = up16((block.rows + np - 1) / np);
  if (!pipelined) {
    // sequential panels on the context stream (measured on C4: the power
    // cap makes the overlapped residues cost the GEMMs' clock, 0.249 vs 0.261 s)
    for (int64_t r0 = 0; r0 < block.rows; r0 += R) {
      const int64_t rp = std::min(R, block.rows - r0);
      run.panel(r0, sub(block, r0, 0, rp, block.cols), sub(y_rows, r0, 0, rp, y_rows.cols), w, amax, 0);
    }
    run.finish(w);
    return true;
  }
  const int nbuf = np > 1 ? 2 : 1;
  for (int b = 0; b < nbuf; ++b) run.reserve(R, b);
  OzState& s = *c.oz;
  if (!s.aux) QLRA_CUDA(cudaStreamCreateWithFlags(&s.aux, cudaStreamNonBlocking));
  // events: residues of buffer b ready / buffer b's GEMMs done / its Y recovered
  struct Ev {
    cudaEvent_t e[6] = {};
    Ev() {
      for (auto& x : e) QLRA_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    }
    ~Ev() {
      for (auto& x : e)
        if (x) cudaEventDestroy(x);
    }
  } ev;
  cudaEvent_t* ready = ev.e;
  cudaEvent_t* gemmed = ev.e + 2;
  cudaEvent_t* recovered = ev.e + 4;
  struct Join {  // the context stream waits for the aux stream on every exit
    Ctx& c;
    cudaStream_t aux;
    cudaEvent_t e;
    ~Join() {
      if (cudaEventRecord(e, aux) == cudaSuccess) cudaStreamWaitEvent(c.stream, e, 0);
      cudaStreamSynchronize(aux);
    }
  };
  cudaEvent_t join_ev;
  QLRA_CUDA(cudaEventCreateWithFlags(&join_ev, cudaEventDisableTiming));
  {
    Join join{c, s.aux, join_ev};
    // the aux stream starts after everything queued so far (buffers, Omega's residues)
    QLRA_CUDA(cudaEventRecord(ready[0], c.stream));
    QLRA_CUDA(cudaStreamWaitEvent(s.aux, ready[0], 0));
    run.open_for(R, amax, 0, w);
    int64_t prev_r0 = -1;
    for (int64_t p = 0, r0 = 0; r0 < block.rows; ++p, r0 += R) {
      const int b = (int)(p % nbuf);
      const int64_t rp = std::min(R, block.rows - r0);
      if (p >= nbuf) {
        // buffer b was last used by panel p - nbuf: its GEMMs and Y recovery first
        QLRA_CUDA(cudaStreamWaitEvent(s.aux, gemmed[b], 0));
      }
      run.prep(r0, sub(block, r0, 0, rp, block.cols), b, s.aux);
      QLRA_CUDA(cudaEventRecord(ready[b], s.aux));
      if (prev_r0 >= 0) {
        // Y rows of the previous panel, on aux behind this panel's residues
        const int pb = (int)((p - 1) % nbuf);
        const int64_t prp = std::min(R, block.rows - prev_r0);
        QLRA_CUDA(cudaStreamWaitEvent(s.aux, gemmed[pb], 0));
        run.recover_y(sub(y_rows, prev_r0, 0, prp, y_rows.cols), pb, s.aux);
        QLRA_CUDA(cudaEventRecord(recovered[pb], s.aux));
      }
      QLRA_CUDA(cudaStreamWaitEvent(c.stream, ready[b], 0));
      if (p >= nbuf) QLRA_CUDA(cudaStreamWaitEvent(c.stream, recovered[b], 0));  // cy[b] read
      // more rows than one int32 accumulation: recover W and start a new
      // epoch (same scale: the block's max)
      run.open_for(up16(rp), amax, 0, w);
      run.gemms(rp, b);
      QLRA_CUDA(cudaEventRecord(gemmed[b], c.stream));
      prev_r0 = r0;
    }
    // the last panel's Y rows
    const int pb = (int)((np - 1) % nbuf);
    run.recover_y(sub(y_rows, prev_r0, 0, std::min(R, block.rows - prev_r0), y_rows.cols), pb, c.stream);
  }
  cudaEventDestroy(join_ev);
  run.finish(w);
  return true;
}

// ---------------------------------------------------------------------------
// General quaternion product on the int8 engine, for the large-K products of
// the QB stage (Psi H, Psi Q0 -- sketching.cpp:184 -- and the Grams H^* H of
// the rangefinders, rangefinders.cpp:68,102): C = alpha op(A) op(B) + beta C,
// exact integer products of per-row (left) / per-column (right) 52-bit
// images, K in chunks of < 2^17 (int32), each chunk recovered and added.
// Every buffer is allocated on the calling stream (the early core solve
// issues its products on a second stream).
bool oz_gemm_try(Ctx& c, int op_a, int op_b, double alpha, const QView& A, const QView& B, double beta,
                 const QView& C) {
  const int64_t M = C.rows, N = C.cols, K = op_a ? A.rows : A.cols;
  if (M == 0 || N == 0 || K == 0) return false;
  int engine = c.sketch_engine;
  if (engine == QLRA_SKETCH_AUTO) {
    const char* e = std::getenv("QLRA_SKETCH_ENGINE");
    if (e && std::string(e) == "dmma") engine = QLRA_SKETCH_DMMA;
  }
  if (engine == QLRA_SKETCH_DMMA) return false;
  // worth it when the contraction is long and the output not tiny: the
  // residues cost ~(M + N) K, the recovery ~M N (128 int32 reads + the CRT
  // per element), the DMMA product 16 M N K flop
  if (K < 4096 || M < 64 || N < 64 || (double)M * (double)N * (double)K < 1.5e9) return false;
  OzState& s = state(c);
  const bool same = A.p[0] == B.p[0] && A.rows == B.rows && A.cols == B.cols && op_a == QLRA_OP_C && op_b == QLRA_OP_N;
  // K-major rows: L (M x K) = op(A), R (N x K) = op(B)^T
  DevQMat lt, rt;
  auto transpose = [&](const QView& x, DevQMat& out) {
    out = DevQMat(c, x.cols, x.rows);
    k_transpose<<<dim3((unsigned)((x.cols + 31) / 32), (unsigned)((x.rows + 31) / 32)), dim3(32, 8), 0, c.stream>>>(
        x, out.v);
    QLRA_LAUNCH_CHECK();
    count_launch();
    return out.v;
  };
  const QView L = op_a == QLRA_OP_N ? A : transpose(A, lt);
  const int lconj = op_a == QLRA_OP_N ? 0 : 1;
  const QView R = op_b == QLRA_OP_C ? B : (same ? L : transpose(B, rt));
  const int rconj = op_b == QLRA_OP_C ? 1 : 0;
  const int64_t mpad = up16(M), npad = up16(N);
  DeviceBuffer mx(c, sizeof(unsigned long long) * (size_t)(M + N));
  auto* lmax = mx.as<unsigned long long>();
  auto* rmax = lmax + M;
  k_rowmax<<<(unsigned)M, 256, 0, c.stream>>>(L, lmax);
  QLRA_LAUNCH_CHECK();
  count_launch();
  if (same) {
    QLRA_CUDA(cudaMemcpyAsync(rmax, lmax, sizeof(unsigned long long) * (size_t)M, cudaMemcpyDeviceToDevice, c.stream));
  } else {
    k_rowmax<<<(unsigned)N, 256, 0, c.stream>>>(R, rmax);
    QLRA_LAUNCH_CHECK();
    count_launch();
  }
  const bool tc05 = oz_gemm_tcgen05();
  // K pad: whole 128-byte residue rows for the tcgen05 kernel's TMA boxes (the pad is zero)
  const int64_t nch = (K + KMAX - 1) / KMAX, kc = (K + nch - 1) / nch, kpad = tc05 ? up128(kc) : up16(kc);
  DeviceBuffer lres(c, (size_t)NB * mpad * kpad), rres(c, (size_t)NB * npad * kpad);
  DeviceBuffer ci(c, sizeof(int32_t) * (size_t)NB * mpad * npad), ws(c, tc05 ? 0 : s.lt_ws_bytes);
  // col-major C (npad x mpad) = Rres^T (npad x kpad) * Lres (kpad x mpad)
  OzState::Plan* pl = tc05 ? nullptr
                           : &plan(s, true, npad, mpad, kpad, kpad, kpad, npad, npad * kpad, mpad * kpad, mpad * npad, NB);
  for (int64_t ch = 0; ch < nch; ++ch) {
    const int64_t k0 = ch * kc, kn = std::min(kc, K - k0);
    k_res_rows<true><<<blocks_for(mpad * (kpad / 4), 128), 128, 0, c.stream>>>(L, lconj, lmax, k0, kn, kpad, mpad,
                                                                               lres.as<int8_t>(), mpad * kpad);
    QLRA_LAUNCH_CHECK();
    k_res_rows<false><<<blocks_for(npad * (kpad / 4), 128), 128, 0, c.stream>>>(R, rconj, rmax, k0, kn, kpad, npad,
                                                                                rres.as<int8_t>(), npad * kpad);
    QLRA_LAUNCH_CHECK();
    count_launch();
    count_launch();
    if (tc05)  // ci[b][m][n] = sum_k Lres[b][m][k] Rres[b][n][k]
      i8gemm_batched(c, 0, mpad, npad, kpad, lres.as<int8_t>(), kpad, mpad * kpad, rres.as<int8_t>(), kpad,
                     npad * kpad, ci.as<int32_t>(), npad, mpad * npad, NB, 0, c.stream);
    else
      run_gemm(c, s, *pl, rres.ptr, lres.ptr, ci.ptr, 0, ws.ptr);
    k_crt_gen<<<blocks_for(M * N, 128), 128, 0, c.stream>>>(ci.as<int32_t>(), mpad * npad, npad, C, lmax, rmax,
                                                             alpha, ch == 0 ? beta : 1.0);
    QLRA_LAUNCH_CHECK();
    count_launch();
  }
  return true;
}

// INT8 tensor-core peak of this GPU as the engine sees it: back-to-back
// cuBLASLt int8 GEMMs of 8192^3 (the roofline denominator of the int8
// engine's GEMMs, measured in the same run as them).
double oz_measure_int8_peak(Ctx& c, double ms) {
  OzState& s = state(c);
  const int64_t N = 8192;
  DeviceBuffer a(c, (size_t)N * N), b(c, (size_t)N * N), d(c, sizeof(int32_t) * (size_t)N * N);
  QLRA_CUDA(cudaMemsetAsync(a.ptr, 1, (size_t)N * N, c.stream));
  QLRA_CUDA(cudaMemsetAsync(b.ptr, 1, (size_t)N * N, c.stream));
  OzState::Plan& p = plan(s, true, N, N, N, N, N, N, N * N, N * N, N * N, 1);
  for (int i = 0; i < 3; ++i) run_gemm(c, s, p, a.ptr, b.ptr, d.ptr, 0);
  cudaEvent_t e0, e1;
  QLRA_CUDA(cudaEventCreate(&e0));
  QLRA_CUDA(cudaEventCreate(&e1));
  QLRA_CUDA(cudaEventRecord(e0, c.stream));
  run_gemm(c, s, p, a.ptr, b.ptr, d.ptr, 0);
  QLRA_CUDA(cudaEventRecord(e1, c.stream));
  QLRA_CUDA(cudaEventSynchronize(e1));
  float one = 0.f;
  QLRA_CUDA(cudaEventElapsedTime(&one, e0, e1));
  const int reps = std::max(1, (int)(ms / std::max(0.01f, one)));
  QLRA_CUDA(cudaEventRecord(e0, c.stream));
  for (int i = 0; i < reps; ++i) run_gemm(c, s, p, a.ptr, b.ptr, d.ptr, 0);
  QLRA_CUDA(cudaEventRecord(e1, c.stream));
  QLRA_CUDA(cudaEventSynchronize(e1));
  float t = 0.f;
  QLRA_CUDA(cudaEventElapsedTime(&t, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return 2.0 * N * N * (double)N * reps / (t * 1e-3) / 1e12;
}

const char* oz_kernel_name() {
  return oz_gemm_tcgen05()
             ? "int8 tensor-core sketch (Ozaki/CRT: 15-16 moduli x 8 combinations; residue GEMMs on the engine's own "
               "tcgen05 kernel i8gemm_tc05[_2sm]_kernel: TMA ring, tcgen05.mma kind::i8, TMEM accumulators, TMA "
               "store / reduce-add epilogue; + residue/CRT kernels)"
             : "int8 tensor-core sketch (Ozaki/CRT: 15-16 moduli x 8 combinations, cuBLASLt sm_100 IMMA batched GEMM "
               "[QLRA_OZ_GEMM=lt] + residue/CRT kernels)";
}

}  // namespace qlra_dev
