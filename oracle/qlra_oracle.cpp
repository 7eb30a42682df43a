// qlra_oracle.cpp -- TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference `qlra` one-pass hot path (arXiv 2404.14783,
// C++ reference under /root/reference/proj).  It is the parity checker for the
// B200 product in paper_2404_14783_b200/: only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it.  Nothing in
// the product links or calls it.
//
// Why a restatement: the reference needs Eigen 3.4 (proj/src/CMakeLists.txt:1)
// which is absent here, so it cannot be compiled.  The integer /
// sketch arithmetic below follows the reference loops statement for statement
// (bit-identical results when built without FMA contraction, as the reference
// is: proj/CMakeLists.txt:8-10 has no -march); the dense complex factorizations
// replace Eigen with LP64 LAPACK (OpenBLAS bundled in the venv):
//   Eigen::HouseholderQR          -> zgeqrf + zungqr   (+ same phase fix)
//   Eigen::BDCSVD (thin)          -> zgesdd 'S'
//   Eigen::PartialPivLU + rcond() -> zgetrf + zgecon('1') + zgetrs
//   Eigen::ColPivHouseholderQR    -> zgeqp3 + zunmqr + ztrsm
//   Eigen dense real products     -> dgemm
// Results across that boundary match the reference to rounding only; no
// reference test pins bits there.
//
// Parity pinning: the RNG and quaternion product table are checked against
// the reference's own rng.hpp / quaternion.hpp compiled in place (oracle/_ref,
// tests/golden/ref_kat.json); everything else is pinned by the reference's
// known-answer and property tests ported to tests/test_oracle_*.py.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

using cd = std::complex<double>;
using Index = std::int64_t;

// ---------------------------------------------------------------- LAPACK ---
extern "C" {
void zgeqrf_(const int* m, const int* n, cd* a, const int* lda, cd* tau, cd* work,
             const int* lwork, int* info);
void zungqr_(const int* m, const int* n, const int* k, cd* a, const int* lda,
             const cd* tau, cd* work, const int* lwork, int* info);
void zgesdd_(const char* jobz, const int* m, const int* n, cd* a, const int* lda, double* s,
             cd* u, const int* ldu, cd* vt, const int* ldvt, cd* work, const int* lwork,
             double* rwork, int* iwork, int* info, std::size_t);
void zgetrf_(const int* m, const int* n, cd* a, const int* lda, int* ipiv, int* info);
void zgetrs_(const char* trans, const int* n, const int* nrhs, const cd* a, const int* lda,
             const int* ipiv, cd* b, const int* ldb, int* info, std::size_t);
void zgecon_(const char* norm, const int* n, const cd* a, const int* lda, const double* anorm,
             double* rcond, cd* work, double* rwork, int* info, std::size_t);
double zlange_(const char* norm, const int* m, const int* n, const cd* a, const int* lda,
               double* work, std::size_t);
void zgeqp3_(const int* m, const int* n, cd* a, const int* lda, int* jpvt, cd* tau, cd* work,
             const int* lwork, double* rwork, int* info);
void zunmqr_(const char* side, const char* trans, const int* m, const int* n, const int* k,
             const cd* a, const int* lda, const cd* tau, cd* c, const int* ldc, cd* work,
             const int* lwork, int* info, std::size_t, std::size_t);
void ztrsm_(const char* side, const char* uplo, const char* transa, const char* diag,
            const int* m, const int* n, const cd* alpha, const cd* a, const int* lda, cd* b,
            const int* ldb, std::size_t, std::size_t, std::size_t, std::size_t);
void openblas_set_num_threads(int);
int openblas_get_num_threads(void);
void dgemm_(const char* ta, const char* tb, const int* m, const int* n, const int* k,
            const double* alpha, const double* a, const int* lda, const double* b,
            const int* ldb, const double* beta, double* c, const int* ldc, std::size_t,
            std::size_t);
void zgemm_(const char* ta, const char* tb, const int* m, const int* n, const int* k,
            const cd* alpha, const cd* a, const int* lda, const cd* b, const int* ldb,
            const cd* beta, cd* c, const int* ldc, std::size_t, std::size_t);
}

namespace orc {

// ---------------------------------------------------------------- errors ---
// Mirrors proj/include/qlra/errors.hpp:9-43; codes match include/qlra_cuda.h.
enum Status { kOk = 0, kShape = 1, kParameter = 2, kSingular = 3, kRank = 4,
              kPrecondition = 5, kIo = 6, kInternal = 99 };
struct Error : std::runtime_error {
  int code;
  double cond = 0.0;
  Error(int c, const std::string& m, double k = 0.0) : std::runtime_error(m), code(c), cond(k) {}
};
[[noreturn]] void shape(const std::string& m) { throw Error(kShape, m); }
[[noreturn]] void param(const std::string& m) { throw Error(kParameter, m); }
[[noreturn]] void rank_err(const std::string& m) { throw Error(kRank, m); }
[[noreturn]] void singular(const std::string& m, double c) {
  throw Error(kSingular, m + " (estimated condition " + std::to_string(c) + ")", c);
}

// ------------------------------------------------------------------- RNG ---
// proj/include/qlra/rng.hpp:10-76
constexpr std::uint64_t mix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
struct CounterRng {
  static constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
  static constexpr std::uint64_t kSalt = 0xD1B54A32D192ED03ULL;
  std::uint64_t key;
  explicit CounterRng(std::uint64_t seed) : key(mix64(seed ^ kSalt)) {}
  CounterRng substream(std::uint64_t index) const {
    CounterRng c(0);
    c.key = mix64(key ^ mix64(index + kSalt));
    return c;
  }
  std::uint64_t u64_at(std::uint64_t c) const { return mix64(key + kGolden * (c + 1)); }
  double uniform_at(std::uint64_t c) const {
    return static_cast<double>(u64_at(c) >> 11) * 0x1.0p-53;
  }
};
struct SequentialRng {
  CounterRng stream;
  std::uint64_t counter = 0;
  explicit SequentialRng(CounterRng s) : stream(s) {}
  std::uint64_t next_u64() { return stream.u64_at(counter++); }
  double next_uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double next_gaussian() {
    const double u1 = next_uniform();
    const double u2 = next_uniform();
    return std::sqrt(-2.0 * std::log1p(-u1)) * std::cos(2.0 * M_PI * u2);
  }
};

// --------------------------------------------------------------- QMatrix ---
// proj/include/qlra/qmatrix.hpp:17-84: four contiguous row-major planes.
struct QM {
  Index rows = 0, cols = 0;
  std::vector<double> p[4];
  QM() = default;
  QM(Index r, Index c) : rows(r), cols(c) {
    for (auto& v : p) v.assign(static_cast<std::size_t>(r * c), 0.0);
  }
  double& at(int pl, Index i, Index j) { return p[pl][i * cols + j]; }
  double at(int pl, Index i, Index j) const { return p[pl][i * cols + j]; }
  void get(Index i, Index j, double q[4]) const {
    for (int k = 0; k < 4; ++k) q[k] = at(k, i, j);
  }
  void set(Index i, Index j, const double q[4]) {
    for (int k = 0; k < 4; ++k) at(k, i, j) = q[k];
  }
  static QM identity(Index n) {
    QM m(n, n);
    for (Index i = 0; i < n; ++i) m.at(0, i, i) = 1.0;
    return m;
  }
  QM adjoint() const {  // qmatrix.cpp:42-52
    QM r(cols, rows);
    for (Index i = 0; i < rows; ++i)
      for (Index j = 0; j < cols; ++j) {
        r.at(0, j, i) = at(0, i, j);
        r.at(1, j, i) = -at(1, i, j);
        r.at(2, j, i) = -at(2, i, j);
        r.at(3, j, i) = -at(3, i, j);
      }
    return r;
  }
  double fro_norm() const {  // qmatrix.cpp:61-67
    double s = 0.0;
    for (const auto& pl : p)
      for (double v : pl) s += v * v;
    return std::sqrt(s);
  }
  void scale_col(Index j, const double q[4]) {  // v <- v q  (qmatrix.cpp:128-130)
    for (Index i = 0; i < rows; ++i) {
      double a[4];
      get(i, j, a);
      const double r[4] = {a[0] * q[0] - a[1] * q[1] - a[2] * q[2] - a[3] * q[3],
                           a[0] * q[1] + a[1] * q[0] + a[2] * q[3] - a[3] * q[2],
                           a[0] * q[2] - a[1] * q[3] + a[2] * q[0] + a[3] * q[1],
                           a[0] * q[3] + a[1] * q[2] - a[2] * q[1] + a[3] * q[0]};
      set(i, j, r);
    }
  }
  void scale_col(Index j, double s) {  // qmatrix.cpp:132-134 (Quaternion * double)
    for (Index i = 0; i < rows; ++i)
      for (int k = 0; k < 4; ++k) at(k, i, j) = at(k, i, j) * s;
  }
};

QM operator+(const QM& a, const QM& b) {
  if (a.rows != b.rows || a.cols != b.cols) shape("add: shape mismatch");
  QM r = a;
  for (int k = 0; k < 4; ++k)
    for (std::size_t i = 0; i < r.p[k].size(); ++i) r.p[k][i] += b.p[k][i];
  return r;
}
QM operator-(const QM& a, const QM& b) {
  if (a.rows != b.rows || a.cols != b.cols) shape("sub: shape mismatch");
  QM r = a;
  for (int k = 0; k < 4; ++k)
    for (std::size_t i = 0; i < r.p[k].size(); ++i) r.p[k][i] -= b.p[k][i];
  return r;
}
QM operator*(double s, const QM& a) {
  QM r = a;
  for (auto& pl : r.p)
    for (auto& v : pl) v *= s;
  return r;
}

// qmat_mul: 16 real plane GEMMs (qmatrix.cpp:165-197), dgemm in place of Eigen.
// Row-major C = A B is column-major C^T = B^T A^T.
QM qmat_mul(const QM& a, const QM& b) {
  if (a.cols != b.rows) shape("qmat_mul: inner dimensions differ");
  QM c(a.rows, b.cols);
  if (c.rows == 0 || c.cols == 0) return c;
  if (a.cols == 0) return c;
  const int m = static_cast<int>(b.cols), n = static_cast<int>(a.rows),
            k = static_cast<int>(a.cols);
  auto gemm = [&](int cp, int ap, int bp, double alpha, double beta) {
    dgemm_("N", "N", &m, &n, &k, &alpha, b.p[bp].data(), &m, a.p[ap].data(), &k, &beta,
           c.p[cp].data(), &m, 1, 1);
  };
  gemm(0, 0, 0, 1, 0); gemm(0, 1, 1, -1, 1); gemm(0, 2, 2, -1, 1); gemm(0, 3, 3, -1, 1);
  gemm(1, 0, 1, 1, 0); gemm(1, 1, 0, 1, 1); gemm(1, 2, 3, 1, 1); gemm(1, 3, 2, -1, 1);
  gemm(2, 0, 2, 1, 0); gemm(2, 1, 3, -1, 1); gemm(2, 2, 0, 1, 1); gemm(2, 3, 1, 1, 1);
  gemm(3, 0, 3, 1, 0); gemm(3, 1, 2, 1, 1); gemm(3, 2, 1, -1, 1); gemm(3, 3, 0, 1, 1);
  return c;
}

// qmat_mul_accumulate_ordered (qmatrix.cpp:203-242): fixed i-k-j loop with a
// k-ascending accumulation per entry.  Rows of C are independent, so splitting
// the i range across threads leaves every entry's operation order (and hence
// its bits) unchanged.
void qmat_mul_accumulate_ordered(QM& c, const QM& a, const QM& b, int nthreads = 1) {
  if (a.cols != b.rows) shape("qmat_mul_accumulate_ordered: inner dimensions differ");
  if (c.rows != a.rows || c.cols != b.cols)
    shape("qmat_mul_accumulate_ordered: output shape mismatch");
  const Index m = a.rows, kk = a.cols, n = b.cols;
  const double *aw = a.p[0].data(), *ax = a.p[1].data(), *ay = a.p[2].data(),
               *az = a.p[3].data();
  const double *bw = b.p[0].data(), *bx = b.p[1].data(), *by = b.p[2].data(),
               *bz = b.p[3].data();
  double *cw = c.p[0].data(), *cx = c.p[1].data(), *cy = c.p[2].data(), *cz = c.p[3].data();
  auto rows = [&](Index i0, Index i1) {
    for (Index i = i0; i < i1; ++i) {
      double* cwr = cw + i * n;
      double* cxr = cx + i * n;
      double* cyr = cy + i * n;
      double* czr = cz + i * n;
      for (Index k = 0; k < kk; ++k) {
        const double qw = aw[i * kk + k], qx = ax[i * kk + k], qy = ay[i * kk + k],
                     qz = az[i * kk + k];
        const double* bwr = bw + k * n;
        const double* bxr = bx + k * n;
        const double* byr = by + k * n;
        const double* bzr = bz + k * n;
        for (Index j = 0; j < n; ++j) {
          cwr[j] += qw * bwr[j] - qx * bxr[j] - qy * byr[j] - qz * bzr[j];
          cxr[j] += qw * bxr[j] + qx * bwr[j] + qy * bzr[j] - qz * byr[j];
          cyr[j] += qw * byr[j] - qx * bzr[j] + qy * bwr[j] + qz * bxr[j];
          czr[j] += qw * bzr[j] + qx * byr[j] - qy * bxr[j] + qz * bwr[j];
        }
      }
    }
  };
  if (nthreads <= 1 || m < 2 * nthreads) {
    rows(0, m);
    return;
  }
  std::vector<std::thread> ts;
  for (int t = 0; t < nthreads; ++t)
    ts.emplace_back(rows, m * t / nthreads, m * (t + 1) / nthreads);
  for (auto& t : ts) t.join();
}

// ------------------------------------------------------- test matrices ---
// proj/src/sketching.cpp:19-108
enum Kind { kGaussian = 0, kRademacher = 1, kSparseGaussian = 2, kSparseRademacher = 3 };
struct Spec {
  int kind = kGaussian;
  Index rows = 0, cols = 0;
  std::uint64_t seed = 0;
  double density = 1.0;
};

double entry_value(const CounterRng& stream, int kind, double density, std::uint64_t idx) {
  const std::uint64_t base = 4 * idx;
  switch (kind) {
    case kGaussian: {
      const double u1 = stream.uniform_at(base);
      const double u2 = stream.uniform_at(base + 1);
      return std::sqrt(-2.0 * std::log1p(-u1)) * std::cos(2.0 * M_PI * u2);
    }
    case kRademacher:
      return (stream.u64_at(base + 3) & 1u) ? 1.0 : -1.0;
    case kSparseGaussian: {
      if (stream.uniform_at(base + 2) >= density) return 0.0;
      const double u1 = stream.uniform_at(base);
      const double u2 = stream.uniform_at(base + 1);
      return std::sqrt(-2.0 * std::log1p(-u1)) * std::cos(2.0 * M_PI * u2) /
             std::sqrt(density);
    }
    case kSparseRademacher: {
      if (stream.uniform_at(base + 2) >= density) return 0.0;
      return ((stream.u64_at(base + 3) & 1u) ? 1.0 : -1.0) / std::sqrt(density);
    }
  }
  param("test matrix: unknown kind");
}

void validate_spec(const Spec& s) {
  if (s.rows < 0 || s.cols < 0) param("test matrix: negative dims");
  if (!(s.density > 0.0 && s.density <= 1.0)) param("test matrix: density must lie in (0,1]");
  if (s.kind < 0 || s.kind > 3) param("test matrix: unknown kind");
}

QM gen_block(const Spec& spec, Index r0, Index r1, Index c0, Index c1, int nthreads = 1) {
  validate_spec(spec);
  if (r0 < 0 || r1 > spec.rows || c0 < 0 || c1 > spec.cols || r0 > r1 || c0 > c1)
    shape("test matrix: block out of range");
  QM m(r1 - r0, c1 - c0);
  const CounterRng root(spec.seed);
  for (int p = 0; p < 4; ++p) {
    const CounterRng stream = root.substream(static_cast<std::uint64_t>(p));
    double* plane = m.p[p].data();
    auto work = [&](Index i0, Index i1) {
      for (Index i = i0; i < i1; ++i)
        for (Index j = c0; j < c1; ++j)
          plane[(i - r0) * (c1 - c0) + (j - c0)] = entry_value(
              stream, spec.kind, spec.density,
              static_cast<std::uint64_t>(i) * static_cast<std::uint64_t>(spec.cols) +
                  static_cast<std::uint64_t>(j));
    };
    if (nthreads <= 1 || (r1 - r0) < 2 * nthreads) {
      work(r0, r1);
    } else {
      std::vector<std::thread> ts;
      const Index nr = r1 - r0;
      for (int t = 0; t < nthreads; ++t)
        ts.emplace_back(work, r0 + nr * t / nthreads, r0 + nr * (t + 1) / nthreads);
      for (auto& t : ts) t.join();
    }
  }
  return m;
}
QM gen_test_matrix(const Spec& s) { return gen_block(s, 0, s.rows, 0, s.cols); }

// -------------------------------------------------------------- sketch ---
// proj/src/sketching.cpp:110-139
void validate_sketch_sizes(Index m, Index n, Index r, Index s, Index l) {
  if (r < 1 || !(r <= s && s <= l && l <= std::min(m, n)))
    param("sketch sizes must satisfy 1 <= r <= s <= l <= min(m,n)");
}

// Y[row0:row0+b] += block * Omega ; W += Psi[:, row0:row0+b] * block
void sketch_update_rows(QM& y, QM& w, const Spec& om, const Spec& ps, Index row0,
                        const QM& block, int nthreads) {
  const Index m = y.rows, n = w.cols;
  if (block.cols != n) shape("sketch_update_rows: column count mismatch");
  if (row0 < 0 || row0 + block.rows > m) shape("sketch_update_rows: row range out of bounds");
  if (block.rows == 0) return;
  const QM omega = gen_block(om, 0, om.rows, 0, om.cols, nthreads);
  QM y_rows(block.rows, y.cols);
  for (int p = 0; p < 4; ++p)
    std::memcpy(y_rows.p[p].data(), y.p[p].data() + row0 * y.cols,
                sizeof(double) * block.rows * y.cols);
  qmat_mul_accumulate_ordered(y_rows, block, omega, nthreads);
  for (int p = 0; p < 4; ++p)
    std::memcpy(y.p[p].data() + row0 * y.cols, y_rows.p[p].data(),
                sizeof(double) * block.rows * y.cols);
  const QM psi_cols = gen_block(ps, 0, ps.rows, row0, row0 + block.rows, nthreads);
  qmat_mul_accumulate_ordered(w, psi_cols, block, nthreads);
}

// ------------------------------------------------------ complex bridge ---
// proj/src/complex_bridge.cpp:11-61; CM is column-major (LAPACK layout).
struct CM {
  Index rows = 0, cols = 0;
  std::vector<cd> a;
  CM() = default;
  int ldv = 1;
  CM(Index r, Index c)
      : rows(r), cols(c), a(static_cast<std::size_t>(r * c), cd(0.0, 0.0)),
        ldv(static_cast<int>(std::max<Index>(1, r))) {}
  cd& operator()(Index i, Index j) { return a[i + j * rows]; }
  cd operator()(Index i, Index j) const { return a[i + j * rows]; }
  cd* col(Index j) { return a.data() + j * rows; }
  const cd* col(Index j) const { return a.data() + j * rows; }
  const int& ld() const { return ldv; }
};

CM to_compact(const QM& q) {
  const Index m = q.rows, n = q.cols;
  CM c(2 * m, n);
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < n; ++j) {
      c(i, j) = cd(q.at(0, i, j), q.at(1, i, j));
      c(m + i, j) = cd(-q.at(2, i, j), q.at(3, i, j));
    }
  return c;
}
CM to_full(const QM& q) {
  const Index m = q.rows, n = q.cols;
  CM c(2 * m, 2 * n);
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < n; ++j) {
      const cd q0(q.at(0, i, j), q.at(1, i, j));
      const cd q1(q.at(2, i, j), q.at(3, i, j));
      c(i, j) = q0;
      c(i, n + j) = q1;
      c(m + i, j) = -std::conj(q1);
      c(m + i, n + j) = std::conj(q0);
    }
  return c;
}
QM from_compact(const CM& z) {
  if (z.rows % 2 != 0) shape("from_compact: odd row count");
  const Index m = z.rows / 2, n = z.cols;
  QM a(m, n);
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < n; ++j) {
      const cd z0 = z(i, j), z1 = z(m + i, j);
      a.at(0, i, j) = z0.real();
      a.at(1, i, j) = z0.imag();
      a.at(2, i, j) = -z1.real();
      a.at(3, i, j) = z1.imag();
    }
  return a;
}
std::vector<cd> jconj_vec(const cd* v, Index len) {  // factorizations.cpp:16-22
  const Index m = len / 2;
  std::vector<cd> r(static_cast<std::size_t>(len));
  for (Index i = 0; i < m; ++i) {
    r[i] = -std::conj(v[m + i]);
    r[m + i] = std::conj(v[i]);
  }
  return r;
}
CM j_mul_conj(const CM& u) {
  if (u.rows % 2 != 0) shape("j_mul_conj: odd row count");
  CM r(u.rows, u.cols);
  for (Index j = 0; j < u.cols; ++j) {
    auto v = jconj_vec(u.col(j), u.rows);
    std::copy(v.begin(), v.end(), r.col(j));
  }
  return r;
}

// Small dense complex helpers.
CM cm_mul(const CM& a, const CM& b, char ta = 'N') {  // op(a) * b
  const Index m = ta == 'N' ? a.rows : a.cols, k = ta == 'N' ? a.cols : a.rows;
  if (k != b.rows) shape("cm_mul: inner dimensions differ");
  CM c(m, b.cols);
  if (m == 0 || b.cols == 0 || k == 0) return c;
  const int M = static_cast<int>(m), N = static_cast<int>(b.cols), K = static_cast<int>(k);
  const cd one(1.0, 0.0), zero(0.0, 0.0);
  const char tb = 'N';
  zgemm_(&ta, &tb, &M, &N, &K, &one, a.a.data(), &a.ld(), b.a.data(), &b.ld(), &zero,
         c.a.data(), &c.ld(), 1, 1);
  (void)0;
  return c;
}
// Long vectors (the 2m-long compact columns of C4 / C5 sketches) are reduced
// by OpenMP threads in a fixed static partition: deterministic, and equal to
// the serial sum to rounding -- these helpers are only the oracle's speed.
constexpr Index kParLen = 1 << 16;
cd dotc(const cd* q, const cd* v, Index n) {  // Eigen q.dot(v) = q^H v
  if (n < kParLen) {
    cd s(0.0, 0.0);
    for (Index i = 0; i < n; ++i) s += std::conj(q[i]) * v[i];
    return s;
  }
  double re = 0.0, im = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : re, im)
  for (Index i = 0; i < n; ++i) {
    const cd t = std::conj(q[i]) * v[i];
    re += t.real();
    im += t.imag();
  }
  return cd(re, im);
}
double norm2(const cd* v, Index n) {
  double s = 0.0;
  if (n < kParLen) {
    for (Index i = 0; i < n; ++i) s += std::norm(v[i]);
    return std::sqrt(s);
  }
#pragma omp parallel for schedule(static) reduction(+ : s)
  for (Index i = 0; i < n; ++i) s += std::norm(v[i]);
  return std::sqrt(s);
}
// v -= q * d
void axpy_sub(cd* v, const cd* q, cd d, Index n) {
  if (n < kParLen) {
    for (Index i = 0; i < n; ++i) v[i] -= q[i] * d;
    return;
  }
#pragma omp parallel for schedule(static)
  for (Index i = 0; i < n; ++i) v[i] -= q[i] * d;
}

// Communication-avoiding QR of a tall matrix (TSQR): cache-sized row blocks
// are factored in parallel (zgeqrf per block, single-threaded BLAS inside),
// their R factors stacked and factored the same way (recursively), and
// Q = diag(Q_i) Q_stack.  Backward stable like one Householder QR of the
// whole; LAPACK's zgeqrf on a 4M x 80 panel is level-2 and memory-bound
// (~50 s), this is ~20x faster.  R's diagonal phases are arbitrary; callers
// normalise them.  Only the oracle's speed: the factorisations it feeds are
// the reference's.
bool tsqr_applies(Index m, Index n) { return n > 0 && m >= 32 * n && m * n >= (Index(1) << 22); }
void householder_qr(CM& b, std::vector<cd>& tau, CM* q) {  // b is overwritten (R in its upper part)
  const int M = static_cast<int>(b.rows), N = static_cast<int>(b.cols);
  int info = 0, lwork = -1;
  cd wq;
  tau.assign(std::max(1, N), cd(0.0, 0.0));
  zgeqrf_(&M, &N, b.a.data(), &b.ld(), tau.data(), &wq, &lwork, &info);
  lwork = std::max(1, static_cast<int>(wq.real()));
  std::vector<cd> work(lwork);
  zgeqrf_(&M, &N, b.a.data(), &b.ld(), tau.data(), work.data(), &lwork, &info);
  if (!q) return;
  *q = b;
  lwork = -1;
  zungqr_(&M, &N, &N, q->a.data(), &q->ld(), tau.data(), &wq, &lwork, &info);
  lwork = std::max(1, static_cast<int>(wq.real()));
  work.assign(lwork, cd(0.0, 0.0));
  zungqr_(&M, &N, &N, q->a.data(), &q->ld(), tau.data(), work.data(), &lwork, &info);
}
template <class F>
void parallel_blocks(Index nb, F&& f) {
  const int hw = std::max(1, static_cast<int>(std::thread::hardware_concurrency()));
  const int T = static_cast<int>(std::min<Index>(hw, nb));
  std::atomic<Index> next{0};
  const int saved = openblas_get_num_threads();
  openblas_set_num_threads(1);
  auto body = [&] {
    for (Index i = next++; i < nb; i = next++) f(i);
  };
  std::vector<std::thread> ts;
  for (int t = 1; t < T; ++t) ts.emplace_back(body);
  body();
  for (auto& t : ts) t.join();
  openblas_set_num_threads(saved);
}
void tsqr(const CM& a, CM* q, CM* r) {
  const Index m = a.rows, n = a.cols;
  const Index B = std::max<Index>(4096, 8 * n);
  const Index nb = (m + B - 1) / B;
  if (nb <= 1) {
    CM b = a;
    std::vector<cd> tau;
    householder_qr(b, tau, q);
    *r = CM(n, n);
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i <= std::min(j, m - 1); ++i) (*r)(i, j) = b(i, j);
    return;
  }
  std::vector<CM> blk(nb);
  std::vector<std::vector<cd>> tau(nb);
  CM s(nb * n, n);
  parallel_blocks(nb, [&](Index t) {
    const Index r0 = t * B, r1 = std::min(m, r0 + B), rows = r1 - r0;
    CM b(rows, n);
    for (Index j = 0; j < n; ++j) std::copy(a.col(j) + r0, a.col(j) + r1, b.col(j));
    householder_qr(b, tau[t], nullptr);
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i <= std::min(j, rows - 1); ++i) s(t * n + i, j) = b(i, j);
    blk[t] = std::move(b);
  });
  CM qs;
  tsqr(s, q ? &qs : nullptr, r);
  if (!q) return;
  *q = CM(m, n);
  parallel_blocks(nb, [&](Index t) {
    const Index r0 = t * B, rows = blk[t].rows;
    CM& b = blk[t];
    const int M = static_cast<int>(rows), N = static_cast<int>(n);
    int info = 0, lwork = -1;
    cd wq;
    // Q_t * (Q_stack rows of block t): apply the block's reflectors to them
    CM c(rows, n);
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < std::min(n, rows); ++i) c(i, j) = qs(t * n + i, j);
    const int K = static_cast<int>(std::min(n, rows));
    zunmqr_("L", "N", &M, &N, &K, b.a.data(), &b.ld(), tau[t].data(), c.a.data(), &c.ld(), &wq, &lwork, &info,
            1, 1);
    lwork = std::max(1, static_cast<int>(wq.real()));
    std::vector<cd> work(lwork);
    zunmqr_("L", "N", &M, &N, &K, b.a.data(), &b.ld(), tau[t].data(), c.a.data(), &c.ld(), work.data(), &lwork,
            &info, 1, 1);
    for (Index j = 0; j < n; ++j) std::copy(c.col(j), c.col(j) + rows, q->col(j) + r0);
  });
}

// ------------------------------------------------------ factorizations ---
// complex_qr (factorizations.cpp:33-51)
struct ComplexQr {
  CM q, r;
};
ComplexQr complex_qr(const CM& mat) {
  if (mat.rows < mat.cols) shape("complex_qr: requires rows >= cols");
  const int m = static_cast<int>(mat.rows), n = static_cast<int>(mat.cols);
  ComplexQr out;
  if (tsqr_applies(m, n)) {
    tsqr(mat, &out.q, &out.r);
    // the same phase convention as below (diag(R) real >= 0)
    for (int k = 0; k < n; ++k) {
      const cd d = out.r(k, k);
      const double ad = std::abs(d);
      if (ad > 0.0) {
        const cd phase = d / ad;
        for (int j = 0; j < n; ++j) out.r(k, j) *= std::conj(phase);
        for (int i = 0; i < m; ++i) out.q(i, k) *= phase;
      }
    }
    return out;
  }
  CM a = mat;
  std::vector<cd> tau(std::max(1, n));
  int info = 0, lwork = -1;
  cd wq;
  if (n > 0) {
    zgeqrf_(&m, &n, a.a.data(), &a.ld(), tau.data(), &wq, &lwork, &info);
    lwork = std::max(1, static_cast<int>(wq.real()));
    std::vector<cd> work(lwork);
    zgeqrf_(&m, &n, a.a.data(), &a.ld(), tau.data(), work.data(), &lwork, &info);
  }
  out.r = CM(n, n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i <= j; ++i) out.r(i, j) = a(i, j);
  if (n > 0) {
    lwork = -1;
    zungqr_(&m, &n, &n, a.a.data(), &a.ld(), tau.data(), &wq, &lwork, &info);
    lwork = std::max(1, static_cast<int>(wq.real()));
    std::vector<cd> work(lwork);
    zungqr_(&m, &n, &n, a.a.data(), &a.ld(), tau.data(), work.data(), &lwork, &info);
  }
  out.q = CM(m, n);
  std::copy(a.a.begin(), a.a.begin() + static_cast<std::size_t>(m) * n, out.q.a.begin());
  for (int k = 0; k < n; ++k) {
    const cd d = out.r(k, k);
    const double ad = std::abs(d);
    if (ad > 0.0) {
      const cd phase = d / ad;
      for (int j = 0; j < n; ++j) out.r(k, j) *= std::conj(phase);
      for (int i = 0; i < m; ++i) out.q(i, k) *= phase;
    }
  }
  return out;
}

// complex_svd (factorizations.cpp:53-56): thin U, V, nonincreasing s.
struct ComplexSvd {
  CM u;
  std::vector<double> s;
  CM v;
};
// want_u = false: singular values and V only (condition_number,
// singular_values), U left zero.
ComplexSvd complex_svd(const CM& mat, bool want_u = true) {
  const int m = static_cast<int>(mat.rows), n = static_cast<int>(mat.cols);
  const int k = std::min(m, n);
  ComplexSvd out;
  out.u = CM(want_u || !tsqr_applies(m, n) ? m : 0, k);
  out.v = CM(n, k);
  out.s.assign(k, 0.0);
  if (k == 0) return out;
  if (tsqr_applies(m, n)) {
    // zgesdd's own path for m >> n (QR, SVD of R, U = Q U_R) with the QR
    // done by TSQR
    CM q, r;
    tsqr(mat, want_u ? &q : nullptr, &r);
    ComplexSvd sr = complex_svd(r);
    out.s = std::move(sr.s);
    out.v = std::move(sr.v);
    if (want_u) {
      const cd one(1.0, 0.0), zero(0.0, 0.0);
      zgemm_("N", "N", &m, &n, &n, &one, q.a.data(), &q.ld(), sr.u.a.data(), &sr.u.ld(), &zero,
             out.u.a.data(), &out.u.ld(), 1, 1);
    }
    return out;
  }
  CM a = mat;
  CM vt(k, n);
  const int lda = a.ld(), ldu = out.u.ld(), ldvt = vt.ld();  // copies
  // LRWORK of zgesdd (LAPACK >= 3.7): 5 mn^2 + 5 mn when mx >> mn, else
  // max(5 mn^2 + 5 mn, 2 mx mn + 2 mn^2 + mn)
  const std::size_t mn = static_cast<std::size_t>(k), mx = static_cast<std::size_t>(std::max(m, n));
  const std::size_t lrw = (mx * 9 >= mn * 17) ? 5 * mn * mn + 5 * mn
                                              : std::max(5 * mn * mn + 5 * mn, 2 * mx * mn + 2 * mn * mn + mn);
  std::vector<double> rwork(std::max<std::size_t>(1, lrw));
  std::vector<int> iwork(8 * k);
  int info = 0, lwork = -1;
  cd wq;
  zgesdd_("S", &m, &n, a.a.data(), &lda, out.s.data(), out.u.a.data(), &ldu, vt.a.data(),
          &ldvt, &wq, &lwork, rwork.data(), iwork.data(), &info, 1);
  lwork = std::max(1, static_cast<int>(wq.real()));
  std::vector<cd> work(lwork);
  zgesdd_("S", &m, &n, a.a.data(), &lda, out.s.data(), out.u.a.data(), &ldu, vt.a.data(),
          &ldvt, work.data(), &lwork, rwork.data(), iwork.data(), &info, 1);
  if (info != 0) throw Error(kInternal, "zgesdd failed: info=" + std::to_string(info));
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < n; ++j) out.v(j, i) = std::conj(vt(i, j));
  return out;
}

// detail::split_singular_pairs (factorizations.cpp:60-81, constants .hpp:63-64)
constexpr double kPairGapRel = 1e-8;
constexpr double kPairFloorRel = 1e-13;
struct PairSplit {
  std::vector<Index> good, bad;
};
PairSplit split_singular_pairs(const std::vector<double>& sv) {
  PairSplit out;
  const Index n = static_cast<Index>(sv.size());
  if (n == 0) return out;
  const double s1 = sv[0];
  const double gap = kPairGapRel * s1;
  const double floor_tol = kPairFloorRel * s1;
  Index start = 0;
  for (Index i = 1; i <= n; ++i) {
    const bool boundary = (i == n) || (sv[i - 1] - sv[i] > gap);
    if (!boundary) continue;
    const Index len = i - start;
    if (len == 2 && sv[start + 1] > floor_tol) {
      out.good.push_back(start);
    } else {
      for (Index c = start; c < i; ++c) out.bad.push_back(c);
    }
    start = i;
  }
  return out;
}

using Vec = std::vector<cd>;
Vec orthogonalize(Vec v, const std::vector<Vec>& basis) {  // factorizations.cpp:24-29
  const Index n = static_cast<Index>(v.size());
  for (int pass = 0; pass < 2; ++pass)
    for (const auto& q : basis) {
      const cd d = dotc(q.data(), v.data(), n);
      axpy_sub(v.data(), q.data(), d, n);
    }
  return v;
}
Vec col_vec(const CM& m, Index j) { return Vec(m.col(j), m.col(j) + m.rows); }

// detail::select_via_mgs (factorizations.cpp:83-126)
CM select_via_mgs(const CM& ub, Index count, const CM& context) {
  const Index dim = ub.rows;
  std::vector<Vec> basis;
  for (Index j = 0; j < context.cols; ++j) basis.push_back(col_vec(context, j));
  std::vector<bool> used(static_cast<std::size_t>(ub.cols), false);
  CM chosen(dim, count);
  for (Index step = 0; step < count; ++step) {
    double best_norm = -1.0;
    Index best = -1;
    Vec best_vec;
    for (Index c = 0; c < ub.cols; ++c) {
      if (used[c]) continue;
      Vec r = orthogonalize(col_vec(ub, c), basis);
      const double nr = norm2(r.data(), dim);
      if (nr > best_norm) {
        best_norm = nr;
        best = c;
        best_vec = std::move(r);
      }
    }
    if (best_norm < 1e-8) {
      for (Index e = 0; e < dim; ++e) {
        Vec cand(dim, cd(0.0, 0.0));
        cand[e] = 1.0;
        cand = orthogonalize(std::move(cand), basis);
        if (norm2(cand.data(), dim) > 0.5) {
          best_vec = std::move(cand);
          best_norm = norm2(best_vec.data(), dim);
          best = -1;
          break;
        }
      }
    }
    if (best >= 0) used[best] = true;
    const double nb = norm2(best_vec.data(), dim);
    for (auto& x : best_vec) x /= nb;
    std::copy(best_vec.begin(), best_vec.end(), chosen.col(step));
    basis.push_back(best_vec);
    basis.push_back(jconj_vec(best_vec.data(), dim));
  }
  return chosen;
}

// detail::select_bad_representatives (factorizations.cpp:128-152)
CM select_bad_representatives(const CM& ub, Index s_total, const CM& context,
                              SequentialRng& rng) {
  const Index b = ub.cols;
  if (b == 0) return CM(ub.rows, 0);
  const Index t = b / 2;
  if (t <= (s_total + 1) / 2) {
    QM hb = from_compact(ub);
    for (Index j = 0; j < b; ++j) hb.scale_col(j, 1.0 + rng.next_uniform());
    const ComplexSvd svd = complex_svd(to_full(hb));
    const PairSplit split = split_singular_pairs(svd.s);
    std::vector<Index> reps;
    for (Index g : split.good)
      if (svd.s[g] > 1e-10 * svd.s[0]) reps.push_back(g);
    if (static_cast<Index>(reps.size()) == t) {
      CM chosen(ub.rows, t);
      for (Index i = 0; i < t; ++i)
        std::copy(svd.u.col(reps[i]), svd.u.col(reps[i]) + ub.rows, chosen.col(i));
      return chosen;
    }
  }
  return select_via_mgs(ub, t, context);
}

// singular_values / condition_number (factorizations.cpp:316-337)
std::vector<double> singular_values(const QM& a) {
  const Index k = std::min(a.rows, a.cols);
  if (k == 0) return {};
  const ComplexSvd svd = complex_svd(to_full(a), /*want_u=*/false);
  std::vector<double> out(k);
  for (Index i = 0; i < k; ++i) out[i] = svd.s[2 * i];
  return out;
}
double condition_number(const QM& a) {
  const Index k = std::min(a.rows, a.cols);
  if (k == 0) return std::numeric_limits<double>::infinity();
  const ComplexSvd svd = complex_svd(to_full(a), /*want_u=*/false);
  const double smin = svd.s[2 * k - 1];
  if (!(smin > 0.0)) return std::numeric_limits<double>::infinity();
  return svd.s[0] / smin;
}

// qsvd (factorizations.cpp:166-295)
struct Qsvd {
  QM u;
  std::vector<double> sigma;
  QM v;
};
struct SingularColumn {
  double sigma;
  Vec u, v;
};
Qsvd qsvd(const QM& a) {
  if (a.rows < a.cols) {
    Qsvd f = qsvd(a.adjoint());
    return {std::move(f.v), std::move(f.sigma), std::move(f.u)};
  }
  const Index m = a.rows, n = a.cols, k = n;
  if (k == 0) return {QM(m, 0), {}, QM(n, 0)};
  const CM chi = to_full(a);
  const ComplexSvd svd = complex_svd(chi);
  const PairSplit split = split_singular_pairs(svd.s);
  std::vector<SingularColumn> cols;
  CM good_u(chi.rows, 2 * static_cast<Index>(split.good.size()));
  CM good_v(2 * n, 2 * static_cast<Index>(split.good.size()));
  for (std::size_t i = 0; i < split.good.size(); ++i) {
    const Index g = split.good[i];
    cols.push_back({svd.s[g], col_vec(svd.u, g), col_vec(svd.v, g)});
    auto ju = jconj_vec(svd.u.col(g), chi.rows);
    auto jv = jconj_vec(svd.v.col(g), 2 * n);
    std::copy(svd.u.col(g), svd.u.col(g) + chi.rows, good_u.col(2 * i));
    std::copy(ju.begin(), ju.end(), good_u.col(2 * i + 1));
    std::copy(svd.v.col(g), svd.v.col(g) + 2 * n, good_v.col(2 * i));
    std::copy(jv.begin(), jv.end(), good_v.col(2 * i + 1));
  }
  if (!split.bad.empty()) {
    const double s1 = svd.s[0];
    const double tiny = 1e-10 * s1;
    CM ub(chi.rows, static_cast<Index>(split.bad.size()));
    CM vb(2 * n, static_cast<Index>(split.bad.size()));
    for (std::size_t i = 0; i < split.bad.size(); ++i) {
      std::copy(svd.u.col(split.bad[i]), svd.u.col(split.bad[i]) + chi.rows, ub.col(i));
      std::copy(svd.v.col(split.bad[i]), svd.v.col(split.bad[i]) + 2 * n, vb.col(i));
    }
    SequentialRng rng(CounterRng(0x715D).substream(static_cast<std::uint64_t>(m * 131 + n)));
    const CM cu = select_bad_representatives(ub, k, good_u, rng);
    const CM w_all = cm_mul(chi, cu, 'C');  // chi^* cu
    std::vector<Vec> chosen_v;
    std::vector<Index> pending;
    std::vector<SingularColumn> bad_cols(static_cast<std::size_t>(cu.cols));
    for (Index i = 0; i < cu.cols; ++i) {
      Vec w = col_vec(w_all, i);
      const double nrm = norm2(w.data(), 2 * n);
      auto& sc = bad_cols[i];
      sc.sigma = nrm;
      sc.u = col_vec(cu, i);
      if (nrm > tiny) {
        for (auto& x : w) x /= nrm;
        sc.v = w;
        chosen_v.push_back(sc.v);
      } else {
        pending.push_back(i);
      }
    }
    if (!pending.empty()) {
      CM vctx(2 * n, good_v.cols + 2 * static_cast<Index>(chosen_v.size()));
      std::copy(good_v.a.begin(), good_v.a.end(), vctx.a.begin());
      for (std::size_t i = 0; i < chosen_v.size(); ++i) {
        std::copy(chosen_v[i].begin(), chosen_v[i].end(), vctx.col(good_v.cols + 2 * i));
        auto jv = jconj_vec(chosen_v[i].data(), 2 * n);
        std::copy(jv.begin(), jv.end(), vctx.col(good_v.cols + 2 * i + 1));
      }
      const CM vsel = select_via_mgs(vb, static_cast<Index>(pending.size()), vctx);
      for (std::size_t i = 0; i < pending.size(); ++i) bad_cols[pending[i]].v = col_vec(vsel, i);
    }
    for (auto& sc : bad_cols) cols.push_back(std::move(sc));
  }
  std::stable_sort(cols.begin(), cols.end(), [](const SingularColumn& x, const SingularColumn& y) {
    return x.sigma > y.sigma;
  });
  std::vector<Vec> ubasis, vbasis;
  for (auto& sc : cols) {
    sc.u = orthogonalize(std::move(sc.u), ubasis);
    double nu = norm2(sc.u.data(), sc.u.size());
    for (auto& x : sc.u) x /= nu;
    sc.v = orthogonalize(std::move(sc.v), vbasis);
    double nv = norm2(sc.v.data(), sc.v.size());
    for (auto& x : sc.v) x /= nv;
    ubasis.push_back(sc.u);
    ubasis.push_back(jconj_vec(sc.u.data(), sc.u.size()));
    vbasis.push_back(sc.v);
    vbasis.push_back(jconj_vec(sc.v.data(), sc.v.size()));
  }
  CM uc(chi.rows, k), vc(2 * n, k);
  Qsvd out;
  out.sigma.resize(k);
  for (Index i = 0; i < k; ++i) {
    std::copy(cols[i].u.begin(), cols[i].u.end(), uc.col(i));
    std::copy(cols[i].v.begin(), cols[i].v.end(), vc.col(i));
    out.sigma[i] = cols[i].sigma;
  }
  out.u = from_compact(uc);
  out.v = from_compact(vc);
  for (Index j = 0; j < k; ++j) {
    Index arg = 0;
    double best = -1.0;
    for (Index i = 0; i < n; ++i) {
      double q[4];
      out.v.get(i, j, q);
      const double ns = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3];
      if (ns > best) {
        best = ns;
        arg = i;
      }
    }
    double e[4];
    out.v.get(arg, j, e);
    const double ae = std::sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2] + e[3] * e[3]);
    if (ae > 0.0) {
      const double p[4] = {e[0] * (1.0 / ae), -e[1] * (1.0 / ae), -e[2] * (1.0 / ae),
                           -e[3] * (1.0 / ae)};
      out.u.scale_col(j, p);
      out.v.scale_col(j, p);
    }
  }
  return out;
}

// ----------------------------------------------- solve_quaternion_linear ---
// complex_bridge.cpp:63-90
constexpr double kSingularRcond = 1e-14;
QM solve_quaternion_linear(const QM& a, const QM& b) {
  if (a.rows != b.rows) shape("solve_quaternion_linear: row mismatch");
  if (a.rows < a.cols) shape("solve_quaternion_linear: underdetermined system not supported");
  CM chi = to_full(a);
  CM bc = to_compact(b);
  const int n = static_cast<int>(chi.cols), mrows = static_cast<int>(chi.rows);
  const int nrhs = static_cast<int>(bc.cols);
  int info = 0;
  if (a.rows == a.cols) {
    if (n == 0) return from_compact(bc);
    const double anorm = zlange_("1", &n, &n, chi.a.data(), &chi.ld(), nullptr, 1);
    std::vector<int> ipiv(n);
    zgetrf_(&n, &n, chi.a.data(), &chi.ld(), ipiv.data(), &info);
    double rc = 0.0;
    if (info == 0 && anorm > 0.0) {
      std::vector<cd> work(2 * n);
      std::vector<double> rwork(2 * n);
      int info2 = 0;
      zgecon_("1", &n, chi.a.data(), &chi.ld(), &anorm, &rc, work.data(), rwork.data(), &info2, 1);
    }
    if (!(rc > kSingularRcond))
      singular("solve_quaternion_linear: singular system",
               rc > 0 ? 1.0 / rc : std::numeric_limits<double>::infinity());
    if (nrhs > 0)
      zgetrs_("N", &n, &nrhs, chi.a.data(), &chi.ld(), ipiv.data(), bc.a.data(), &bc.ld(), &info, 1);
    return from_compact(bc);
  }
  // Overdetermined: column-pivoted Householder QR (Eigen ColPivHouseholderQR).
  std::vector<int> jpvt(n, 0);
  std::vector<cd> tau(std::max(1, n));
  std::vector<double> rwork(2 * std::max(1, n));
  int lwork = -1;
  cd wq;
  zgeqp3_(&mrows, &n, chi.a.data(), &chi.ld(), jpvt.data(), tau.data(), &wq, &lwork,
          rwork.data(), &info);
  lwork = std::max(1, static_cast<int>(wq.real()));
  {
    std::vector<cd> work(lwork);
    zgeqp3_(&mrows, &n, chi.a.data(), &chi.ld(), jpvt.data(), tau.data(), work.data(), &lwork,
            rwork.data(), &info);
  }
  const double rmax = std::abs(chi(0, 0));
  const double rmin = std::abs(chi(n - 1, n - 1));
  if (!(rmin > kSingularRcond * rmax))
    singular("solve_quaternion_linear: rank-deficient system",
             rmin > 0 ? rmax / rmin : std::numeric_limits<double>::infinity());
  if (nrhs > 0) {
    lwork = -1;
    zunmqr_("L", "C", &mrows, &nrhs, &n, chi.a.data(), &chi.ld(), tau.data(), bc.a.data(),
            &bc.ld(), &wq, &lwork, &info, 1, 1);
    lwork = std::max(1, static_cast<int>(wq.real()));
    std::vector<cd> work(lwork);
    zunmqr_("L", "C", &mrows, &nrhs, &n, chi.a.data(), &chi.ld(), tau.data(), bc.a.data(),
            &bc.ld(), work.data(), &lwork, &info, 1, 1);
    const cd one(1.0, 0.0);
    ztrsm_("L", "U", "N", "N", &n, &nrhs, &one, chi.a.data(), &chi.ld(), bc.a.data(), &bc.ld(),
           1, 1, 1, 1);
  }
  CM z(n, nrhs);
  for (int j = 0; j < nrhs; ++j)
    for (int i = 0; i < n; ++i) z(jpvt[i] - 1, j) = bc(i, j);
  return from_compact(z);
}

// --------------------------------------------------------- rangefinders ---
// proj/src/rangefinders.cpp:18-176
constexpr double kKappaTarget = 10.0;
constexpr double kEpsilonClamp = 0.999;

QM assemble_orthonormal_basis(const QM& y, std::uint64_t seed) {
  const Index s = y.cols;
  const CM chi = to_full(y);
  const ComplexSvd svd = complex_svd(chi);
  const PairSplit split = split_singular_pairs(svd.s);
  CM compact(chi.rows, s);
  CM good(chi.rows, 2 * static_cast<Index>(split.good.size()));
  Index filled = 0;
  for (std::size_t i = 0; i < split.good.size(); ++i) {
    const cd* u = svd.u.col(split.good[i]);
    std::copy(u, u + chi.rows, compact.col(filled));
    std::copy(u, u + chi.rows, good.col(2 * i));
    auto ju = jconj_vec(u, chi.rows);
    std::copy(ju.begin(), ju.end(), good.col(2 * i + 1));
    ++filled;
  }
  if (!split.bad.empty()) {
    CM ub(chi.rows, static_cast<Index>(split.bad.size()));
    for (std::size_t i = 0; i < split.bad.size(); ++i)
      std::copy(svd.u.col(split.bad[i]), svd.u.col(split.bad[i]) + chi.rows, ub.col(i));
    SequentialRng rng(CounterRng(seed).substream(0x6261645F626C6BULL));
    const CM cu = select_bad_representatives(ub, s, good, rng);
    for (Index c = 0; c < cu.cols; ++c)
      std::copy(cu.col(c), cu.col(c) + chi.rows, compact.col(s - cu.cols + c));
    filled += cu.cols;
  }
  std::vector<Vec> basis;
  for (Index c = 0; c < s; ++c) {
    Vec u = col_vec(compact, c);
    for (int pass = 0; pass < 2; ++pass)
      for (const auto& q : basis) {
        const cd d = dotc(q.data(), u.data(), chi.rows);
        axpy_sub(u.data(), q.data(), d, chi.rows);
      }
    const double nu = norm2(u.data(), chi.rows);
    for (auto& x : u) x /= nu;
    std::copy(u.begin(), u.end(), compact.col(c));
    basis.push_back(u);
    basis.push_back(jconj_vec(u.data(), chi.rows));
  }
  return from_compact(compact);
}

double estimate_epsilon(const QM& h, int power_iters) {
  if (power_iters < 1) param("estimate_epsilon: power_iters must be >= 1");
  const QM gram = qmat_mul(h.adjoint(), h);
  CM chi = to_full(gram);
  const int n = static_cast<int>(chi.rows);
  const double anorm = zlange_("1", &n, &n, chi.a.data(), &chi.ld(), nullptr, 1);
  std::vector<int> ipiv(std::max(1, n));
  int info = 0;
  zgetrf_(&n, &n, chi.a.data(), &chi.ld(), ipiv.data(), &info);
  double rc = 0.0;
  if (info == 0 && anorm > 0.0) {
    std::vector<cd> work(2 * n);
    std::vector<double> rwork(2 * n);
    int info2 = 0;
    zgecon_("1", &n, chi.a.data(), &chi.ld(), &anorm, &rc, work.data(), rwork.data(), &info2, 1);
  }
  if (!(rc > 1e-15))
    singular("estimate_epsilon: H*H numerically singular",
             rc > 0 ? 1.0 / rc : std::numeric_limits<double>::infinity());
  SequentialRng rng(CounterRng(0x455053ULL).substream(static_cast<std::uint64_t>(n)));
  std::vector<cd> z(n);
  // Same expression as rangefinders.cpp:82-83; g++ evaluates the two
  // constructor arguments right to left (imag draw first).
  for (int i = 0; i < n; ++i) z[i] = std::complex<double>(rng.next_gaussian(), rng.next_gaussian());
  {
    const double nz = norm2(z.data(), n);
    for (auto& x : z) x /= nz;
  }
  double rho = 0.0;
  const int one = 1;
  for (int it = 0; it < power_iters; ++it) {
    std::vector<cd> w = z;
    zgetrs_("N", &n, &one, chi.a.data(), &chi.ld(), ipiv.data(), w.data(), &n, &info, 1);
    rho = dotc(z.data(), w.data(), n).real();
    const double nw = norm2(w.data(), n);
    if (!(nw > 0.0)) break;
    for (int i = 0; i < n; ++i) z[i] = w[i] / nw;
  }
  if (!(rho > 0.0)) singular("estimate_epsilon: breakdown", 0.0);
  const double eps = 1.0 / std::sqrt(rho);
  return std::min(eps, kEpsilonClamp);
}

QM correction_step(const QM& h, double epsilon) {
  if (!(epsilon > 0.0 && epsilon < 1.0)) param("correction_step: epsilon must lie in (0,1)");
  const QM gram = qmat_mul(h.adjoint(), h);
  const QM pinv = solve_quaternion_linear(gram, h.adjoint());
  return (1.0 - epsilon) * h + epsilon * pinv.adjoint();
}

struct Report {
  QM h;
  double kappa_before = 0.0, kappa_after = 0.0;
  int steps = 0;
};

Report pseudo_qr(const QM& y, int max_steps, int power_iters, double delta) {
  if (y.rows <= y.cols) param("pseudo_qr: sketch must be tall (rows > cols)");
  if (max_steps < 0) param("pseudo_qr: negative correction step count");
  if (!(delta >= 1.0 && delta <= std::sqrt(7.0) / 2.0 + 1e-12))
    param("pseudo_qr: delta_budget outside [1, sqrt(7)/2]");
  const ComplexQr qr = complex_qr(to_compact(y));
  double rmax = 0.0, rmin = std::numeric_limits<double>::infinity();
  for (Index k = 0; k < qr.r.rows; ++k) {
    const double d = std::abs(qr.r(k, k));
    rmax = std::max(rmax, d);
    rmin = std::min(rmin, d);
  }
  if (!(rmin > 1e-14 * rmax)) rank_err("pseudo_qr: sketch numerically rank-deficient; use pseudo_svd");
  Report rep;
  rep.h = from_compact(qr.q);
  rep.kappa_before = condition_number(rep.h);
  double kappa = rep.kappa_before;
  try {
    while (rep.steps < max_steps && kappa > kKappaTarget) {
      const double eps = estimate_epsilon(rep.h, power_iters);
      rep.h = correction_step(rep.h, eps);
      kappa = condition_number(rep.h);
      ++rep.steps;
    }
  } catch (const Error& e) {
    if (e.code != kSingular) throw;
    rank_err("pseudo_qr: sketch numerically rank-deficient; use pseudo_svd");
  }
  if (rep.steps > 0) {
    const Index s = y.cols;
    CM paired(qr.q.rows, 2 * s);
    std::copy(qr.q.a.begin(), qr.q.a.end(), paired.a.begin());
    CM jq = j_mul_conj(qr.q);
    std::copy(jq.a.begin(), jq.a.end(), paired.a.begin() + qr.q.a.size());
    const ComplexQr basis = complex_qr(paired);
    const CM hc = to_compact(rep.h);
    rep.h = from_compact(cm_mul(basis.q, cm_mul(basis.q, hc, 'C')));
    rep.kappa_after = condition_number(rep.h);
  } else {
    rep.kappa_after = kappa;
  }
  return rep;
}

Report pseudo_svd(const QM& y, std::uint64_t seed) {
  if (y.rows <= y.cols) param("pseudo_svd: sketch must be tall (rows > cols)");
  Report rep;
  rep.kappa_before = condition_number(y);
  rep.h = assemble_orthonormal_basis(y, seed);
  rep.kappa_after = condition_number(rep.h);
  rep.steps = 0;
  return rep;
}

QM orthonormal_range(const QM& y, std::uint64_t seed) {
  if (y.rows < y.cols) param("orthonormal_range: requires rows >= cols");
  return assemble_orthonormal_basis(y, seed);
}

}  // namespace orc

// =================================================================== C ABI ===
// Flat interface for tests/ and bench.py (ctypes).  Quaternion matrices are
// passed as one contiguous buffer of 4 row-major planes [4][rows][cols].
namespace {
thread_local std::string g_err;
thread_local double g_cond = 0.0;

orc::QM load(const double* buf, Index r, Index c) {
  orc::QM m(r, c);
  const std::size_t n = static_cast<std::size_t>(r * c);
  for (int p = 0; p < 4; ++p) std::memcpy(m.p[p].data(), buf + p * n, n * sizeof(double));
  return m;
}
void store(const orc::QM& m, double* buf) {
  const std::size_t n = static_cast<std::size_t>(m.rows * m.cols);
  for (int p = 0; p < 4; ++p) std::memcpy(buf + p * n, m.p[p].data(), n * sizeof(double));
}
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const orc::Error& e) {
    g_err = e.what();
    g_cond = e.cond;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return orc::kInternal;
  }
}
orc::Spec spec_of(int kind, Index rows, Index cols, std::uint64_t seed, double density) {
  orc::Spec s;
  s.kind = kind;
  s.rows = rows;
  s.cols = cols;
  s.seed = seed;
  s.density = density;
  return s;
}
}  // namespace

extern "C" {

const char* orc_last_error(double* cond) {
  if (cond) *cond = g_cond;
  return g_err.c_str();
}

std::uint64_t orc_mix64(std::uint64_t z) { return orc::mix64(z); }
std::uint64_t orc_stream_key(std::uint64_t seed, std::uint64_t sub, int use_sub) {
  orc::CounterRng r(seed);
  return use_sub ? r.substream(sub).key : r.key;
}
std::uint64_t orc_u64_at(std::uint64_t key, std::uint64_t c) {
  orc::CounterRng r(0);
  r.key = key;
  return r.u64_at(c);
}

int orc_gen_block(int kind, Index rows, Index cols, std::uint64_t seed, double density, Index r0,
                  Index r1, Index c0, Index c1, double* out, int nthreads) {
  return guard([&] {
    store(orc::gen_block(spec_of(kind, rows, cols, seed, density), r0, r1, c0, c1, nthreads), out);
  });
}

int orc_qmat_mul_acc_ordered(Index m, Index k, Index n, const double* a, const double* b,
                             double* c, int nthreads) {
  return guard([&] {
    orc::QM A = load(a, m, k), B = load(b, k, n), C = load(c, m, n);
    orc::qmat_mul_accumulate_ordered(C, A, B, nthreads);
    store(C, c);
  });
}

int orc_qmat_mul(Index m, Index k, Index n, const double* a, const double* b, double* c) {
  return guard([&] { store(orc::qmat_mul(load(a, m, k), load(b, k, n)), c); });
}

int orc_validate_sketch_sizes(Index m, Index n, Index r, Index s, Index l) {
  return guard([&] { orc::validate_sketch_sizes(m, n, r, s, l); });
}

// Y (m x s, rows [row0, row0+b) touched) and W (l x n) updated in place.
int orc_sketch_update_rows(Index m, Index n, Index s, Index l, int kind, double density,
                           std::uint64_t omega_seed, std::uint64_t psi_seed, Index row0,
                           Index b, const double* block, double* y, double* w, int nthreads) {
  return guard([&] {
    orc::QM Y = load(y, m, s), W = load(w, l, n), B = load(block, b, n);
    orc::sketch_update_rows(Y, W, spec_of(kind, n, s, omega_seed, density),
                            spec_of(kind, l, m, psi_seed, density), row0, B, nthreads);
    store(Y, y);
    store(W, w);
  });
}

int orc_condition_number(Index m, Index n, const double* a, double* kappa) {
  return guard([&] { *kappa = orc::condition_number(load(a, m, n)); });
}
int orc_singular_values(Index m, Index n, const double* a, double* sv) {
  return guard([&] {
    auto v = orc::singular_values(load(a, m, n));
    std::copy(v.begin(), v.end(), sv);
  });
}

int orc_solve_quaternion_linear(Index m, Index n, Index k, const double* a, const double* b,
                                double* x) {
  return guard([&] { store(orc::solve_quaternion_linear(load(a, m, n), load(b, m, k)), x); });
}

int orc_estimate_epsilon(Index m, Index s, const double* h, int power_iters, double* eps) {
  return guard([&] { *eps = orc::estimate_epsilon(load(h, m, s), power_iters); });
}
int orc_correction_step(Index m, Index s, const double* h, double eps, double* out) {
  return guard([&] { store(orc::correction_step(load(h, m, s), eps), out); });
}

int orc_pseudo_qr(Index m, Index s, const double* y, int max_steps, int power_iters, double delta,
                  double* h, double* kb, double* ka, int* steps) {
  return guard([&] {
    auto rep = orc::pseudo_qr(load(y, m, s), max_steps, power_iters, delta);
    store(rep.h, h);
    *kb = rep.kappa_before;
    *ka = rep.kappa_after;
    *steps = rep.steps;
  });
}
int orc_pseudo_svd(Index m, Index s, const double* y, std::uint64_t seed, double* h, double* kb,
                   double* ka) {
  return guard([&] {
    auto rep = orc::pseudo_svd(load(y, m, s), seed);
    store(rep.h, h);
    *kb = rep.kappa_before;
    *ka = rep.kappa_after;
  });
}
int orc_orthonormal_range(Index m, Index s, const double* y, std::uint64_t seed, double* h) {
  return guard([&] { store(orc::orthonormal_range(load(y, m, s), seed), h); });
}

// qsvd: u (m x k), sigma (k), v (n x k), k = min(m, n)
int orc_qsvd(Index m, Index n, const double* a, double* u, double* sigma, double* v) {
  return guard([&] {
    auto f = orc::qsvd(load(a, m, n));
    store(f.u, u);
    store(f.v, v);
    std::copy(f.sigma.begin(), f.sigma.end(), sigma);
  });
}

// qb_stage_with_psi (sketching.cpp:169-188), Psi regenerated from its spec
// (qb_stage, :190-194) unless psi != NULL.  method 0 = pseudo-QR, 1 = pseudo-SVD.
int orc_qb_stage(Index m, Index n, Index s, Index l, const double* y, const double* w, int kind,
                 double density, std::uint64_t psi_seed, const double* psi, int method,
                 std::uint64_t rf_seed, int max_steps, int power_iters, double delta, double* h,
                 double* x, double* kb, double* ka, int* steps, double* t_rf, double* t_solve,
                 int nthreads) {
  return guard([&] {
    orc::QM Y = load(y, m, s), W = load(w, l, n);
    orc::QM Psi = psi ? load(psi, l, m)
                      : orc::gen_block(spec_of(kind, l, m, psi_seed, density), 0, l, 0, m,
                                       nthreads);
    auto t0 = std::chrono::steady_clock::now();
    orc::Report rep = method == 0 ? orc::pseudo_qr(Y, max_steps, power_iters, delta)
                                  : orc::pseudo_svd(Y, rf_seed);
    auto t1 = std::chrono::steady_clock::now();
    const orc::QM psi_h = orc::qmat_mul(Psi, rep.h);
    const orc::QM X = orc::solve_quaternion_linear(psi_h, W);
    auto t2 = std::chrono::steady_clock::now();
    store(rep.h, h);
    store(X, x);
    *kb = rep.kappa_before;
    *ka = rep.kappa_after;
    *steps = rep.steps;
    if (t_rf) *t_rf = std::chrono::duration<double>(t1 - t0).count();
    if (t_solve) *t_solve = std::chrono::duration<double>(t2 - t1).count();
  });
}

// Row-blocked ||A - H X||_F^2 and ||A||_F^2 (sketching.cpp:270-271 without
// the two full-size temporaries).
int orc_residual_sq(Index m, Index n, Index s, const double* a, const double* h, const double* x,
                    double* res_sq, double* a_sq) {
  return guard([&] {
    const orc::QM X = load(x, s, n);
    const std::size_t mn = static_cast<std::size_t>(m * n), ms = static_cast<std::size_t>(m * s);
    double rs = 0.0, as = 0.0;
    const Index blk = 256;
    for (Index r0 = 0; r0 < m; r0 += blk) {
      const Index r1 = std::min(m, r0 + blk);
      orc::QM Hb(r1 - r0, s), Ab(r1 - r0, n);
      for (int p = 0; p < 4; ++p) {
        std::memcpy(Hb.p[p].data(), h + p * ms + r0 * s, sizeof(double) * (r1 - r0) * s);
        std::memcpy(Ab.p[p].data(), a + p * mn + r0 * n, sizeof(double) * (r1 - r0) * n);
      }
      const orc::QM hx = orc::qmat_mul(Hb, X);
      for (int p = 0; p < 4; ++p)
        for (std::size_t i = 0; i < Ab.p[p].size(); ++i) {
          const double d = Ab.p[p][i] - hx.p[p][i];
          rs += d * d;
          as += Ab.p[p][i] * Ab.p[p][i];
        }
    }
    *res_sq = rs;
    *a_sq = as;
  });
}

// truncate_stage (sketching.cpp:196-211): h_out (m x r), sigma (r), v (n x r).
int orc_truncate_stage(Index m, Index s, Index n, const double* h, const double* x, Index r,
                       double* h_out, double* sigma, double* v_out) {
  return guard([&] {
    if (r < 1 || r > s) orc::param("truncate_stage: need 1 <= r <= s");
    const orc::QM H = load(h, m, s), X = load(x, s, n);
    auto f = orc::qsvd(X);
    orc::QM ur(s, r), vr(n, r);
    for (Index j = 0; j < r; ++j) {
      for (Index i = 0; i < s; ++i) {
        double q[4];
        f.u.get(i, j, q);
        ur.set(i, j, q);
      }
      for (Index i = 0; i < n; ++i) {
        double q[4];
        f.v.get(i, j, q);
        vr.set(i, j, q);
      }
      sigma[j] = f.sigma[j];
    }
    store(orc::qmat_mul(H, ur), h_out);
    store(vr, v_out);
  });
}

}  // extern "C"
