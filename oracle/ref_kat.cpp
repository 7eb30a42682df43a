// ref_kat.cpp -- TEST INFRASTRUCTURE ONLY.  Known-answer vectors produced by
// the REFERENCE's own code: proj/include/qlra/rng.hpp (CounterRng,
// SequentialRng, mix64) and proj/include/qlra/quaternion.hpp (Hamilton
// product), compiled in place from /root/reference by oracle/Makefile.ref
// (outputs only into oracle/_ref/).  The rest of the reference needs Eigen
// (absent), so entry_value (proj/src/sketching.cpp:27-51) is restated here in
// terms of the reference's CounterRng to pin the test-matrix draws.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include "qlra/rng.hpp"
#include "qlra/quaternion.hpp"

using namespace qlra;

static double entry_value(const CounterRng& s, int kind, double density, std::uint64_t idx) {
  const std::uint64_t base = 4 * idx;
  switch (kind) {
    case 0: { const double u1 = s.uniform_at(base), u2 = s.uniform_at(base + 1);
              return std::sqrt(-2.0 * std::log1p(-u1)) * std::cos(2.0 * M_PI * u2); }
    case 1: return (s.u64_at(base + 3) & 1u) ? 1.0 : -1.0;
    case 2: { if (s.uniform_at(base + 2) >= density) return 0.0;
              const double u1 = s.uniform_at(base), u2 = s.uniform_at(base + 1);
              return std::sqrt(-2.0 * std::log1p(-u1)) * std::cos(2.0 * M_PI * u2) / std::sqrt(density); }
    default: if (s.uniform_at(base + 2) >= density) return 0.0;
             return ((s.u64_at(base + 3) & 1u) ? 1.0 : -1.0) / std::sqrt(density);
  }
}

static void hexd(double v, bool comma) { std::uint64_t b; __builtin_memcpy(&b, &v, 8); printf("\"%016llx\"%s", (unsigned long long)b, comma ? "," : ""); }

int main() {
  printf("{\n\"mix64\": [");
  const std::uint64_t zs[] = {0ull, 1ull, 2ull, 0x9E3779B97F4A7C15ull, 0xFFFFFFFFFFFFFFFFull, 123456789ull};
  for (int i = 0; i < 6; ++i) printf("\"%016llx\"%s", (unsigned long long)mix64(zs[i]), i < 5 ? "," : "");
  printf("],\n\"keys\": [");
  const std::uint64_t seeds[] = {0, 1, 2, 7, 100, 0x9E3779B9ull, 0x455053ull};
  for (int i = 0; i < 7; ++i) {
    CounterRng r(seeds[i]);
    printf("{\"seed\": %llu, \"key\": \"%016llx\", \"sub\": [", (unsigned long long)seeds[i], (unsigned long long)r.key());
    for (int p = 0; p < 4; ++p) printf("\"%016llx\"%s", (unsigned long long)r.substream(p).key(), p < 3 ? "," : "");
    printf("], \"u64\": [");
    for (int c = 0; c < 8; ++c) printf("\"%016llx\"%s", (unsigned long long)r.u64_at(c), c < 7 ? "," : "");
    printf("], \"uniform\": [");
    for (int c = 0; c < 8; ++c) hexd(r.uniform_at(c), c < 7);
    printf("], \"gaussian_at\": [");
    for (int c = 0; c < 8; ++c) hexd(r.gaussian_at(c), c < 7);
    printf("], \"seq_gaussian\": [");
    SequentialRng q(r);
    for (int c = 0; c < 8; ++c) hexd(q.next_gaussian(), c < 7);
    printf("]}%s\n", i < 6 ? "," : "");
  }
  // test-matrix entries: kind, rows, cols, seed, density -> 4 planes of the full matrix
  printf("],\n\"test_matrices\": [");
  struct S { int kind; long rows, cols; std::uint64_t seed; double density; } specs[] = {
    {0, 6, 5, 1, 1.0}, {0, 4, 7, 2, 1.0}, {1, 5, 4, 3, 1.0}, {2, 6, 6, 15, 0.3}, {3, 5, 5, 9, 0.5}, {0, 3, 3, 0x455053ull, 1.0}};
  for (int si = 0; si < 6; ++si) {
    const S& sp = specs[si];
    printf("{\"kind\": %d, \"rows\": %ld, \"cols\": %ld, \"seed\": %llu, \"density\": %.17g, \"planes\": [",
           sp.kind, sp.rows, sp.cols, (unsigned long long)sp.seed, sp.density);
    const CounterRng root(sp.seed);
    for (int p = 0; p < 4; ++p) {
      const CounterRng st = root.substream(p);
      printf("[");
      for (long i = 0; i < sp.rows; ++i)
        for (long j = 0; j < sp.cols; ++j)
          hexd(entry_value(st, sp.kind, sp.density, (std::uint64_t)(i * sp.cols + j)), !(i == sp.rows - 1 && j == sp.cols - 1));
      printf("]%s", p < 3 ? "," : "");
    }
    printf("]}%s\n", si < 5 ? "," : "");
  }
  // Hamilton products (quaternion.hpp:33-38)
  printf("],\n\"products\": [");
  const Quaternion qs[] = {{0,1,0,0},{0,0,1,0},{0,0,0,1},{1,1,0,0},{1,0,1,0},{0.5,-1.25,2.0,3.5},{-2.0,0.75,-0.125,1.5}};
  bool first = true;
  for (int a = 0; a < 7; ++a) for (int b = 0; b < 7; ++b) {
    const Quaternion r = qs[a] * qs[b];
    printf("%s[%d,%d,%.17g,%.17g,%.17g,%.17g]", first ? "" : ",", a, b, r.w, r.x, r.y, r.z);
    first = false;
  }
  printf("],\n\"operands\": [");
  for (int a = 0; a < 7; ++a) printf("[%.17g,%.17g,%.17g,%.17g]%s", qs[a].w, qs[a].x, qs[a].y, qs[a].z, a < 6 ? "," : "");
  printf("]\n}\n");
  return 0;
}
