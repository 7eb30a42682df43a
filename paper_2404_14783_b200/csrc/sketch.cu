// sketch.cu -- K1+K2: the fused dual sketch  Y += A Omega,  W += Psi A.
//
// Replaces sketch_update_rows (proj/src/sketching.cpp:125-139):
// gen_test_matrix(Omega) + qmat_mul_accumulate_ordered(Y, A, Omega) +
// gen_test_matrix_cols(Psi, rows) + qmat_mul_accumulate_ordered(W, Psi, A).
//
// The block of A is walked in row panels sized to stay resident in the 126 MB
// L2.  Each panel is ONE launch of sketch_fused_kernel whose CTAs are either
// Y-tasks (64x64 tile of Y_panel = A_panel * Omega over a K-chunk of the n
// columns) or W-tasks (64x64 tile of W += Psi[:, panel] * A_panel over a
// chunk of the panel rows), both on the DMMA tile core (qtile.cuh).  The
// panel is read from HBM once and re-served from L2 to every task that
// stages it, so HBM traffic for A is 32*m*n bytes -- the "A is read once"
// contract of the one-pass method.  Split-K partials
// go to workspaces reduced in fixed order afterwards: deterministic, no
// atomics.  Omega (n x s) and the Psi column slice (l x b) are generated on
// device by K1 (embed.cu) from the reference's counter RNG.
#include <array>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "qtile.cuh"

namespace qlra_dev {

namespace {

using qt::BK;
using qt::BM;
using qt::BN;
using qt::NT;

struct FusedArgs {
  qt::Operands yop;  // A_panel (k-fast) x Omega (j-fast): M = panel rows, N = s, K = n
  qt::Operands wop;  // Psi_panel (k-fast) x A_panel (j-fast): M = l, N = n, K = panel rows
  int64_t ky, kw;    // K extents
  int y_tm, y_tn, zy;
  int64_t ky_chunk;
  int w_tm, w_tn, zw;
  int64_t kw_chunk;
  int y_tnf, w_tmf;  // full (no padding) Y column tiles / W row tiles
  double* y[4];
  int64_t ldy;
  double* yp;  // [zy][4][My][Ny] partials when zy > 1
  double* w[4];
  int64_t ldw;
  double* wp;  // [zw][4][l][n] partials when zw > 1
};

__device__ __forceinline__ void store_tile(const qt::Acc& acc, int64_t i0, int64_t j0, int64_t M,
                                           int64_t N, double* const* c, int64_t ldc,
                                           double* part, bool rmw) {
#pragma unroll
  for (int rb = 0; rb < qt::WRB; ++rb) {
    const int64_t gi = i0 + qt::acc_row(rb);
    if (gi >= M) continue;
#pragma unroll
    for (int cb = 0; cb < qt::WCB; ++cb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gj = j0 + qt::acc_col(cb) + h;
        if (gj >= N) continue;
        if (part) {
#pragma unroll
          for (int p = 0; p < 4; ++p) part[(int64_t)p * M * N + gi * N + gj] = acc[rb][cb][p][h];
        } else {
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            double* dst = c[p] + gi * ldc + gj;
            *dst = rmw ? *dst + acc[rb][cb][p][h] : acc[rb][cb][p][h];
          }
        }
      }
  }
}

// Task order = longest first (LPT list scheduling by the hardware CTA
// dispatcher): full W tiles, full Y tiles, then the Y tiles of the padded
// last column tile (s % 64 != 0) and the W tiles of the padded last row tile
// (l % 64 != 0), whose out-of-range 8x8 blocks issue no DMMA (qtile.cuh).
__global__ void __launch_bounds__(NT, 1) sketch_fused_kernel(FusedArgs f) {
  extern __shared__ __align__(16) double smem[];
  qt::Acc acc;
  qt::zero_acc(acc);
  const int nwf = f.w_tmf * f.w_tn * f.zw;
  const int nyf = f.y_tm * f.y_tnf * f.zy;
  const int nyp = f.y_tm * (f.y_tn - f.y_tnf) * f.zy;
  int t = blockIdx.x;
  bool is_w;
  int tm, tn, z;
  if (t < nwf) {
    is_w = true;
    z = t % f.zw; t /= f.zw;
    tm = t % f.w_tmf; tn = t / f.w_tmf;  // a-tiles fastest: neighbours share A columns
  } else if ((t -= nwf) < nyf) {
    is_w = false;
    z = t % f.zy; t /= f.zy;
    tn = t % f.y_tnf; tm = t / f.y_tnf;
  } else if ((t -= nyf) < nyp) {
    is_w = false;
    z = t % f.zy; t /= f.zy;
    tn = f.y_tnf + t % (f.y_tn - f.y_tnf); tm = t / (f.y_tn - f.y_tnf);
  } else {
    t -= nyp;
    is_w = true;
    z = t % f.zw; t /= f.zw;
    tm = f.w_tmf + t % (f.w_tm - f.w_tmf); tn = t / (f.w_tm - f.w_tmf);
  }
  if (!is_w) {
    const int64_t kb = (int64_t)z * f.ky_chunk, ke = min(f.ky, kb + f.ky_chunk);
    qt::mma_tile<false, false>(f.yop, smem, (int64_t)tm * BM, (int64_t)tn * BN, kb, ke, acc);
    double* part = f.zy > 1 ? f.yp + (int64_t)z * 4 * f.yop.M * f.yop.N : nullptr;
    store_tile(acc, (int64_t)tm * BM, (int64_t)tn * BN, f.yop.M, f.yop.N, f.y, f.ldy, part, true);
  } else {
    const int64_t kb = (int64_t)z * f.kw_chunk, ke = min(f.kw, kb + f.kw_chunk);
    qt::mma_tile<false, false>(f.wop, smem, (int64_t)tm * BM, (int64_t)tn * BN, kb, ke, acc);
    double* part = f.zw > 1 ? f.wp + (int64_t)z * 4 * f.wop.M * f.wop.N : nullptr;
    store_tile(acc, (int64_t)tm * BM, (int64_t)tn * BN, f.wop.M, f.wop.N, f.w, f.ldw, part, true);
  }
}


}  // namespace

const char* sketch_kernel_name() { return "sketch_fused_kernel(dmma_64x64x8, mbarrier ring, panels <= 2 GB)"; }

namespace {

struct SketchWork {
  DeviceBuffer yp, wp;  // split-K partial workspaces, grown on demand
};

// Makespan of one fused launch under greedy list scheduling on 148 SMs
// (1 CTA per SM), tasks in kernel order.
double simulate_panel(int64_t rp, int64_t n, int64_t s, int64_t l, int zy, int zw) {
  const int64_t kyc = ((n + zy - 1) / zy + BK - 1) / BK * BK, kwc = ((rp + zw - 1) / zw + BK - 1) / BK * BK;
  const int64_t ny_chunks = (n + kyc - 1) / kyc, nw_chunks = (rp + kwc - 1) / kwc;
  const int64_t y_tm = (rp + BM - 1) / BM, y_tn = (s + BN - 1) / BN, w_tm = (l + BM - 1) / BM,
                w_tn = (n + BN - 1) / BN;
  const int64_t y_tnf = s / BN, w_tmf = l / BM;
  auto frac = [](int64_t valid) { return (double)((valid + 7) / 8) / 8.0; };  // 8-blocks of 64
  const double y_part = frac(s - y_tnf * BN), w_part = frac(l - w_tmf * BM);
  struct Group { int64_t count; double cost; };
  const Group groups[4] = {{w_tmf * w_tn * nw_chunks, (double)(kwc / BK)},
                           {y_tm * y_tnf * ny_chunks, (double)(kyc / BK)},
                           {y_tm * (y_tn - y_tnf) * ny_chunks, (double)(kyc / BK) * y_part},
                           {(w_tm - w_tmf) * w_tn * nw_chunks, (double)(kwc / BK) * w_part}};
  // Greedy assignment on buckets of SMs that free at the same time (tasks of
  // a group cost the same, so whole buckets advance together): O(tasks/148)
  // per group instead of a heap operation per CTA.
  std::map<double, int64_t> sm{{0.0, 148}};
  for (const Group& g : groups) {
    const double d = g.cost + 2.0;  // + prologue/epilogue (~2 k-steps)
    int64_t c = g.count;
    while (c > 0) {
      auto it = sm.begin();
      const double t0 = it->first;
      const int64_t k = it->second;
      sm.erase(it);
      const int64_t take = std::min(c, k);
      if (k > take) sm[t0] += k - take;
      sm[t0 + d] += take;
      c -= take;
    }
  }
  const double mk = sm.rbegin()->first;
  // split-K partials cost a reduction pass over zy Y / zw W copies
  // (~1 k-step of time per 25 MB of partials)
  const double red = (zy > 1 ? (double)zy * rp * s : 0.0) + (zw > 1 ? (double)zw * l * n : 0.0);
  return mk + red * 32.0 / 25e6;
}

std::pair<int, int> choose_panel_splits(int64_t rp, int64_t n, int64_t s, int64_t l) {
  static std::mutex mu;
  static std::map<std::array<int64_t, 4>, std::pair<int, int>> cache;
  const std::array<int64_t, 4> key{rp, n, s, l};
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  const int64_t wt = ((l + BM - 1) / BM) * ((n + BN - 1) / BN);
  // W split-K only while W has fewer than 4 waves of tiles (its partials are
  // l x n each: 868 MB at C4)
  const int zw_max = wt >= 4 * 148 ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(wt >= 148 ? 8 : 64, rp / 64));
  const int zy_max = (int)std::max<int64_t>(1, std::min<int64_t>(256, n / 32));
  // candidates: every value up to 16, then geometric steps of ~12%
  auto candidates = [](int hi) {
    std::vector<int> v;
    for (int z = 1; z <= hi; z = z < 16 ? z + 1 : std::max(z + 1, z * 9 / 8)) v.push_back(z);
    if (v.back() != hi) v.push_back(hi);
    return v;
  };
  double best = 1e300;
  std::pair<int, int> arg{1, 1};
  for (int zw : candidates(zw_max))
    for (int zy : candidates(zy_max)) {
      const double mk = simulate_panel(rp, n, s, l, zy, zw);
      if (mk < best - 1e-9) { best = mk; arg = {zy, zw}; }
    }
  {
    std::lock_guard<std::mutex> lock(mu);
    cache[key] = arg;
  }
  if (std::getenv("QLRA_DEBUG_SPLITS")) {
    // ideal = total cost / 148 (perfect balance, no per-CTA overhead)
    const int64_t y_tm = (rp + BM - 1) / BM, y_tn = (s + BN - 1) / BN, w_tm = (l + BM - 1) / BM,
                  w_tn = (n + BN - 1) / BN;
    auto frac = [](int64_t valid) { return (double)((valid + 7) / 8) / 8.0; };
    const double yc = (double)y_tm * ((double)(s / BN) + (y_tn > s / BN ? frac(s - (s / BN) * BN) : 0.0)) * (double)n / BK;
    const double wc = (double)w_tn * ((double)(l / BM) + (w_tm > l / BM ? frac(l - (l / BM) * BM) : 0.0)) * (double)rp / BK;
    std::fprintf(stderr, "[qlra] panel %lldx%lld s=%lld l=%lld: zy=%d zw=%d makespan %.0f ideal %.0f (%.1f%%)\n",
                 (long long)rp, (long long)n, (long long)s, (long long)l, arg.first, arg.second, best,
                 (yc + wc) / 148.0, 100.0 * (yc + wc) / 148.0 / best);
  }
  return arg;
}

// One fused launch (+ ordered partial reductions) for a row panel `ap` of A
// whose Psi columns are ps[:, pc0 : pc0 + ap.rows].
void sketch_panel(Ctx& ctx, const QView& om, const QView& ps, int64_t pc0, const QView& ap,
                  const QView& yv, const QView& w, SketchWork& ws) {
  const int64_t rp = ap.rows, n = ap.cols, s = om.cols, l = ps.rows;
  const int w_tm = (int)((l + BM - 1) / BM), w_tn = (int)((n + BN - 1) / BN);
  DeviceBuffer& yp = ws.yp;
  DeviceBuffer& wp = ws.wp;
  {
    FusedArgs f{};
    for (int p = 0; p < 4; ++p) {
      f.yop.a[p] = ap.p[p];
      f.yop.b[p] = om.p[p];
      f.wop.a[p] = ps.p[p] + pc0;  // Psi[:, pc0:pc0+rp]
      f.wop.b[p] = ap.p[p];
      f.y[p] = yv.p[p];
      f.w[p] = w.p[p];
    }
    f.yop.a_si = ap.ld; f.yop.a_sk = 1; f.yop.b_sk = om.ld; f.yop.b_sj = 1;
    f.yop.M = rp; f.yop.N = s;
    f.wop.a_si = ps.ld; f.wop.a_sk = 1; f.wop.b_sk = ap.ld; f.wop.b_sj = 1;
    f.wop.M = l; f.wop.N = n;
    f.ky = n;
    f.kw = rp;
    f.ldy = yv.ld;
    f.ldw = w.ld;
    f.y_tm = (int)((rp + BM - 1) / BM);
    f.y_tn = (int)((s + BN - 1) / BN);
    f.w_tm = w_tm;
    f.w_tn = w_tn;
    // Split counts (zy over n, zw over the panel rows) from a simulation of
    // the dispatcher: CTAs in kernel order (longest first) go to the SM that
    // frees first; cost = k-steps x fraction of 8x8 blocks inside M x N.
    // Cached per panel shape.
    f.y_tnf = (int)(s / BN);
    f.w_tmf = (int)(l / BM);
    const auto choice = choose_panel_splits(rp, n, s, l);
    const int best_zy = choice.first, best_zw = choice.second;
    f.kw_chunk = ((rp + best_zw - 1) / best_zw + BK - 1) / BK * BK;
    f.zw = (int)((rp + f.kw_chunk - 1) / f.kw_chunk);
    f.ky_chunk = ((n + best_zy - 1) / best_zy + BK - 1) / BK * BK;
    f.zy = (int)((n + f.ky_chunk - 1) / f.ky_chunk);
    if (f.zy > 1) {
      const size_t need = (size_t)f.zy * 4 * rp * s * sizeof(double);
      if (yp.bytes < need) yp = DeviceBuffer(ctx, need);
      f.yp = yp.as<double>();
    }
    if (f.zw > 1) {
      const size_t need = (size_t)f.zw * 4 * l * n * sizeof(double);
      if (wp.bytes < need) wp = DeviceBuffer(ctx, need);
      f.wp = wp.as<double>();
    }
    const int64_t ctas = (int64_t)f.y_tm * f.y_tn * f.zy + (int64_t)w_tm * w_tn * f.zw;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx.ktimer.on) {
      if (!ctx.ktimer.pool.empty()) {
        e0 = ctx.ktimer.pool.back().first;
        e1 = ctx.ktimer.pool.back().second;
        ctx.ktimer.pool.pop_back();
      } else {
        QLRA_CUDA(cudaEventCreate(&e0));
        QLRA_CUDA(cudaEventCreate(&e1));
      }
      QLRA_CUDA(cudaEventRecord(e0, ctx.stream));
    }
    sketch_fused_kernel<<<(unsigned)ctas, NT, qt::SMEM_BYTES, ctx.stream>>>(f);
    QLRA_LAUNCH_CHECK();
    count_launch();
    if (ctx.ktimer.on) {
      QLRA_CUDA(cudaEventRecord(e1, ctx.stream));
      ctx.ktimer.ev.emplace_back(e0, e1);
      ctx.ktimer.flops += 32.0 * (double)rp * (double)n * (double)(s + l);
      ctx.ktimer.a_bytes += 32.0 * (double)rp * (double)n;
      ++ctx.ktimer.launches;
    }
    if (f.zy > 1) splitk_reduce(ctx, f.yp, f.zy, yv, 1.0, 1.0);
    if (f.zw > 1) splitk_reduce(ctx, f.wp, f.zw, w, 1.0, 1.0);
  }
}

void set_kernel_attrs() {
  set_func_attr((const void*)sketch_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                (int)qt::SMEM_BYTES);
}

// Rows per fused launch.  Device-resident A: panels of up to kPanelBytes --
// the kernel does ~300 flop per byte of A, so an A tile re-read from HBM
// instead of L2 costs nothing measurable, while one long launch balances the
// CTAs over the SMs far better than many short ones (C2: 16.3 ms as one
// launch vs 19.9 ms as 32 L2-sized panels).  Host-streamed A: chunks of
// kStreamBytes so the H2D copy of the next chunk overlaps the sketch of this
// one (about 16 chunks per block, at least kStreamBytes each).  Multiples of
// 64 rows, at least 256.  QLRA_PANEL_BYTES / QLRA_STREAM_BYTES override
// (tuning).
constexpr double kPanelBytes = 2e9;
constexpr double kStreamBytes = 64e6;
double env_or(const char* name, double dflt) {
  const char* e = std::getenv(name);
  return e ? std::atof(e) : dflt;
}
int64_t rows_for(double bytes, int64_t n, int64_t b) {
  int64_t R = (int64_t)(bytes / (32.0 * (double)n));
  R = std::max<int64_t>(256, (R / 64) * 64);
  return std::min<int64_t>(R, ((b + 63) / 64) * 64);
}
int64_t panel_rows(int64_t n, int64_t b) {
  static const double bytes = env_or("QLRA_PANEL_BYTES", kPanelBytes);
  return rows_for(bytes, n, b);
}
int64_t stream_rows(int64_t n, int64_t b) {
  // ~16 chunks per block (each DMA call and chunk boundary costs; measured
  // C2: 16 x 96 MB 28.6 ms vs 32 x 48 MB 29.0 ms, plain copy 27.6 ms), never
  // below kStreamBytes: small chunks of a narrow A (C5: n = 300) make short,
  // inefficient launches
  static const double floor_bytes = env_or("QLRA_STREAM_BYTES", kStreamBytes);
  const double bytes = std::max(floor_bytes, 32.0 * (double)n * (double)b / 16.0);
  return rows_for(bytes, n, b);
}

}  // namespace

namespace {
QView view_of_buf(double* base, int64_t rows, int64_t cols) {
  QView v{};
  for (int p = 0; p < 4; ++p) v.p[p] = base + (size_t)p * rows * cols;
  v.rows = rows;
  v.cols = cols;
  v.ld = cols;
  return v;
}
bool same_spec(const qlra_spec_t& a, const qlra_spec_t& b) {
  return a.kind == b.kind && a.rows == b.rows && a.cols == b.cols && a.seed == b.seed && a.density == b.density;
}
}  // namespace

QView psi_for_sketch(Ctx& ctx, const qlra_spec_t& psi, int64_t row0, int64_t rows, DevQMat& tmp) {
  static const double cap = env_or("QLRA_PSI_KEEP_BYTES", 8e9);
  const int64_t l = psi.rows;
  const size_t bytes = (size_t)4 * l * rows * sizeof(double);
  Ctx::PsiKeep& k = ctx.psi_keep;
  k.valid = false;
  if ((double)bytes > cap || bytes == 0) {
    tmp = DevQMat(ctx, l, rows);
    launch_gen(ctx.stream, psi, 0, row0, l, rows, tmp.v, false);
    return tmp.v;
  }
  if (k.bytes < bytes) {
    if (k.buf) QLRA_CUDA(cudaFreeAsync(k.buf, ctx.stream));
    k.buf = nullptr;
    k.bytes = 0;
    QLRA_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&k.buf), bytes, ctx.stream));
    k.bytes = bytes;
  }
  const QView v = view_of_buf(k.buf, l, rows);
  launch_gen(ctx.stream, psi, 0, row0, l, rows, v, false);
  k.valid = true;
  k.spec = psi;
  k.row0 = row0;
  k.rows = rows;
  return v;
}

QView psi_for_solve(Ctx& ctx, const qlra_spec_t& psi, int64_t row0, int64_t rows, DevQMat& tmp) {
  const Ctx::PsiKeep& k = ctx.psi_keep;
  if (k.valid && same_spec(k.spec, psi) && k.row0 == row0 && k.rows == rows) return view_of_buf(k.buf, psi.rows, rows);
  tmp = DevQMat(ctx, psi.rows, rows);
  launch_gen(ctx.stream, psi, 0, row0, psi.rows, rows, tmp.v, false);
  return tmp.v;
}

void psi_keep_release(Ctx& ctx) {
  Ctx::PsiKeep& k = ctx.psi_keep;
  if (k.buf) cudaFreeAsync(k.buf, ctx.stream);
  k = Ctx::PsiKeep{};
}

void sketch_update_rows(Ctx& ctx, const qlra_spec_t& omega, const qlra_spec_t& psi, int64_t row0,
                        const QView& block, const QView& y_rows, const QView& w) {
  const int64_t b = block.rows, n = block.cols, s = omega.cols, l = psi.rows;
  if (b == 0 || n == 0) return;
  set_kernel_attrs();
  DevQMat om(ctx, n, s), ps_tmp;
  launch_gen(ctx.stream, omega, 0, 0, n, s, om.v, false);
  const QView ps = psi_for_sketch(ctx, psi, row0, b, ps_tmp);
  const int64_t R = panel_rows(n, b);
  SketchWork ws;
  for (int64_t r0 = 0; r0 < b; r0 += R) {
    const int64_t rp = std::min(R, b - r0);
    sketch_panel(ctx, om.v, ps, r0, sub(block, r0, 0, rp, n), sub(y_rows, r0, 0, rp, s), w, ws);
  }
}

// Streaming ingestion (sketch_from_source, sketching.cpp:156-167, with the
// source in host memory): row panels are copied H2D on a dedicated stream into
// a double buffer while the previous panel is sketched, so the PCIe transfer
// of A overlaps the FP64 work.  A is still read exactly once.
void sketch_update_rows_host(Ctx& ctx, const qlra_spec_t& omega, const qlra_spec_t& psi,
                             int64_t row0, const QView& host_block, const QView& y_rows,
                             const QView& w, int64_t block_rows) {
  const int64_t b = host_block.rows, n = host_block.cols, s = omega.cols, l = psi.rows;
  if (b == 0 || n == 0) return;
  set_kernel_attrs();
  int64_t R = block_rows > 0 ? block_rows : stream_rows(n, b);
  R = std::min(R, b);
  DevQMat om(ctx, n, s), ps_tmp;
  DevQMat buf[2] = {DevQMat(ctx, R, n), DevQMat(ctx, R, n)};
  cudaStream_t cs;
  QLRA_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaEvent_t copied[2], freed[2];
  for (int i = 0; i < 2; ++i) {
    QLRA_CUDA(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
    QLRA_CUDA(cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming));
  }
  // the buffers were allocated on ctx.stream: the copy stream waits for
  // that, and only that -- Omega / Psi generation below overlaps the first
  // H2D chunk
  QLRA_CUDA(cudaEventRecord(freed[0], ctx.stream));
  QLRA_CUDA(cudaEventRecord(freed[1], ctx.stream));
  launch_gen(ctx.stream, omega, 0, 0, n, s, om.v, false);
  const QView ps = psi_for_sketch(ctx, psi, row0, b, ps_tmp);
  SketchWork ws;
  // The last R rows go in quarter-size chunks: the sketch of the final chunk
  // is the one part of the pipeline nothing overlaps (the copy stream is the
  // bottleneck before it), so it should be short.
  const int64_t tail_start = b > 2 * R ? b - R : b;
  const int64_t Rt = std::max<int64_t>(64, ((R / 4 + 63) / 64) * 64);
  int idx = 0;
  for (int64_t r0 = 0, rp = 0; r0 < b; r0 += rp, idx ^= 1) {
    rp = std::min(r0 >= tail_start ? Rt : std::min(R, tail_start - r0), b - r0);
    const QView dst = sub(buf[idx].v, 0, 0, rp, n);
    QLRA_CUDA(cudaStreamWaitEvent(cs, freed[idx], 0));
    for (int p = 0; p < 4; ++p) {
      const double* src = host_block.p[p] + r0 * host_block.ld;
      if (host_block.ld == n && dst.ld == n) {
        // contiguous rows: one linear DMA (2D copies of narrow rows, e.g.
        // C5's 2400-byte rows, run far below PCIe bandwidth)
        QLRA_CUDA(cudaMemcpyAsync(dst.p[p], src, sizeof(double) * (size_t)(rp * n), cudaMemcpyHostToDevice, cs));
      } else {
        QLRA_CUDA(cudaMemcpy2DAsync(dst.p[p], (size_t)dst.ld * sizeof(double), src,
                                    (size_t)host_block.ld * sizeof(double), (size_t)n * sizeof(double),
                                    (size_t)rp, cudaMemcpyHostToDevice, cs));
      }
    }
    QLRA_CUDA(cudaEventRecord(copied[idx], cs));
    QLRA_CUDA(cudaStreamWaitEvent(ctx.stream, copied[idx], 0));
    sketch_panel(ctx, om.v, ps, r0, dst, sub(y_rows, r0, 0, rp, s), w, ws);
    QLRA_CUDA(cudaEventRecord(freed[idx], ctx.stream));
  }
  QLRA_CUDA(cudaStreamSynchronize(cs));
  for (int i = 0; i < 2; ++i) {
    cudaEventDestroy(copied[i]);
    cudaEventDestroy(freed[i]);
  }
  cudaStreamDestroy(cs);
}

}  // namespace qlra_dev
