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

__global__ void __launch_bounds__(NT, 1) sketch_fused_kernel(FusedArgs f) {
  extern __shared__ __align__(16) double smem[];
  qt::Acc acc;
  qt::zero_acc(acc);
  const int ny = f.y_tm * f.y_tn * f.zy;
  int t = blockIdx.x;
  if (t < ny) {
    const int z = t % f.zy;
    t /= f.zy;
    const int tn = t % f.y_tn, tm = t / f.y_tn;
    const int64_t kb = (int64_t)z * f.ky_chunk, ke = min(f.ky, kb + f.ky_chunk);
    qt::mma_tile<false, false>(f.yop, smem, (int64_t)tm * BM, (int64_t)tn * BN, kb, ke, acc);
    double* part = f.zy > 1 ? f.yp + (int64_t)z * 4 * f.yop.M * f.yop.N : nullptr;
    store_tile(acc, (int64_t)tm * BM, (int64_t)tn * BN, f.yop.M, f.yop.N, f.y, f.ldy, part, true);
  } else {
    t -= ny;
    const int z = t % f.zw;
    t /= f.zw;
    const int tm = t % f.w_tm, tn = t / f.w_tm;  // a-tiles fastest: neighbours share A columns
    const int64_t kb = (int64_t)z * f.kw_chunk, ke = min(f.kw, kb + f.kw_chunk);
    qt::mma_tile<false, false>(f.wop, smem, (int64_t)tm * BM, (int64_t)tn * BN, kb, ke, acc);
    double* part = f.zw > 1 ? f.wp + (int64_t)z * 4 * f.wop.M * f.wop.N : nullptr;
    store_tile(acc, (int64_t)tm * BM, (int64_t)tn * BN, f.wop.M, f.wop.N, f.w, f.ldw, part, true);
  }
}

constexpr double kL2Budget = 48e6;  // bytes of A panel kept L2-resident

}  // namespace

const char* sketch_kernel_name() { return "sketch_fused_kernel(dmma_64x64x8,L2-panel)"; }

namespace {

struct SketchWork {
  DeviceBuffer yp, wp;  // split-K partial workspaces, grown on demand
};

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
    // Task lengths (in k-steps) are balanced with a makespan model: every
    // CTA runs one task, the launch takes ~waves * (longest task), and we
    // maximise useful work / (148 * waves * longest).  W is split over the
    // panel rows only when its tiles cannot fill the GPU (C5-like shapes).
    const int64_t wt = (int64_t)w_tm * w_tn, yt = (int64_t)f.y_tm * f.y_tn;
    const double work = (double)yt * n + (double)wt * rp;
    double best = -1.0;
    int best_zw = 1, best_zy = 1;
    const int zw_max = wt >= 148 ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(64, rp / 64));
    for (int zw = 1; zw <= zw_max; ++zw) {
      const int64_t kwc = ((rp + zw - 1) / zw + BK - 1) / BK * BK;
      const int zy_max = (int)std::max<int64_t>(1, std::min<int64_t>(512, n / 32));
      for (int zy = 1; zy <= zy_max; ++zy) {
        const int64_t kyc = ((n + zy - 1) / zy + BK - 1) / BK * BK;
        const int64_t ctas = yt * ((n + kyc - 1) / kyc) + wt * ((rp + kwc - 1) / kwc);
        const int64_t waves = (ctas + 147) / 148;
        const double score = work / (148.0 * (double)waves * (double)std::max(kyc, kwc) + 16.0 * ctas);
        if (score > best) { best = score; best_zw = zw; best_zy = zy; }
      }
    }
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
    const int64_t ctas = yt * f.zy + wt * f.zw;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx.ktimer.on) {
      QLRA_CUDA(cudaEventCreate(&e0));
      QLRA_CUDA(cudaEventCreate(&e1));
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
  static bool attr = false;
  if (!attr) {
    QLRA_CUDA(cudaFuncSetAttribute(sketch_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)qt::SMEM_BYTES));
    attr = true;
  }
}

// Panel rows: L2 budget, multiple of 64, at least 256 (keeps W tasks dense).
int64_t panel_rows(int64_t n, int64_t b) {
  int64_t R = (int64_t)(kL2Budget / (32.0 * (double)n));
  R = std::max<int64_t>(256, (R / 64) * 64);
  return std::min<int64_t>(R, ((b + 63) / 64) * 64);
}

}  // namespace

void sketch_update_rows(Ctx& ctx, const qlra_spec_t& omega, const qlra_spec_t& psi, int64_t row0,
                        const QView& block, const QView& y_rows, const QView& w) {
  const int64_t b = block.rows, n = block.cols, s = omega.cols, l = psi.rows;
  if (b == 0 || n == 0) return;
  set_kernel_attrs();
  DevQMat om(ctx, n, s);
  launch_gen(ctx.stream, omega, 0, 0, n, s, om.v, false);
  DevQMat ps(ctx, l, b);
  launch_gen(ctx.stream, psi, 0, row0, l, b, ps.v, false);
  const int64_t R = panel_rows(n, b);
  SketchWork ws;
  for (int64_t r0 = 0; r0 < b; r0 += R) {
    const int64_t rp = std::min(R, b - r0);
    sketch_panel(ctx, om.v, ps.v, r0, sub(block, r0, 0, rp, n), sub(y_rows, r0, 0, rp, s), w, ws);
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
  DevQMat om(ctx, n, s);
  launch_gen(ctx.stream, omega, 0, 0, n, s, om.v, false);
  DevQMat ps(ctx, l, b);
  launch_gen(ctx.stream, psi, 0, row0, l, b, ps.v, false);
  int64_t R = block_rows > 0 ? block_rows : panel_rows(n, b);
  R = std::min(R, b);
  DevQMat buf[2] = {DevQMat(ctx, R, n), DevQMat(ctx, R, n)};
  cudaStream_t cs;
  QLRA_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaEvent_t copied[2], freed[2];
  for (int i = 0; i < 2; ++i) {
    QLRA_CUDA(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
    QLRA_CUDA(cudaEventCreateWithFlags(&freed[i], cudaEventDisableTiming));
  }
  // buffers were allocated on ctx.stream: make the copy stream wait for that
  QLRA_CUDA(cudaEventRecord(freed[0], ctx.stream));
  QLRA_CUDA(cudaEventRecord(freed[1], ctx.stream));
  SketchWork ws;
  int idx = 0;
  for (int64_t r0 = 0; r0 < b; r0 += R, idx ^= 1) {
    const int64_t rp = std::min(R, b - r0);
    const QView dst = sub(buf[idx].v, 0, 0, rp, n);
    QLRA_CUDA(cudaStreamWaitEvent(cs, freed[idx], 0));
    for (int p = 0; p < 4; ++p)
      QLRA_CUDA(cudaMemcpy2DAsync(dst.p[p], (size_t)dst.ld * sizeof(double),
                                  host_block.p[p] + r0 * host_block.ld,
                                  (size_t)host_block.ld * sizeof(double),
                                  (size_t)n * sizeof(double), (size_t)rp, cudaMemcpyHostToDevice, cs));
    QLRA_CUDA(cudaEventRecord(copied[idx], cs));
    QLRA_CUDA(cudaStreamWaitEvent(ctx.stream, copied[idx], 0));
    sketch_panel(ctx, om.v, ps.v, r0, dst, sub(y_rows, r0, 0, rp, s), w, ws);
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
