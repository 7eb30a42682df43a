// sketch.cu -- K1+K2: the dual sketch Y += A Omega, W += Psi A.
//
// Replaces sketch_update_rows (proj/src/sketching.cpp:125-139), i.e.
// gen_test_matrix(Omega) + qmat_mul_accumulate_ordered(Y, A, Omega) +
// gen_test_matrix_cols(Psi, rows) + qmat_mul_accumulate_ordered(W, Psi, A).
//
// v1 layout: Omega (n x s) and the Psi column slice (l x b) are generated into
// HBM by K1 and both products run on the DFMA quaternion GEMM.
#include "common.cuh"
#include "kernels.cuh"

namespace qlra_dev {

const char* sketch_kernel_name() { return "qgemm_dfma_64x64x8_v1"; }

void sketch_update_rows(Ctx& ctx, const qlra_spec_t& omega, const qlra_spec_t& psi, int64_t row0,
                        const QView& block, const QView& y_rows, const QView& w) {
  const int64_t b = block.rows, n = block.cols, s = omega.cols, l = psi.rows;
  if (b == 0) return;
  DevQMat om(ctx, n, s);
  launch_gen(ctx.stream, omega, 0, 0, n, s, om.v, false);
  qgemm(ctx, QLRA_OP_N, QLRA_OP_N, 1.0, block, om.v, 1.0, y_rows);
  DevQMat ps(ctx, l, b);
  launch_gen(ctx.stream, psi, 0, row0, l, b, ps.v, false);
  qgemm(ctx, QLRA_OP_N, QLRA_OP_N, 1.0, ps.v, block, 1.0, w);
}

}  // namespace qlra_dev
