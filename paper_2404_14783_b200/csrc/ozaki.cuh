// ozaki.cuh -- the int8 tensor-core sketch engine (ozaki.cu).
#pragma once

#include "kernels.cuh"

namespace qlra_dev {

// true when sketch_update_rows should take the int8 engine for these shapes
bool oz_wanted(const Ctx& c, int64_t n, int64_t s, int64_t l);
int64_t oz_kmax();
bool oz_gemm_tcgen05();
const char* oz_kernel_name();
// C = alpha op(A) op(B) + beta C on the int8 engine when the contraction is
// long enough to pay (false: not taken, nothing launched)
bool oz_gemm_try(Ctx& c, int op_a, int op_b, double alpha, const QView& A, const QView& B, double beta,
                 const QView& C);
// int8 TOPS of back-to-back cuBLASLt 8192^3 int8 GEMMs for ~ms milliseconds
double oz_measure_int8_peak(Ctx& c, double ms);

// One sketch call on the int8 engine: Omega's residues and the embeddings'
// scales are prepared at construction; panel() adds a row panel's Y rows and
// accumulates its W^* products (int32, exact) until flush() recovers W.
struct OzRun {
  Ctx& ctx;
  QView omega, psi;  // Omega (n x s), the Psi block (l x b) of the call
  int64_t n = 0, npad = 0, scols = 0, spad = 0, l = 0, lpad = 0;
  // row pitch of the A / Omega residues: whole 128-byte lines per row, so that
  // the GEMMs' 128-byte operand rows (TMA boxes) never straddle two lines
  int64_t npitch = 0;
  unsigned long long* om_colmax = nullptr;  // device: max |Omega(:, j)| bits
  unsigned long long* ps_rowmax = nullptr;  // device: max |Psi(k, :)| bits
  int8_t* ores = nullptr;                   // Omega residues (128 x s x npad)
  int32_t* cw = nullptr;                    // W^* products (128 x l x npad), int32
  int nmod = 16, tab = 0, beta = 52, nb = 128;  // moduli, CRT table, operand bits, batch (8 nmod)
  int64_t kcap = 0;  // rows per int32 accumulation (epoch)
  bool epoch_open = false;
  int64_t epoch_rows = 0;
  int sigma = 0;  // A' = rint(A 2^sigma) in the open epoch
  // rows: the block's row count (the moduli are chosen from it and n)
  OzRun(Ctx& c, const QView& om, const QView& ps, int64_t rows);

  OzRun(const OzRun&) = delete;
  OzRun& operator=(const OzRun&) = delete;
  // max |a| on `stream` into slot 0..2 (device) and its pinned host copy
  void amax_async(const QView& a, cudaStream_t stream, int slot);
  double amax_host(int slot) const;
  // rows [pc0, pc0 + ap.rows) of the block: Y rows yr += ap Omega; W^*
  // products accumulated; amax bounds max |ap|; headroom: spare bits of the
  // epoch scale for later panels (streamed blocks)
  void panel(int64_t pc0, const QView& ap, const QView& yr, const QView& w, double amax, int headroom);
  // phases of a panel (oz_sketch_block pipelines them over two streams)
  void open_for(int64_t rpad, double amax, int headroom, const QView& w);
  void reserve(int64_t rpad, int buf);
  void prep(int64_t pc0, const QView& ap, int buf, cudaStream_t st);
  void gemms(int64_t R, int buf);
  void recover_y(const QView& yr, int buf, cudaStream_t st);
  void flush(const QView& w);
  void finish(const QView& w);
};

// the whole sketch of a device-resident block; false (nothing added) when A
// holds NaN or inf: the caller takes the FP64 engine
bool oz_sketch_block(Ctx& c, const QView& om, const QView& ps, const QView& block, const QView& y_rows,
                     const QView& w);

}  // namespace qlra_dev
