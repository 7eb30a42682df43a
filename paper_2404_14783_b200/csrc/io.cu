// io.cu -- QMAT1 / QSKT1 checkpoint I/O for device matrices and sketch state
// (SURVEY 8(f) #3), byte-compatible with the reference (proj/src/io.cpp:77-145,
// proj/include/qlra/io.hpp:13-44):
//   QMAT1 = "QMAT1\0", u64 rows, u64 cols, 4 row-major little-endian f64 planes
//   QSKT1 = "QSKT1\0", omega spec, psi spec (u32 kind, u64 rows, u64 cols,
//           u64 seed, f64 density), u64 r, s, l, then Y and W as QMAT1.
// Plus streaming ingestion from a QMAT1 file (QmatFileSource + sketch_from_source,
// io.cpp:213-239, sketching.cpp:156-167): row blocks are read into pinned host
// buffers and pushed through the overlapped H2D + fused-sketch pipeline.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace qlra_dev {

namespace {

constexpr char kQmatMagic[6] = {'Q', 'M', 'A', 'T', '1', '\0'};
constexpr char kSketchMagic[6] = {'Q', 'S', 'K', 'T', '1', '\0'};
constexpr std::streamoff kQmatHeaderBytes = 6 + 8 + 8;

void put_u64(std::ostream& os, uint64_t v) { os.write(reinterpret_cast<const char*>(&v), 8); }
void put_f64(std::ostream& os, double v) { os.write(reinterpret_cast<const char*>(&v), 8); }
uint64_t get_u64(std::istream& is) {
  uint64_t v = 0;
  if (!is.read(reinterpret_cast<char*>(&v), 8)) fail(QLRA_ERR_IO, "truncated file: expected u64");
  return v;
}
double get_f64(std::istream& is) {
  double v = 0;
  if (!is.read(reinterpret_cast<char*>(&v), 8)) fail(QLRA_ERR_IO, "truncated file: expected f64");
  return v;
}
void expect_magic(std::istream& is, const char (&magic)[6], const char* what) {
  char buf[6];
  if (!is.read(buf, 6) || std::memcmp(buf, magic, 6) != 0)
    fail(QLRA_ERR_IO, std::string("not a ") + what + " file");
}
void put_spec(std::ostream& os, const qlra_spec_t& s) {
  const uint32_t tag = (uint32_t)s.kind;
  os.write(reinterpret_cast<const char*>(&tag), 4);
  put_u64(os, (uint64_t)s.rows);
  put_u64(os, (uint64_t)s.cols);
  put_u64(os, s.seed);
  put_f64(os, s.density);
}
qlra_spec_t get_spec(std::istream& is) {
  uint32_t tag = 0;
  if (!is.read(reinterpret_cast<char*>(&tag), 4)) fail(QLRA_ERR_IO, "truncated sketch file: spec record");
  if (tag > 3) fail(QLRA_ERR_IO, "sketch file: unknown test matrix kind tag");
  qlra_spec_t s;
  s.kind = (int32_t)tag;
  s.rows = (int64_t)get_u64(is);
  s.cols = (int64_t)get_u64(is);
  s.seed = get_u64(is);
  s.density = get_f64(is);
  return s;
}

// device planes -> stream (row-major, dense), one plane at a time
void write_planes(Ctx& ctx, std::ostream& os, const QView& m) {
  put_u64(os, (uint64_t)m.rows);
  put_u64(os, (uint64_t)m.cols);
  std::vector<double> buf((size_t)(m.rows * m.cols));
  for (int p = 0; p < 4; ++p) {
    if (!buf.empty()) {
      QLRA_CUDA(cudaMemcpy2DAsync(buf.data(), sizeof(double) * m.cols, m.p[p], sizeof(double) * m.ld,
                                  sizeof(double) * m.cols, (size_t)m.rows, cudaMemcpyDeviceToHost,
                                  ctx.stream));
      QLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    }
    os.write(reinterpret_cast<const char*>(buf.data()), (std::streamsize)(buf.size() * sizeof(double)));
  }
  if (!os) fail(QLRA_ERR_IO, "write_qmat: stream failure");
}

void read_planes(Ctx& ctx, std::istream& is, const QView& m) {
  const int64_t rows = (int64_t)get_u64(is), cols = (int64_t)get_u64(is);
  if (rows != m.rows || cols != m.cols) fail(QLRA_ERR_SHAPE, "read_qmat: destination shape mismatch");
  std::vector<double> buf((size_t)(rows * cols));
  for (int p = 0; p < 4; ++p) {
    if (!is.read(reinterpret_cast<char*>(buf.data()), (std::streamsize)(buf.size() * sizeof(double))))
      fail(QLRA_ERR_IO, "read_qmat: truncated plane data");
    if (!buf.empty()) {
      QLRA_CUDA(cudaMemcpy2DAsync(m.p[p], sizeof(double) * m.ld, buf.data(), sizeof(double) * cols,
                                  sizeof(double) * cols, (size_t)rows, cudaMemcpyHostToDevice, ctx.stream));
      QLRA_CUDA(cudaStreamSynchronize(ctx.stream));
    }
  }
}

}  // namespace

void write_qmat(Ctx& ctx, const std::string& path, const QView& m) {
  std::ofstream os(path, std::ios::binary);
  if (!os) fail(QLRA_ERR_IO, "cannot open for writing: " + path);
  os.write(kQmatMagic, 6);
  write_planes(ctx, os, m);
}

void qmat_header(const std::string& path, int64_t* rows, int64_t* cols) {
  std::ifstream is(path, std::ios::binary);
  if (!is) fail(QLRA_ERR_IO, "cannot open: " + path);
  expect_magic(is, kQmatMagic, "QMAT1");
  *rows = (int64_t)get_u64(is);
  *cols = (int64_t)get_u64(is);
}

void read_qmat(Ctx& ctx, const std::string& path, const QView& m) {
  std::ifstream is(path, std::ios::binary);
  if (!is) fail(QLRA_ERR_IO, "cannot open: " + path);
  expect_magic(is, kQmatMagic, "QMAT1");
  read_planes(ctx, is, m);
}

void write_sketch(Ctx& ctx, const std::string& path, const qlra_spec_t& om, const qlra_spec_t& ps,
                  int64_t r, int64_t s, int64_t l, const QView& y, const QView& w) {
  std::ofstream os(path, std::ios::binary);
  if (!os) fail(QLRA_ERR_IO, "cannot open for writing: " + path);
  os.write(kSketchMagic, 6);
  put_spec(os, om);
  put_spec(os, ps);
  put_u64(os, (uint64_t)r);
  put_u64(os, (uint64_t)s);
  put_u64(os, (uint64_t)l);
  os.write(kQmatMagic, 6);
  write_planes(ctx, os, y);
  os.write(kQmatMagic, 6);
  write_planes(ctx, os, w);
  if (!os) fail(QLRA_ERR_IO, "write_sketch: stream failure");
}

void sketch_header(const std::string& path, qlra_spec_t* om, qlra_spec_t* ps, int64_t* rsl) {
  std::ifstream is(path, std::ios::binary);
  if (!is) fail(QLRA_ERR_IO, "cannot open: " + path);
  expect_magic(is, kSketchMagic, "QSKT1");
  *om = get_spec(is);
  *ps = get_spec(is);
  for (int i = 0; i < 3; ++i) rsl[i] = (int64_t)get_u64(is);
}

void read_sketch(Ctx& ctx, const std::string& path, const QView& y, const QView& w) {
  std::ifstream is(path, std::ios::binary);
  if (!is) fail(QLRA_ERR_IO, "cannot open: " + path);
  expect_magic(is, kSketchMagic, "QSKT1");
  get_spec(is);
  get_spec(is);
  const int64_t r = (int64_t)get_u64(is), s = (int64_t)get_u64(is), l = (int64_t)get_u64(is);
  (void)r;
  expect_magic(is, kQmatMagic, "QMAT1");
  read_planes(ctx, is, y);
  expect_magic(is, kQmatMagic, "QMAT1");
  read_planes(ctx, is, w);
  if (y.cols != s || w.rows != l) fail(QLRA_ERR_IO, "read_sketch: inconsistent dimensions");
}

// sketch_from_source over a QMAT1 file: blocks of `block_rows` rows are read
// (four plane seeks per block, io.cpp:221-239) into a pinned double buffer by
// the host while the device sketches the previous block.
void sketch_from_qmat_file(Ctx& ctx, const std::string& path, const qlra_spec_t& omega,
                           const qlra_spec_t& psi, const QView& y, const QView& w, int64_t block_rows) {
  int64_t m = 0, n = 0;
  qmat_header(path, &m, &n);
  if (n != w.cols || m != y.rows) fail(QLRA_ERR_SHAPE, "sketch_from_source: file shape mismatch");
  if (block_rows < 1) fail(QLRA_ERR_PARAMETER, "sketch_from_source: block_rows must be >= 1");
  const int64_t br = std::min(block_rows, std::max<int64_t>(1, m));
  double* pinned[2] = {nullptr, nullptr};
  const size_t bytes = sizeof(double) * 4 * (size_t)(br * n);
  QLRA_CUDA(cudaMallocHost(&pinned[0], std::max<size_t>(bytes, 8)));
  QLRA_CUDA(cudaMallocHost(&pinned[1], std::max<size_t>(bytes, 8)));
  cudaEvent_t done[2];
  QLRA_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
  QLRA_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
  QLRA_CUDA(cudaEventRecord(done[0], ctx.stream));
  QLRA_CUDA(cudaEventRecord(done[1], ctx.stream));
  std::ifstream is(path, std::ios::binary);
  if (!is) fail(QLRA_ERR_IO, "cannot open: " + path);
  int idx = 0;
  try {
    for (int64_t r0 = 0; r0 < m; r0 += br, idx ^= 1) {
      const int64_t rows = std::min(br, m - r0);
      QLRA_CUDA(cudaEventSynchronize(done[idx]));  // buffer free again
      double* hb = pinned[idx];
      for (int p = 0; p < 4; ++p) {
        is.seekg(kQmatHeaderBytes + (std::streamoff)((p * m + r0) * n * 8));
        if (!is.read(reinterpret_cast<char*>(hb + (size_t)p * rows * n), (std::streamsize)(rows * n * 8)))
          fail(QLRA_ERR_IO, "read_rows: truncated file");
      }
      QView hv;
      for (int p = 0; p < 4; ++p) hv.p[p] = hb + (size_t)p * rows * n;
      hv.rows = rows;
      hv.cols = n;
      hv.ld = n;
      sketch_update_rows_host(ctx, omega, psi, r0, hv, sub(y, r0, 0, rows, y.cols), w, rows);
      QLRA_CUDA(cudaEventRecord(done[idx], ctx.stream));
    }
    QLRA_CUDA(cudaStreamSynchronize(ctx.stream));
  } catch (...) {
    cudaStreamSynchronize(ctx.stream);
    cudaFreeHost(pinned[0]);
    cudaFreeHost(pinned[1]);
    cudaEventDestroy(done[0]);
    cudaEventDestroy(done[1]);
    throw;
  }
  cudaFreeHost(pinned[0]);
  cudaFreeHost(pinned[1]);
  cudaEventDestroy(done[0]);
  cudaEventDestroy(done[1]);
}

}  // namespace qlra_dev
