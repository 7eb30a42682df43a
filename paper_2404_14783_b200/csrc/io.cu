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
#include <memory>
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

// Shapes of the Y and W matrices embedded in a QSKT1 file, from their own
// QMAT1 headers (io.cpp:130-145 reads them that way), with the reference's
// consistency test (y.cols == s, w.rows == l, else IoError) and a size check
// against the file length -- before anything is allocated.
void sketch_dims(const std::string& path, int64_t* dims) {
  std::ifstream is(path, std::ios::binary | std::ios::ate);
  if (!is) fail(QLRA_ERR_IO, "cannot open: " + path);
  const std::streamoff size = is.tellg();
  is.seekg(0);
  expect_magic(is, kSketchMagic, "QSKT1");
  get_spec(is);
  get_spec(is);
  get_u64(is);
  const int64_t s = (int64_t)get_u64(is), l = (int64_t)get_u64(is);
  for (int k = 0; k < 2; ++k) {
    expect_magic(is, kQmatMagic, "QMAT1");
    const uint64_t rows = get_u64(is), cols = get_u64(is);
    if (rows > (uint64_t)INT64_MAX / 64 || cols > (uint64_t)INT64_MAX / 64 ||
        (cols && rows > (uint64_t)(size / 32) / cols))
      fail(QLRA_ERR_IO, "read_sketch: truncated file");
    const std::streamoff data = (std::streamoff)(32 * rows * cols);
    if (is.tellg() + data > size) fail(QLRA_ERR_IO, "read_sketch: truncated file");
    dims[2 * k] = (int64_t)rows;
    dims[2 * k + 1] = (int64_t)cols;
    is.seekg(data, std::ios::cur);
  }
  if (dims[1] != s || dims[2] != l) fail(QLRA_ERR_IO, "read_sketch: inconsistent dimensions");
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

// sketch_from_source over a QMAT1 file (QmatFileSource, io.cpp:213-239): the
// file is the only reader of A.  One row pipeline for the whole file (Omega,
// the Psi block and their plane combinations built once): each chunk's rows
// are read from the file -- four plane seeks per chunk, as read_rows does --
// straight into the pipeline's pinned staging while the previous chunk is
// copied and sketched.  block_rows is the chunk height (the reference's
// read granularity); the pipeline enlarges tiny chunks to its own minimum.
void sketch_from_qmat_file(Ctx& ctx, const std::string& path, const qlra_spec_t& omega,
                           const qlra_spec_t& psi, const QView& y, const QView& w, int64_t block_rows) {
  int64_t m = 0, n = 0;
  qmat_header(path, &m, &n);
  if (n != w.cols || m != y.rows) fail(QLRA_ERR_SHAPE, "sketch_from_source: file shape mismatch");
  if (block_rows < 1) fail(QLRA_ERR_PARAMETER, "sketch_from_source: block_rows must be >= 1");
  auto is = std::make_shared<std::ifstream>(path, std::ios::binary);
  if (!*is) fail(QLRA_ERR_IO, "cannot open: " + path);
  RowSource src;
  src.kind = RowSource::kStaged;
  src.fill = [is, m, n](int64_t r0, int64_t rows, double* dst) {
    for (int p = 0; p < 4; ++p) {
      is->seekg(kQmatHeaderBytes + (std::streamoff)((p * m + r0) * n * 8));
      if (!is->read(reinterpret_cast<char*>(dst + (size_t)p * rows * n), (std::streamsize)(rows * n * 8)))
        fail(QLRA_ERR_IO, "read_rows: truncated file");
    }
  };
  // chunks of at least the streaming pipeline's size (tiny chunks make short,
  // inefficient launches), multiples of the requested block height
  const int64_t want = std::max<int64_t>(1, (int64_t)(64e6 / (32.0 * (double)std::max<int64_t>(1, n))));
  const int64_t chunk = std::min<int64_t>(m, ((want + block_rows - 1) / block_rows) * block_rows);
  sketch_rows_pipeline(ctx, omega, psi, 0, m, n, src, y, w, chunk, false);
  QLRA_CUDA(cudaStreamSynchronize(ctx.stream));
}

}  // namespace qlra_dev
