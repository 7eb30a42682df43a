// group.cu -- the in-process communicator: N contexts (one per host thread)
// whose all-reduces are done by the library itself, without NCCL.
//
// The multi-rank hot path (row-sharded A, all-reduced W,
// Grams, Psi H and norms) normally runs one process per GPU over NCCL.  NCCL
// refuses two ranks on one device, so on a single GPU -- and inside one
// process in general -- the same sharded code runs over this backend: every
// rank posts its buffer, each rank sums all posted buffers in RANK ORDER into
// a private temporary (so every rank computes bit-identical results, like a
// deterministic NCCL all-reduce), and copies the sum back once every peer has
// read its input.  Buffers on different devices are read over peer access.
#include <cuda_runtime.h>

#include <chrono>
#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

struct qlra_group {
  int n = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  std::vector<double*> bufs;
  std::vector<size_t> counts;
  std::vector<int> devs;
  std::vector<cudaEvent_t> ready, done;
  std::vector<int> attached;
};

namespace qlra_dev {

namespace {

constexpr int kMaxRanks = 16;
struct RankPtrs {
  const double* p[kMaxRanks];
};

__global__ void k_sum_ranks(RankPtrs in, int n, size_t count, double* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    double s = in.p[0][i];
    for (int r = 1; r < n; ++r) s += in.p[r][i];  // fixed rank order
    out[i] = s;
  }
}

// Host barrier of the group's ranks (one host thread each).  A rank that
// never arrives (it failed before the collective) breaks the group after a
// timeout instead of hanging the others.
void group_barrier(qlra_group& g) {
  std::unique_lock<std::mutex> lk(g.mu);
  if (g.broken) fail(QLRA_ERR_NCCL, "local group: broken by an earlier failure");
  const uint64_t gen = g.gen;
  if (++g.arrived == g.n) {
    g.arrived = 0;
    ++g.gen;
    g.cv.notify_all();
    return;
  }
  const bool ok = g.cv.wait_for(lk, std::chrono::seconds(300), [&] { return g.gen != gen || g.broken; });
  if (!ok || g.broken) {
    g.broken = true;
    g.cv.notify_all();
    fail(QLRA_ERR_NCCL, "local group: a rank did not reach the collective (timeout)");
  }
}

}  // namespace

void group_allreduce_sum(Ctx& ctx, double* buf, size_t count) {
  qlra_group& g = *ctx.group;
  const int r = ctx.rank;
  g.bufs[r] = buf;
  g.counts[r] = count;
  QLRA_CUDA(cudaEventRecord(g.ready[r], ctx.stream));
  group_barrier(g);  // every rank has posted its buffer
  RankPtrs ptrs{};
  for (int q = 0; q < g.n; ++q) {
    if (g.counts[q] != count) fail(QLRA_ERR_NCCL, "local group: all-reduce sizes differ across ranks");
    ptrs.p[q] = g.bufs[q];
    QLRA_CUDA(cudaStreamWaitEvent(ctx.stream, g.ready[q], 0));
  }
  DeviceBuffer tmp(ctx, count * sizeof(double));
  if (count) {
    const int blocks = (int)std::min<size_t>((count + 255) / 256, 148 * 8);
    k_sum_ranks<<<blocks, 256, 0, ctx.stream>>>(ptrs, g.n, count, tmp.as<double>());
    QLRA_LAUNCH_CHECK();
    count_launch();
  }
  QLRA_CUDA(cudaEventRecord(g.done[r], ctx.stream));
  group_barrier(g);  // every rank has enqueued its reads of the posted buffers
  for (int q = 0; q < g.n; ++q) QLRA_CUDA(cudaStreamWaitEvent(ctx.stream, g.done[q], 0));
  if (count)
    QLRA_CUDA(cudaMemcpyAsync(buf, tmp.ptr, count * sizeof(double), cudaMemcpyDeviceToDevice, ctx.stream));
}

void group_attach(Ctx& ctx, qlra_group* g, int rank) {
  if (!g) fail(QLRA_ERR_PARAMETER, "qlra_ctx_create_local: null group");
  if (rank < 0 || rank >= g->n) fail(QLRA_ERR_PARAMETER, "qlra_ctx_create_local: rank out of range");
  std::lock_guard<std::mutex> lk(g->mu);
  if (g->attached[rank]) fail(QLRA_ERR_PARAMETER, "qlra_ctx_create_local: rank already attached");
  for (int q = 0; q < g->n; ++q) {
    if (!g->attached[q] || g->devs[q] == ctx.device) continue;
    int can = 0;
    QLRA_CUDA(cudaDeviceCanAccessPeer(&can, ctx.device, g->devs[q]));
    if (!can) fail(QLRA_ERR_NCCL, "local group: devices without peer access");
    const cudaError_t e1 = cudaDeviceEnablePeerAccess(g->devs[q], 0);
    if (e1 != cudaSuccess && e1 != cudaErrorPeerAccessAlreadyEnabled) QLRA_CUDA(e1);
    cudaGetLastError();
  }
  if (!g->ready[rank]) QLRA_CUDA(cudaEventCreateWithFlags(&g->ready[rank], cudaEventDisableTiming));
  if (!g->done[rank]) QLRA_CUDA(cudaEventCreateWithFlags(&g->done[rank], cudaEventDisableTiming));
  g->devs[rank] = ctx.device;
  g->attached[rank] = 1;
  ctx.group = g;
  ctx.rank = rank;
  ctx.nranks = g->n;
}

// A rank's events outlive its context: a slower peer may still enqueue its
// wait on them after this rank has left the last collective.  They are
// destroyed with the group.
void group_detach(Ctx& ctx) {
  qlra_group* g = ctx.group;
  if (!g) return;
  std::lock_guard<std::mutex> lk(g->mu);
  g->attached[ctx.rank] = 0;
  ctx.group = nullptr;
}

}  // namespace qlra_dev

extern "C" {

int qlra_group_create(qlra_group_t** out, int nranks) {
  if (!out) return QLRA_ERR_PARAMETER;
  *out = nullptr;
  if (nranks < 1 || nranks > qlra_dev::kMaxRanks) return QLRA_ERR_PARAMETER;
  qlra_group* g = new qlra_group();
  g->n = nranks;
  g->bufs.assign(nranks, nullptr);
  g->counts.assign(nranks, 0);
  g->devs.assign(nranks, -1);
  g->ready.assign(nranks, nullptr);
  g->done.assign(nranks, nullptr);
  g->attached.assign(nranks, 0);
  *out = g;
  return QLRA_OK;
}

int qlra_group_destroy(qlra_group_t* g) {
  if (!g) return QLRA_OK;
  for (int a : g->attached)
    if (a) return QLRA_ERR_PRECONDITION;  // contexts still attached
  for (int r = 0; r < g->n; ++r) {
    if (g->ready[r]) cudaEventDestroy(g->ready[r]);
    if (g->done[r]) cudaEventDestroy(g->done[r]);
  }
  delete g;
  return QLRA_OK;
}

}  // extern "C"
