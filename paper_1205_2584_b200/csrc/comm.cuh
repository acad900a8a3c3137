// Collectives of the slab-sharded engine: the engine calls exactly three
// collectives -- an in-place sum allreduce (pass-A partials, residual scalars, ||Y||^2, mode-n
// Grams), an allgather (pass-B rows of the mode-N factor) and a broadcast (slabs for the sharded
// mode-N Gram of the SVD initialisation) -- through this interface.
//
//  * NcclComm: one process per GPU, NCCL over NVLink / NVSwitch (the product path).
//  * LoopbackComm: a TEST transport.  P engines of one process, each driven by its own host
//    thread, exchange through device buffers with stream/event ordering and a host barrier per
//    collective.  No kernel ever waits on another rank's kernel (the pool forbids spin-waiting
//    ranks sharing one GPU, B200_PROFILING.md), so several "ranks" can share one B200 and the
//    multi-rank data path (slab bounds, ragged slabs, packed allreduce, allgather reorder) runs
//    for real.  The reduction order is rank order; every rank computes the identical sum, which
//    is the property the replicated LM state relies on (NCCL guarantees the same).
#pragma once
#include <condition_variable>
#include <chrono>
#include <mutex>
#include <vector>

#include <nccl.h>

namespace cpf {

constexpr int kMaxLoopRanks = 8;

struct Comm {
  virtual ~Comm() = default;
  virtual void allreduce_sum(double* buf, size_t n, cudaStream_t st) = 0;
  virtual void allgather(const double* send, double* recv, size_t n, cudaStream_t st) = 0;
  virtual void broadcast(const double* send, double* recv, size_t n, int root, cudaStream_t st) = 0;
};

struct NcclComm final : Comm {
  ncclComm_t c = nullptr;
  NcclComm(int world, const ncclUniqueId& id, int rank) { NCCL_CHECK(ncclCommInitRank(&c, world, id, rank)); }
  ~NcclComm() override {
    if (c) ncclCommDestroy(c);
  }
  void allreduce_sum(double* buf, size_t n, cudaStream_t st) override {
    NCCL_CHECK(ncclAllReduce(buf, buf, n, ncclDouble, ncclSum, c, st));
  }
  void allgather(const double* send, double* recv, size_t n, cudaStream_t st) override {
    NCCL_CHECK(ncclAllGather(send, recv, n, ncclDouble, c, st));
  }
  void broadcast(const double* send, double* recv, size_t n, int root, cudaStream_t st) override {
    NCCL_CHECK(ncclBroadcast(send, recv, n, ncclDouble, root, c, st));
  }
};

// ---- loopback (test transport) ----------------------------------------------------------------
struct RankPtrs {
  const double* p[kMaxLoopRanks];
};

__global__ void k_loop_sum(RankPtrs src, int world, size_t n, double* __restrict__ out) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double s = src.p[0][i];
    for (int q = 1; q < world; ++q) s += src.p[q][i];
    out[i] = s;
  }
}

struct LoopbackGroup {
  int world = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  const double* ptr[kMaxLoopRanks] = {};
  cudaEvent_t ready[kMaxLoopRanks] = {};
  cudaEvent_t done[kMaxLoopRanks] = {};
  explicit LoopbackGroup(int w) : world(w) {
    if (w < 1 || w > kMaxLoopRanks) throw ApiError(CPF_E_ARG, "loopback world must be in [1, 8]");
    for (int q = 0; q < w; ++q) {
      CPF_CUDA_CHECK(cudaEventCreateWithFlags(&ready[q], cudaEventDisableTiming));
      CPF_CUDA_CHECK(cudaEventCreateWithFlags(&done[q], cudaEventDisableTiming));
    }
  }
  ~LoopbackGroup() {
    for (int q = 0; q < world; ++q) {
      if (ready[q]) cudaEventDestroy(ready[q]);
      if (done[q]) cudaEventDestroy(done[q]);
    }
  }
  // host barrier of the group's threads; a rank that never arrives (diverged control flow) is an
  // error after 600 s instead of a hang
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(600), [&] { return generation != gen; }))
      throw ApiError(CPF_E_NCCL, "loopback collective timed out: ranks diverged");
  }
};

struct LoopbackComm final : Comm {
  LoopbackGroup* g;
  int rank;
  double* scratch = nullptr;
  size_t scratch_n = 0;
  LoopbackComm(LoopbackGroup* grp, int r) : g(grp), rank(r) {}
  ~LoopbackComm() override {
    if (scratch) cudaFree(scratch);
  }
  // publish `p`, order this stream after every rank's producer work
  void arrive(const double* p, cudaStream_t st) {
    g->ptr[rank] = p;
    CPF_CUDA_CHECK(cudaEventRecord(g->ready[rank], st));
    g->barrier();
    for (int q = 0; q < g->world; ++q) CPF_CUDA_CHECK(cudaStreamWaitEvent(st, g->ready[q], 0));
  }
  // every rank's reads of the published buffers are done before any rank reuses its buffer
  void depart(cudaStream_t st) {
    CPF_CUDA_CHECK(cudaEventRecord(g->done[rank], st));
    g->barrier();
    for (int q = 0; q < g->world; ++q) CPF_CUDA_CHECK(cudaStreamWaitEvent(st, g->done[q], 0));
  }
  void allreduce_sum(double* buf, size_t n, cudaStream_t st) override {
    if (scratch_n < n) {
      if (scratch) CPF_CUDA_CHECK(cudaFree(scratch));
      CPF_CUDA_CHECK(cudaMalloc(&scratch, n * sizeof(double)));
      scratch_n = n;
    }
    arrive(buf, st);
    RankPtrs rp{};
    for (int q = 0; q < g->world; ++q) rp.p[q] = g->ptr[q];
    const unsigned blocks = (unsigned)std::min<size_t>(1024, (n + 255) / 256);
    k_loop_sum<<<std::max(1u, blocks), 256, 0, st>>>(rp, g->world, n, scratch);
    CPF_CUDA_CHECK(cudaGetLastError());
    depart(st);
    CPF_CUDA_CHECK(cudaMemcpyAsync(buf, scratch, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  void allgather(const double* send, double* recv, size_t n, cudaStream_t st) override {
    arrive(send, st);
    for (int q = 0; q < g->world; ++q)
      CPF_CUDA_CHECK(cudaMemcpyAsync(recv + (size_t)q * n, g->ptr[q], n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    depart(st);
  }
  void broadcast(const double* send, double* recv, size_t n, int root, cudaStream_t st) override {
    arrive(rank == root ? send : nullptr, st);
    const double* src = g->ptr[root];
    if (recv != src) CPF_CUDA_CHECK(cudaMemcpyAsync(recv, src, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    depart(st);
  }
};

}  // namespace cpf
