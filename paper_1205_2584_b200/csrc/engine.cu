// B200 fLM CP engine: host orchestration of one fit behind the C ABI in include/cpfast_b200.h.
//
// One engine = one GPU = one process.  It owns every device buffer of the fit; the LM control
// state (mu, growth, err, accept/stop flags, the 10-delta tolerance window, the trace) lives on
// the device (LmDeviceState), so an iteration is a fixed launch sequence and the host only polls
// the state once per iteration (or per batch).  Reference semantics: cpfast/solver.py:319-384.
#include <cuda_runtime.h>
#include <nccl.h>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cpfast_b200.h"

struct CudaError : std::runtime_error {
  CudaError(cudaError_t e, const char* expr, const char* file, int line)
      : std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(e) + " at " + file + ":" +
                           std::to_string(line) + " (" + expr + ")") {}
};
struct ApiError : std::runtime_error {
  int code;
  ApiError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#include "cpf_common.cuh"
#include "lu.cuh"
#include "lu3.cuh"
#include "lu4.cuh"
#include "lu_persist.cuh"
#include "tri_inv.cuh"
#include "phi.cuh"
#include "small_ops.cuh"
#include "tensor_pass.cuh"
#include "tensor_pass2.cuh"
#include "tensor_pass_dmma.cuh"
#include "tensor_pass_oz.cuh"
#include "als.cuh"
#include "fdi.cuh"

#define NCCL_CHECK(expr)                                                                   \
  do {                                                                                     \
    ncclResult_t _r = (expr);                                                              \
    if (_r != ncclSuccess) throw ApiError(CPF_E_NCCL, std::string("NCCL error ") + ncclGetErrorString(_r) + " (" #expr ")"); \
  } while (0)

#include "comm.cuh"

#include <nvtx3/nvToolsExt.h>

// NVTX ranges on the host orchestration (SURVEY §5 tracing): what an nsys / ncu --nvtx timeline
// groups by.  Inside a captured iteration they mark the capture; graph replays are marked by
// fit_step's range.  Header-only NVTX3: no library dependency, no cost without a profiler.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

namespace cpf {

// Process-wide cache of tensor-sized device buffers (see Engine::big_alloc): exact-size reuse
// (the next engine of the same problem asks for the same sizes), released on allocation failure.
struct BigCache {
  struct Buf { int dev; size_t bytes; void* p; };
  static std::mutex& mu() { static std::mutex m; return m; }
  static std::vector<Buf>& bufs() { static std::vector<Buf> v; return v; }
  static void* take(int dev, size_t bytes) {
    std::lock_guard<std::mutex> lk(mu());
    auto& v = bufs();
    for (size_t i = 0; i < v.size(); ++i)
      if (v[i].dev == dev && v[i].bytes == bytes) {
        void* p = v[i].p;
        v.erase(v.begin() + (long)i);
        return p;
      }
    return nullptr;
  }
  static void park(int dev, void* p, size_t bytes) {
    std::lock_guard<std::mutex> lk(mu());
    bufs().push_back({dev, bytes, p});
  }
  static size_t parked_bytes(int dev) {
    std::lock_guard<std::mutex> lk(mu());
    size_t n = 0;
    for (const auto& b : bufs())
      if (b.dev == dev) n += b.bytes;
    return n;
  }
  static void release(int dev) {
    std::lock_guard<std::mutex> lk(mu());
    auto& v = bufs();
    for (size_t i = 0; i < v.size();) {
      if (v[i].dev == dev) {
        cudaFree(v[i].p);
        v.erase(v.begin() + (long)i);
      } else {
        ++i;
      }
    }
  }
};

static int padded_rank(int R) {
  static const int table[] = {2, 4, 6, 8, 10, 12, 16, 20, 24, 32, 40, 48, 64};  // even: paired smem loads
  for (int v : table)
    if (v >= R) return v;
  return -1;
}

enum Phase { kPhPassA = 0, kPhPassB = 1, kPhLU = 2, kPhSolve = 3, kPhOther = 4, kNumPhases = 5 };

// ------------------------------------------------------------------------------------------
struct EngineBase {
  virtual ~EngineBase() = default;
  std::string last_error;
  virtual void slab(int64_t* lo, int64_t* hi) const = 0;
  virtual void* stream() = 0;
  virtual void set_tensor(const void* p, int64_t n, int where) = 0;
  virtual void load_cptn(const char* path, int64_t payload_offset) = 0;
  virtual void set_factors(const void* p) = 0;
  virtual void get_factors(void* p) = 0;
  virtual void fit_begin(int variant, double tau, double tol, int max_iters, cpf_status* st) = 0;
  virtual void fit_step(int n, cpf_status* st) = 0;
  virtual int trace(cpf_iter_record* out, int cap) = 0;
  virtual void mttkrp(int mode, void* out) = 0;
  virtual double relative_error() = 0;
  virtual int flm_step(double mu, int variant, int refine, void* out) = 0;
  virtual void profile(int on) = 0;
  virtual void phase_times(double* ms, int64_t* cnt, int n) = 0;
  virtual void phase_max(double* ms, int n) = 0;
  virtual int64_t launches() const = 0;
  virtual int pass_impl() const = 0;
  virtual void pass_guard(int64_t* fallbacks, int* rejected) = 0;
  virtual void unfolding_gram(int mode, void* out) = 0;
  virtual double als_step(int line_search, int t) = 0;
  virtual void set_history(const void* p) = 0;
  virtual int fast_damped_inverse(double mu, int use_kinv, void* gt_out, void* d_out) = 0;
};

template <class T>
struct Engine final : EngineBase {
  // ---- geometry
  int dev = 0, N = 0, R = 0, RP = 0, world = 1, wrank = 0;
  int64_t dims[kMaxModes] = {0};
  int64_t offs[kMaxModes] = {0};
  int64_t Tsum = 0, RT = 0;
  int64_t I1 = 0, Lmid = 1, Lrows = 0, IN = 0, slab_lo = 0, slab_hi = 0, Cloc = 0, Cpad = 0, Jloc = 0;
  int nB = 0;
  Modes md{};
  MidGeom mg{};
  cudaStream_t s = nullptr;
  cudaStream_t ls = nullptr;   // stream the launch helpers target (s, or s3 for the overlapped pass B)
  cudaStream_t s3 = nullptr;   // pass B + gradient of an accepted step, overlapped with the next LU
  cudaEvent_t evF = nullptr, evG = nullptr;
  const bool serial = [] { const char* e = knob("CPF_SERIAL"); return e && e[0] == '1'; }();
  std::unique_ptr<Comm> comm;  // NCCL (world > 1) or the loopback test transport; null: 1 rank
  int64_t nlaunch = 0;

  // ---- tensor
  const T* Y = nullptr;
  T* Yown = nullptr;
  bool have_tensor = false, have_factors = false;
  bool test_singular = false;  // fault-injection kernel in prepare_core (CPF_TEST_SINGULAR)

  // ---- device buffers
  T *A = nullptr, *Ac = nullptr, *M = nullptr, *Mc = nullptr, *D = nullptr, *G = nullptr, *Cand = nullptr;
  T *V1 = nullptr, *V2 = nullptr, *V3 = nullptr, *V4 = nullptr;
  T *Cg = nullptr, *Ccg = nullptr, *Gx = nullptr, *Gp = nullptr, *Gf = nullptr, *Gti = nullptr, *Gi = nullptr;
  T *W1 = nullptr, *Sm = nullptr;
  T *wvec = nullptr, *fvec = nullptr, *xvec = nullptr, *Phi = nullptr;
  // explicit (factored) inverse of Phi: B w = inv(U) inv(L) P w as two triangular mat-vecs
  T *PhiInv = nullptr, *TriTmp = nullptr, *yvec = nullptr, *tmv_part = nullptr;
  bool use_inv = false;
  bool use_blkinv = false;            // !use_inv: substitution over inverted diagonal blocks
  int blk_db = 1024;                  // its diagonal block size (power of two >= 64)
  int tri_cap() const { return use_inv ? nB : std::min(nB, blk_db); }  // merge levels stay below this
  T *A1c = nullptr, *KMc = nullptr, *WNc = nullptr, *zpart = nullptr, *m1part = nullptr, *bpart = nullptr;
  T *A1r = nullptr, *KMr = nullptr, *WNr = nullptr;  // non-conj operands of the direct residual
  T *pa_out = nullptr, *pb_out = nullptr, *pb_all = nullptr;
  double *norms = nullptr, *dscal = nullptr, *red = nullptr;
  int* ibuf = nullptr;
  LuWork lu{};
  LmDeviceState* st = nullptr;
  DevFlags* fl = nullptr;
  IterRecordDev* dtrace = nullptr;
  int* kinv_ok = nullptr;
  LmDeviceState* hst = nullptr;  // pinned mirror
  int trace_cap = 0;
  int epoch = 0;

  // pass-A / pass-B launch geometry
  int pa_threads = 256, pa_TI = 1, pa_TM = 1, pa_tiles = 1, pa_groups = 1;
  int64_t pa_mper = 1;
  size_t pa_smem = 0;
  int pb_threads = 256, pb_TI = 1, pb_TM = 1, pb_tiles = 1, pb_chunks = 1;
  int64_t pb_mper = 1;
  // DMMA (fp64 tensor core) passes for float64 with large I1
  bool use_dmma = false;
  // Ozaki-split int8 tensor passes (tensor_pass_oz.cuh): real tensors, I1 >= 256, R <= 32, large J
  bool use_oz = false;
  OzGeom oa{}, ob{};
  uint8_t *ozYA = nullptr, *ozYB = nullptr, *ozBA = nullptr, *ozBB = nullptr;
  int *ozFrowA = nullptr, *ozFrowB = nullptr, *ozFr = nullptr;  // ozFr: [0, 32) pass A, [32, 64) pass B
  double *ozM1 = nullptr, *ozZ = nullptr, *ozBp = nullptr;          // epilogue partial sums
  // Speculative rejection branch (CPF_SPEC, plan_spec): at the start of an iteration the core
  // system a rejection would need next -- Phi(Grams_t, mu_t * growth_t) -- is factored and inverted
  // on its own streams (sS, sS2) into its own buffers, concurrently with the candidate and pass A.
  // After a rejection the next iteration copies it in (k_copy gated kOnRejectPrev) and the fork's
  // own core system is skipped (gate 2: accepted only); after an acceptance it is discarded.
  bool use_spec = false, spec_capture = false;
  T *PhiS = nullptr, *PhiInvS = nullptr, *TriTmpS = nullptr, *GtiS = nullptr, *GiS = nullptr, *invLS = nullptr;
  int *ibufS = nullptr, *gringS = nullptr, *spec_sing = nullptr;
  LuWork luS{};
  cudaStream_t sS = nullptr, sS2 = nullptr;
  cudaEvent_t evS0 = nullptr, evS1 = nullptr;
  int dm_nt = 0;
  DmmaGeom da{}, db{};
  size_t da_smem = 0, db_smem = 0;
  int da_groups = 1, db_chunks = 1;
  double *WNd = nullptr, *KMd = nullptr;
  // v2 (TMA bulk pipeline) geometry
  bool use_v2 = false;
  int rpt = 1;
  PassGeom ga{}, gb{};
  size_t ga_smem = 0, gb_smem = 0;
  int ga_groups = 1, gb_chunks = 1;
  int lu_kb = 32, lu_cl = 1, lu_rpc = 0;
  int lu3_rpt = 1;      // rows per thread of the register-resident panel (0: use the smem panel)
  T* invL = nullptr;    // 2 slots (double-buffered across look-ahead steps)
  int* gring = nullptr; // 2 gather lists + counts
  cudaStream_t s2 = nullptr;
  // progressive triangular inverse (tri_progress): side stream of the look-ahead LU + its events
  cudaStream_t s4 = nullptr, sS4 = nullptr;
  cudaEvent_t evT = nullptr, evT2 = nullptr;
  bool tri_prog = true;
  bool tri_in_lu = false;  // the last lu_factor already produced PhiInv
  cudaEvent_t evP = nullptr, evB = nullptr, evJ = nullptr;
  cudaEvent_t evB2[2] = {nullptr, nullptr};
  size_t lu_smem = 0;

  // CUDA graph of one iteration (replayed; all control is device-side)
  cudaGraphExec_t gexec = nullptr;
  int64_t graph_nodes = 0;
  bool graph_ok = true;
  static constexpr int kPoll = 4;  // iterations launched between host polls of the state

  // profiling
  bool prof = false;
  // diagnostic section marks on stream s in profiled (eager) iterations (CPF_MARKS=1 prints the
  // per-section totals from phase_times): 0 candidate, 1 normalise + pass A + trial fit + decide,
  // 2 commit, 3 fork (pass B || next core system) to join
  std::vector<std::pair<int, cudaEvent_t>> marks;
  double mark_ms[4] = {0, 0, 0, 0};
  // CPF_MARKS=3: the marks are external event-record nodes of the captured iteration graph, read
  // after every replay (graph-mode section times; diagnostic, one replay per poll)
  const bool gmarks = [] { const char* e = knob("CPF_MARKS"); return e && e[0] == '3'; }();
  cudaEvent_t gmark[9] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  bool capturing = false;
  void mark(int id) {
    if (spec_capture) return;
    if (gmarks && capturing) {
      if (!gmark[id]) CPF_CUDA_CHECK(cudaEventCreate(&gmark[id]));
      CPF_CUDA_CHECK(cudaEventRecordWithFlags(gmark[id], s, cudaEventRecordExternal));
      return;
    }
    if (!prof) return;
    cudaEvent_t e;
    CPF_CUDA_CHECK(cudaEventCreate(&e));
    CPF_CUDA_CHECK(cudaEventRecord(e, s));
    marks.push_back({id, e});
  }
  struct Ev { int ph; cudaEvent_t a, b; };
  std::vector<Ev> evs;
  double ph_ms[kNumPhases] = {0};
  int64_t ph_cnt[kNumPhases] = {0};
  double ph_max[kNumPhases] = {0};  // longest single instance since profiling was switched on

  // ------------------------------------------------------------------------------------------
  Engine(int device, int order, const int64_t* d, int rank, int wr, int ws, const void* uid,
         LoopbackGroup* loop = nullptr) {
    if (order < 2 || order > kMaxModes) throw ApiError(CPF_E_UNSUPPORTED, "order must be in [2, 8]");
    if (rank < 1) throw ApiError(CPF_E_ARG, "rank must be >= 1");
    RP = padded_rank(rank);
    if (RP < 0) throw ApiError(CPF_E_UNSUPPORTED, "rank > 64 is outside the engine envelope");
    dev = device;
    N = order;
    R = rank;
    world = ws;
    wrank = wr;
    CPF_CUDA_CHECK(cudaSetDevice(dev));
    int prio_lo = 0, prio_hi = 0;
    CPF_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    CPF_CUDA_CHECK(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, prio_hi));
    CPF_CUDA_CHECK(cudaStreamCreateWithPriority(&s3, cudaStreamNonBlocking, prio_lo));
    CPF_CUDA_CHECK(cudaEventCreateWithFlags(&evF, cudaEventDisableTiming));
    CPF_CUDA_CHECK(cudaEventCreateWithFlags(&evG, cudaEventDisableTiming));
    ls = s;
    for (int n = 0; n < N; ++n) {
      if (d[n] < 1) throw ApiError(CPF_E_ARG, "dims must be >= 1");
      dims[n] = d[n];
      offs[n] = (int64_t)R * Tsum;
      Tsum += d[n];
    }
    RT = (int64_t)R * Tsum;
    md.N = N;
    md.R = R;
    for (int n = 0; n < N; ++n) { md.dims[n] = dims[n]; md.offs[n] = offs[n]; }
    I1 = dims[0];
    Lmid = 1;
    for (int n = 1; n < N - 1; ++n) Lmid *= dims[n];
    Lrows = I1 * Lmid;
    IN = dims[N - 1];
    mg.nmid = N - 2;
    for (int k = 0; k < N - 2; ++k) { mg.dims[k] = dims[k + 1]; mg.offs[k] = offs[k + 1]; }
    // slab sharding along mode N: ceil(IN / world) per rank
    const int64_t per = (IN + world - 1) / world;
    slab_lo = std::min<int64_t>(IN, per * wrank);
    slab_hi = std::min<int64_t>(IN, slab_lo + per);
    Cloc = slab_hi - slab_lo;
    Cpad = per;
    Jloc = Lrows * Cloc;
    nB = N * R * R;
    if ((int64_t)nB * nB > (int64_t)1 << 31) throw ApiError(CPF_E_UNSUPPORTED, "N*R^2 too large");
    // CPF_FORCE_NCCL=1 runs a single-rank engine through the multi-rank code path (1-rank NCCL
    // communicator, packed allreduce / allgather / reorder kernels) so it can be tested on 1 GPU.
    const char* fe = knob("CPF_FORCE_NCCL");
    const bool force = fe && fe[0] == '1';
    if (loop) {
      // loopback test transport: P engines of one process on one GPU (comm.cuh); its host
      // barriers cannot live inside a captured graph, so these engines launch eagerly
      if (loop->world != world || wrank < 0 || wrank >= world) throw ApiError(CPF_E_ARG, "loopback group / rank mismatch");
      comm.reset(new LoopbackComm(loop, wrank));
      graph_ok = false;
    } else if (world > 1 || force) {
      ncclUniqueId id;
      if (world > 1) {
        if (!uid) throw ApiError(CPF_E_ARG, "world_size > 1 needs an NCCL unique id");
        std::memcpy(&id, uid, sizeof(id));
      } else {
        NCCL_CHECK(ncclGetUniqueId(&id));
      }
      comm.reset(new NcclComm(world, id, wrank));
    }
    configure_pool(dev);
    alloc();
    plan();
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));  // stream-ordered allocations visible to every stream
  }

  ~Engine() override {
    cudaSetDevice(dev);
    if (s) cudaStreamSynchronize(s);
    if (gexec) cudaGraphExecDestroy(gexec);
    if (evP) cudaEventDestroy(evP);
    if (evB) cudaEventDestroy(evB);
    for (auto e : evB2) if (e) cudaEventDestroy(e);
    if (evJ) cudaEventDestroy(evJ);
    if (s2) cudaStreamDestroy(s2);
    if (evT) cudaEventDestroy(evT);
    if (evT2) cudaEventDestroy(evT2);
    if (s4) cudaStreamDestroy(s4);
    if (sS4) cudaStreamDestroy(sS4);
    if (evF) cudaEventDestroy(evF);
    if (evS0) cudaEventDestroy(evS0);
    if (evS1) cudaEventDestroy(evS1);
    if (sS) cudaStreamDestroy(sS);
    if (sS2) cudaStreamDestroy(sS2);
    if (evG) cudaEventDestroy(evG);
    if (s3) cudaStreamDestroy(s3);
    for (auto& e : evs) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
    void* ptrs[] = {Yown, A, Ac, M, Mc, D, G, Cand, V1, V2, V3, V4, Cg, Ccg, Gx, Gp, Gf, Gti, Gi, W1, Sm,
                    wvec, fvec, xvec, Phi, A1c, KMc, WNc, A1r, KMr, WNr, zpart, m1part, bpart, pa_out, pb_out, pb_all,
                    norms, dscal, red, ibuf, st, fl, dtrace, kinv_ok, invL, WNd, KMd, gring, PhiInv, TriTmp, yvec, tmv_part,
                    ozYA, ozYB, ozBA, ozBB, ozFrowA, ozFrowB, ozFr, ozM1, ozZ, ozBp,
                    PhiS, PhiInvS, TriTmpS, GtiS, GiS, invLS, ibufS, gringS, spec_sing, Hist, Pinv,
                    lp.panel_done, lp.u12s, lpS.panel_done, lpS.u12s, TriPart, TriPartS};
    for (void* p : ptrs)
      if (p && std::find_if(big_bufs.begin(), big_bufs.end(), [&](const auto& b) { return b.first == p; }) ==
                   big_bufs.end())
        cudaFreeAsync(p, s);  // back to the device pool (kept for the next engine)
    if (s) cudaStreamSynchronize(s);  // every stream of the engine joins s: nothing uses them now
    for (const auto& b : big_bufs) BigCache::park(dev, b.first, b.second);
    if (hst) cudaFreeHost(hst);
    comm.reset();
    if (s) cudaStreamDestroy(s);
  }

  // Device buffers come from the device's default stream-ordered pool with an unlimited release
  // threshold: an engine's ~50 GB (config 4: tensor + digit-plane images) stays reserved after it
  // closes and the next engine reuses it -- cudaFree/cudaMalloc of that much memory costs up to
  // ~0.5 s per fit (measured inside fit()'s wall time).
  static void configure_pool(int device) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return;
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  // Tensor-sized buffers (the bound slab, the int8 digit-plane images: ~50 GB at config 4) come
  // from cudaMalloc, not the stream-ordered pool: growing the pool by that much costs ~0.9 s on
  // the first fit of a process (measured: cpf_pool_reserve of 50 GB 300 ms, a cold fit() 1.16 s
  // for engine + upload vs 0.30 s warm), cudaMalloc of 16 GB ~3-6 ms.  A destroyed engine parks
  // them in a process-wide cache (BigCache) for the next engine -- as the pool did, without the
  // pool's growth cost -- instead of cudaFree (~0.1 s for 50 GB, on every fit).
  static constexpr size_t kBigAlloc = (size_t)1 << 30;
  std::vector<std::pair<void*, size_t>> big_bufs;
  void* big_alloc(size_t bytes, bool zero) {
    if (bytes < kBigAlloc || knob("CPF_POOL_ONLY")) {
      void* p = nullptr;
      CPF_CUDA_CHECK(cudaMallocAsync(&p, std::max<size_t>(bytes, 1), s));
      if (zero) CPF_CUDA_CHECK(cudaMemsetAsync(p, 0, std::max<size_t>(bytes, 1), s));
      return p;
    }
    void* p = BigCache::take(dev, bytes);
    if (!p) {
      cudaError_t e = cudaMalloc(&p, bytes);
      if (e == cudaErrorMemoryAllocation) {  // release what earlier engines parked and retry
        cudaGetLastError();
        BigCache::release(dev);
        e = cudaMalloc(&p, bytes);
      }
      CPF_CUDA_CHECK(e);
    }
    big_bufs.push_back({p, bytes});
    if (zero) CPF_CUDA_CHECK(cudaMemsetAsync(p, 0, bytes, s));
    return p;
  }
  void big_free(void* p) {
    if (!p) return;
    auto it = std::find_if(big_bufs.begin(), big_bufs.end(), [&](const auto& b) { return b.first == p; });
    if (it == big_bufs.end()) { CPF_CUDA_CHECK(cudaFreeAsync(p, s)); return; }
    const size_t bytes = it->second;
    big_bufs.erase(it);
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    BigCache::park(dev, p, bytes);
  }
  template <class U>
  U* dalloc(size_t n) {
    void* p = nullptr;
    CPF_CUDA_CHECK(cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(U), s));
    CPF_CUDA_CHECK(cudaMemsetAsync(p, 0, std::max<size_t>(n, 1) * sizeof(U), s));
    return static_cast<U*>(p);
  }

  void alloc() {
    const size_t R2 = (size_t)R * R;
    A = dalloc<T>(RT); Ac = dalloc<T>(RT); M = dalloc<T>(RT); Mc = dalloc<T>(RT); D = dalloc<T>(RT);
    G = dalloc<T>(RT); Cand = dalloc<T>(RT);
    V1 = dalloc<T>(RT); V2 = dalloc<T>(RT); V3 = dalloc<T>(RT); V4 = dalloc<T>(RT);
    Cg = dalloc<T>(N * R2); Ccg = dalloc<T>(N * R2); Gx = dalloc<T>(N * R2); Gp = dalloc<T>((size_t)N * N * R2);
    Gf = dalloc<T>(R2); Gti = dalloc<T>(N * R2); Gi = dalloc<T>(N * R2); W1 = dalloc<T>(N * R2); Sm = dalloc<T>(N * R2);
    wvec = dalloc<T>(nB); fvec = dalloc<T>(nB); xvec = dalloc<T>(nB);
    Phi = dalloc<T>((size_t)nB * nB);
    // explicit inverse pays off while its ~(4/3) n^3 flops stay below the latency of six
    // substitutions (measured: n = 1200 yes, n = 4800 no); CPF_NO_INV=1 disables
    use_inv = nB <= 2560;
    if (const char* e = knob("CPF_NO_INV")) if (e[0] == '1') use_inv = false;
    if (use_inv) {
      PhiInv = dalloc<T>((size_t)nB * nB);
      TriTmp = dalloc<T>((size_t)nB * nB);
      if (nB > 256) TriPart = dalloc<T>((size_t)kTriSplit * nB * nB);
      yvec = dalloc<T>(nB);
      tmv_part = dalloc<T>((size_t)((nB + kTmvCols - 1) / kTmvCols) * nB);
    } else {
      // block-inverse substitution (tri_inv.cuh): inverted blk_db x blk_db diagonal blocks
      use_blkinv = true;
      if (const char* e = knob("CPF_BLK_INV")) use_blkinv = e[0] != '0';
      if (const char* e = knob("CPF_BLK_DB")) {
        int v = 64;
        while (v < atoi(e)) v *= 2;
        blk_db = v;
      }
      if (use_blkinv) {
        PhiInv = dalloc<T>((size_t)nB * nB);
        TriTmp = dalloc<T>((size_t)nB * nB);
        TriPart = dalloc<T>((size_t)kTriSplit * nB * nB);
        tmv_part = dalloc<T>((size_t)((nB + kTmvCols - 1) / kTmvCols) * nB);
      }
    }
    A1c = dalloc<T>((size_t)I1 * RP + 2);
    KMc = dalloc<T>((size_t)Lmid * RP + 2);
    WNc = dalloc<T>((size_t)std::max<int64_t>(Cloc, 1) * RP + 2);
    A1r = dalloc<T>((size_t)I1 * RP);
    KMr = dalloc<T>((size_t)Lmid * RP);
    WNr = dalloc<T>((size_t)std::max<int64_t>(Cloc, 1) * RP);
    pa_out = dalloc<T>((size_t)(I1 + Lmid) * R);
    pb_out = dalloc<T>((size_t)Cpad * R);
    pb_all = dalloc<T>((size_t)Cpad * R * world);
    norms = dalloc<double>((size_t)N * R);
    dscal = dalloc<double>(16);
    red = dalloc<double>(4096);
    const int nblk32 = (nB + 31) / 32;
    ibuf = dalloc<int>((size_t)2 * nB + 4 * kLuMaxKB + 8 + 2 * nblk32);
    lu.perm = ibuf;
    lu.ipiv = ibuf + nB;
    lu.gather = ibuf + 2 * nB;
    lu.gcount = lu.gather + 4 * kLuMaxKB;
    lu.info = lu.gcount + 1;
    lu.ticket = lu.info + 1;
    lu.ready = lu.ticket + 4;
    st = dalloc<LmDeviceState>(1);
    fl = dalloc<DevFlags>(1);
    kinv_ok = dalloc<int>(1);
    CPF_CUDA_CHECK(cudaMallocHost(&hst, sizeof(LmDeviceState)));
    std::memset(hst, 0, sizeof(LmDeviceState));
  }

  // Launch geometry for the tensor passes and the LU panel.
  int nsm_ = 148;
  // SMs left to the LU while pass B runs alongside it (CPF_LU_RESERVE overrides)
  // (HBM-bound Ozaki pass B: 40, measured best of 24..48 at config 4; DMMA pass B: 24)
  int kLuReserveSms = 24;
  int kSpecReserveSms = 20;  // SMs pass A leaves to a speculated core system (plan_spec)
  bool spec_a_side = true;   // pass A beside the speculated core system runs on the low-priority stream
  // pass B overlapped with the LU runs as a persistent grid on nsm - kLuReserveSms SMs, so the LU's
  // small panel clusters and GEMM updates always find free SMs (CPF_PERSISTENT_B=0: plain grid)
  const bool persistent_b = [] { const char* e = knob("CPF_PERSISTENT_B"); return !(e && e[0] == '0'); }();
  // next-block update fused into the panel load (PanelPrev, lu3.cuh): removes the gather / U12 /
  // GEMM launches between consecutive panels.  Measured (1 x B200): C1 43.3 -> 51.1 it/s, C2 359 ->
  // 405, C4 131.4 -> 131.4 (there the LU is hidden behind pass B).  CPF_LU_FUSE=0: unfused.
  bool lu_fuse = true;
  // programmatic dependent launch for the launch() helper's kernels (CPF_PDL=0: off)
  // Only the single-stream chain from the candidate to the commit uses it: in the fork (pass B beside
  // the LU) early-scheduled CTAs would park on the SMs left to the LU (measured 162 -> 140 it/s).
  const bool use_pdl = [] { const char* e = knob("CPF_PDL"); return !(e && e[0] == '0'); }();
  bool pdl_now = false;
  // programmatic launch of consecutive LU panels (CPF_PDL_PANEL=1; measured no gain at C4 / C1:
  // the inter-panel gap shrinks from ~4 to ~1 us but the parked next panel slows the running one)
  const bool pdl_panels = [] { const char* e = knob("CPF_PDL_PANEL"); return e && e[0] == '1'; }();
  void plan() {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    nsm_ = nsm;
    if (const char* e = knob("CPF_LU_FUSE")) lu_fuse = e[0] == '1';
    const size_t es = sizeof(T);
    // pass A: threads sized so 2*threads*RP*es (+W stage) fits ~160 KB
    pa_threads = 256;
    while (pa_threads > 32 && (2 * (size_t)pa_threads * RP + kPassCK * RP) * es > 160 * 1024) pa_threads /= 2;
    pa_TI = (int)std::min<int64_t>(I1, pa_threads);
    pa_TM = pa_threads / pa_TI;
    pa_tiles = (int)((I1 + pa_TI - 1) / pa_TI);
    const int64_t target = (int64_t)nsm * 4;
    int64_t groups = std::max<int64_t>(1, target / pa_tiles);
    groups = std::min<int64_t>(groups, (Lmid + pa_TM - 1) / pa_TM);
    pa_mper = (Lmid + groups - 1) / groups;
    pa_mper = ((pa_mper + pa_TM - 1) / pa_TM) * pa_TM;
    pa_groups = (int)((Lmid + pa_mper - 1) / pa_mper);
    pa_smem = (2 * (size_t)pa_threads * RP + kPassCK * RP) * es;
    zpart = dalloc<T>((size_t)pa_tiles * Lmid * RP);
    m1part = dalloc<T>((size_t)pa_groups * I1 * RP);
    // pass B
    pb_threads = 256;
    pb_TI = (int)std::min<int64_t>(I1, pb_threads);
    pb_TM = pb_threads / pb_TI;
    pb_tiles = (int)((I1 + pb_TI - 1) / pb_TI);
    int64_t per_c = std::max<int64_t>(1, target / std::max<int64_t>(1, Cloc * pb_tiles));
    per_c = std::min<int64_t>(per_c, (Lmid + pb_TM - 1) / pb_TM);
    pb_mper = (Lmid + per_c - 1) / per_c;
    pb_chunks = (int)((Lmid + pb_mper - 1) / pb_mper);
    bpart = dalloc<T>((size_t)std::max<int64_t>(Cloc, 1) * pb_chunks * pb_tiles * RP);
    // LU panel: smallest cluster whose smem holds the (full-height) first panel
    lu_kb = std::min(kLuMaxKB, nB);
    const size_t cap = 200 * 1024;
    for (;;) {
      bool ok = false;
      for (int cl = 1; cl <= kLuMaxCluster; cl *= 2) {
        int rpc = (nB + cl - 1) / cl;
        if (panel_smem_bytes<T>(rpc, lu_kb, cl) <= cap) { lu_cl = cl; lu_rpc = rpc; ok = true; break; }
      }
      if (ok) break;
      if (lu_kb <= 4) throw ApiError(CPF_E_UNSUPPORTED, "N*R^2 too large for the LU panel");
      lu_kb /= 2;
    }
    lu_smem = panel_smem_bytes<T>(lu_rpc, lu_kb, lu_cl);
    plan_lu3();
    plan_lp();
    plan_v2(nsm);
    plan_dmma(nsm);
    plan_oz();
    plan_spec();
    // pass A beside a speculated core system: evict-first like pass B, so the image stream does not
    // push the branch's matrix out of L2 (config 4: 184.5 -> 190.3 it/s; alone the hint cost 3 %)
    if (use_oz && use_spec && !knob("CPF_OZ_DBG")) oa.dbg = 0;
    kLuReserveSms = use_oz ? 40 : 24;
    if (const char* e = knob("CPF_LU_RESERVE")) kLuReserveSms = atoi(e);
    CPF_CUDA_CHECK(cudaFuncSetAttribute(k_panel_lu<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lu_smem));
    if (lu_cl > 8) CPF_CUDA_CHECK(cudaFuncSetAttribute(k_panel_lu<T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    set_pass_attrs();
    CPF_CUDA_CHECK(cudaFuncSetAttribute(k_damped_inverses<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)(2 * R * R * sizeof(T))));
  }

  int lu3_thr = 128;  // threads per CTA of the register panel
  // rotating-frame panel (lu4.cuh): rows/thread and threads/CTA; 0 = use k_panel_lu3
  // LU v5 (lu_persist.cuh): the whole factorization in one persistent kernel, panel rows in one
  // CTA's registers (n_B <= 1280 real / 512 complex).  EXPERIMENTAL, off by default (CPF_LU=5):
  // measured slower than the v4 path (n_B = 1200 alone: 2.05-2.14 vs 1.46 ms for LU + inverses,
  // profiles/r02_lu_persist.txt) -- the single-CTA column loop costs ~2700 cycles per column,
  // no better than v4's cluster exchange, and its 16-column steps double the step count.
  // lp_cfg: 0 off, else the (threads, rows per thread) instantiation.
  int lp_cfg = 0, lp_grid = 0;
  LuPersist lp{}, lpS{};
  void alloc_lp(LuPersist& q) {
    const int np = (nB + kLpKB - 1) / kLpKB;
    q.n = nB;
    q.np = np;
    int* ib = dalloc<int>((size_t)3 * np + nB + (size_t)np * kLpKB + 4);
    q.panel_done = ib;
    q.block_ready = ib + np;
    q.blk_done = ib + 2 * np;
    q.ret = ib + 3 * np;
    q.piv = q.ret + nB;
    q.bar = q.piv + (size_t)np * kLpKB;
    q.u12s = dalloc<T>((size_t)np * kLpKB * kLpKB);
  }
  void plan_lp() {
    const char* e = knob("CPF_LU");
    if (!(e && e[0] == '5')) return;
    if (!use_inv) return;  // the final gather uses TriTmp (allocated with the explicit inverse)
    if constexpr (sizeof(T) == 8) {
      lp_cfg = nB <= 512 ? 1 : nB <= 1024 ? 2 : nB <= 1280 ? 3 : 0;
    } else {
      lp_cfg = nB <= 512 ? 11 : 0;
    }
    if (!lp_cfg) return;
    lp_dispatch([&](auto kern, int) {
      CPF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lp_smem_bytes<T>(nB)));
    });
    alloc_lp(lp);
    lp.perm = lu.perm;
    lp.info = lu.info;
    lp.tmp = TriTmp;
  }
  template <class F>
  void lp_dispatch(F&& f) {
    if constexpr (sizeof(T) == 8) {
      if (lp_cfg == 1) f(k_lu_persist<T, 256, 2>, 256);
      else if (lp_cfg == 2) f(k_lu_persist<T, 256, 4>, 256);
      else f(k_lu_persist<T, 256, 5>, 256);
    } else {
      f(k_lu_persist<T, 256, 2>, 256);
    }
  }
  void lu_factor_lp(int gate_running) {
    const LuPersist& q = lp;
    const int np = q.np;
    // helpers: the SMs the fork leaves to the LU, at most one per column block
    LuPersist a = q;
    a.nhelp = std::max(1, std::min(std::max(1, kLuReserveSms - 1), np));
    launch(k_lp_init, nblocks(std::max(nB, np), 256), 256, 0, a);
    lp_dispatch([&](auto kern, int nt) {
      launch(kern, dim3(1 + a.nhelp), dim3(nt), lp_smem_bytes<T>(nB), Phi, a, (const LmDeviceState*)st, gate_running);
    });
  }

  static constexpr int kLu4Rpt = sizeof(T) == 8 ? 2 : 1;
  static constexpr int kLu4Thr = 256;
  bool use_lu4 = false;
  void plan_lu3() {
    invL = dalloc<T>(2 * kLuMaxKB * kLuMaxKB);
    gring = dalloc<int>(2 * (4 * kLuMaxKB + 4));
    {
      int plo = 0, phi = 0;
      CPF_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&plo, &phi));
      CPF_CUDA_CHECK(cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, phi));
      // one level below the panels / trailing updates: the merges fill SMs the LU leaves idle and
      // must not hold up a panel cluster's launch
      int ptri = std::min(plo, phi + 1);
      if (const char* e = knob("CPF_TRI_PRIO")) ptri = std::max(phi, std::min(plo, phi + atoi(e)));
      CPF_CUDA_CHECK(cudaStreamCreateWithPriority(&s4, cudaStreamNonBlocking, ptri));
      CPF_CUDA_CHECK(cudaStreamCreateWithPriority(&sS4, cudaStreamNonBlocking, ptri));
    }
    CPF_CUDA_CHECK(cudaEventCreateWithFlags(&evT, cudaEventDisableTiming));
    CPF_CUDA_CHECK(cudaEventCreateWithFlags(&evT2, cudaEventDisableTiming));
    if (const char* e = knob("CPF_TRI_PROG")) tri_prog = e[0] != '0';
    CPF_CUDA_CHECK(cudaEventCreateWithFlags(&evP, cudaEventDisableTiming));
    CPF_CUDA_CHECK(cudaEventCreateWithFlags(&evB, cudaEventDisableTiming));
    CPF_CUDA_CHECK(cudaEventCreateWithFlags(&evJ, cudaEventDisableTiming));
    for (auto& e : evB2) CPF_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    lu3_rpt = 0;
    // CPF_PANEL_SMEM=1: the shared-memory cluster panel (lu.cuh k_panel_lu), otherwise used only
    // when n_B exceeds 16 register-panel CTAs (n_B > 8192) -- lets the tests cover it at small n_B
    if (const char* e = knob("CPF_PANEL_SMEM")) if (e[0] == '1') return;
    // (rows/thread, threads/CTA) candidates, smallest per-SM work first; cluster <= 16 CTAs
    const int cand[2][2] = {{1, 128}, {sizeof(T) == 8 ? 2 : 1, 256}};
    int start = 0;
    if (const char* e = knob("CPF_PANEL_WIDE")) if (e[0] == '1') start = 1;  // experiment knob
    for (int ci = start; ci < 2; ++ci) {
      const auto& c = cand[ci];
      if ((nB + c[0] * c[1] - 1) / (c[0] * c[1]) <= 16) { lu3_rpt = c[0]; lu3_thr = c[1]; break; }
    }
    if (!lu3_rpt) return;  // fall back to the smem panel
    // the rotating-frame panel wins from n_B ~ 1000 up (config 4: 1200, config 1: 4800; measured
    // slower at 300 / 900), and its 2-3 CTA clusters co-schedule next to the persistent pass B
    use_lu4 = nB > 1024 && (nB + kLu4Rpt * kLu4Thr - 1) / (kLu4Rpt * kLu4Thr) <= 16;
    if (const char* e = knob("CPF_PANEL_V3")) if (e[0] == '1') use_lu4 = false;
    if (use_lu4) {
      const size_t smem = panel4_smem_bytes<T>(16, kLu4Thr, kLu4Rpt);
      CPF_CUDA_CHECK(cudaFuncSetAttribute(k_panel_lu4<T, kLu4Rpt, kLu4Thr>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
      CPF_CUDA_CHECK(cudaFuncSetAttribute(k_panel_lu4<T, kLu4Rpt, kLu4Thr>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    auto setattr = [&](auto kern, int thr) {
      const size_t smem = panel3_smem_bytes<T>(16, kLuMaxKB, thr);
      CPF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      CPF_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    };
    setattr(k_panel_lu3<T, kLuMaxKB, 1, 128>, 128);
    if constexpr (sizeof(T) == 8) setattr(k_panel_lu3<T, kLuMaxKB, 2, 256>, 256);
    else setattr(k_panel_lu3<T, kLuMaxKB, 1, 256>, 256);
  }

  void launch_panel4(int k0, int kb, int cl, int gate_running, LuWork wk, T* invl, PanelPrev<T> pv) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(kLu4Thr);
    cfg.dynamicSmemBytes = panel4_smem_bytes<T>(cl, kLu4Thr, kLu4Rpt);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    // consecutive panels on stream s: the next panel's launch overlaps this one's tail
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_panels ? 2 : 1;
    CPF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_panel_lu4<T, kLu4Rpt, kLu4Thr>, Phi, nB, nB, k0, kb, wk, invl,
                                      (const LmDeviceState*)st, gate_running, pv));
    ++nlaunch;
  }

  template <int RPTc, int THR>
  void launch_panel3(int k0, int kb, int cl, int gate_running, LuWork wk, T* invl, PanelPrev<T> pv) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cl);
    cfg.blockDim = dim3(THR);
    cfg.dynamicSmemBytes = panel3_smem_bytes<T>(cl, kLuMaxKB, THR);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_panels ? 2 : 1;
    CPF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_panel_lu3<T, kLuMaxKB, RPTc, THR>, Phi, nB, nB, k0, kb, wk, invl,
                                      (const LmDeviceState*)st, gate_running, pv));
    ++nlaunch;
  }

  template <int NT>
  void set_dmma_attrs() {
    CPF_CUDA_CHECK(cudaFuncSetAttribute(k_pass_dmma<NT, 0, kDmmaCK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)da_smem));
    CPF_CUDA_CHECK(cudaFuncSetAttribute(k_pass_dmma<NT, 1, kDmmaCK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)db_smem));
    CPF_CUDA_CHECK(cudaFuncSetAttribute(k_pass_b_dmma_pers<NT, kDmmaCK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)db_smem));
  }
  template <class F>
  void dispatch_nt(F&& f) {
    switch (dm_nt) {
      case 1: f(IC<1>{}); break;
      case 2: f(IC<2>{}); break;
      case 3: f(IC<3>{}); break;
      case 4: f(IC<4>{}); break;
      case 5: f(IC<5>{}); break;
      case 6: f(IC<6>{}); break;
      case 8: f(IC<8>{}); break;
      default: throw ApiError(CPF_E_UNSUPPORTED, "unsupported DMMA n-tile count");
    }
  }

  // Ozaki passes: chosen for large real tensors (config 4: 2.45 ms per pass instead of 3.3 ms on
  // DMMA); CPF_OZ=1 forces them for any real tensor with R <= 32 (tests), CPF_OZ=0 disables.
  void plan_oz() {
    use_oz = false;
    if constexpr (sizeof(T) != 8) return;
    else {
      const char* e = knob("CPF_OZ");
      const bool force = e && e[0] == '1';
      if (e && e[0] == '0') return;
      // int32 accumulators: 8 pairs x 127^2 per K element -> K <= 16384 per contraction
      if (R > kOzN || Cloc < 1 || Cloc > 16384 || Lmid > 16384) return;
      if (!force && (I1 < 256 || Jloc < ((int64_t)1 << 26))) return;
      const int nb = (int)((I1 + kOzM - 1) / kOzM);
      oa = OzGeom{I1, Lmid, Cloc, nb, (int)((Cloc + kOzK - 1) / kOzK), Lmid, (int64_t)nb * Lmid, R, 0};
      ob = OzGeom{I1, Lmid, Cloc, nb, (int)((Lmid + kOzK - 1) / kOzK), Cloc, (int64_t)nb * Cloc, R, 0};
      // pass A streams alone: no L2 hint (measured 3 % faster); pass B runs beside the LU: evict-first
      oa.dbg = 4;
      if (const char* d = knob("CPF_OZ_DBG")) oa.dbg = ob.dbg = atoi(d);  // experiments
      // the two digit-plane images (~2 x 8 B per element) must fit next to everything else with
      // 2 GB to spare; otherwise stay on the fp64 DMMA passes
      const size_t need = ((size_t)oa.ntiles * oa.nkb + (size_t)ob.ntiles * ob.nkb) * kOzABytes;
      size_t free_b = 0, total_b = 0;
      CPF_CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
      // memory the stream-ordered pool holds but does not use is available to this engine too
      // (cudaMemGetInfo counts it as used; the pool never releases it, see configure_pool)
      {
        cudaMemPool_t pool;
        uint64_t reserved = 0, used = 0;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess &&
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
            cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && reserved > used)
          free_b += (size_t)(reserved - used);
      }
      // so are the tensor-sized buffers an earlier engine of this process parked in the reuse cache
      // (big_alloc takes them back or releases them): the plan must not depend on what ran before
      free_b += BigCache::parked_bytes(dev);
      if (!force && need + ((size_t)2 << 30) + (size_t)Jloc * sizeof(T) > free_b) return;
      ozYA = static_cast<uint8_t*>(big_alloc((size_t)oa.ntiles * oa.nkb * kOzABytes, true));
      ozYB = static_cast<uint8_t*>(big_alloc((size_t)ob.ntiles * ob.nkb * kOzABytes, true));
      ozFrowA = dalloc<int>((size_t)oa.ntiles * kOzM);
      ozFrowB = dalloc<int>((size_t)ob.ntiles * kOzM);
      ozBA = dalloc<uint8_t>((size_t)oa.nkb * kOzBBytes);  // zero: padding columns / K tail
      ozBB = dalloc<uint8_t>((size_t)ob.nkb * kOzBBytes);
      ozFr = dalloc<int>(2 * kOzN);
      ozM1 = dalloc<double>((size_t)std::max(1, nsm_ / nb) * I1 * RP);
      ozZ = dalloc<double>((size_t)nb * Lmid * RP);
      ozBp = dalloc<double>((size_t)Cloc * nb * RP);
      CPF_CUDA_CHECK(cudaFuncSetAttribute(k_oz_pass<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOzSmem));
      CPF_CUDA_CHECK(cudaFuncSetAttribute(k_oz_pass<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOzSmem));
      use_oz = true;
    }
  }
  // speculative rejection branch: on for the FMA-pass tensors (C2 416 -> 446, C3 693 -> 732 it/s)
  // and, since pass A runs on the low-priority stream beside it (spec_a_side), for the int8 passes
  // (config 4: 172.6 -> 183 it/s; with pass A on the LU's own priority level the branch's trailing
  // updates were held back until the pass's persistent grid retired and the branch lost).  Off
  // for the fp64 DMMA passes (not measured with the side stream).  CPF_SPEC=0/1 overrides.
  void plan_spec() {
    use_spec = use_inv && lu3_rpt && (use_oz || !use_dmma);
    if (const char* e = knob("CPF_SPEC")) use_spec = e[0] == '1' && use_inv && lu3_rpt;
    // the experimental persistent LU's CTAs read the gate state themselves (no latch): never beside
    // a running k_decide
    if (lp_cfg) use_spec = false;
    if (!use_spec) return;
    if (const char* e = knob("CPF_SPEC_RESERVE")) kSpecReserveSms = atoi(e);
    if (const char* e = knob("CPF_SPEC_A_SIDE")) spec_a_side = e[0] != '0';
    const size_t R2 = (size_t)R * R;
    PhiS = dalloc<T>((size_t)nB * nB);
    PhiInvS = dalloc<T>((size_t)nB * nB);
    TriTmpS = dalloc<T>((size_t)nB * nB);
    if (nB > 256) TriPartS = dalloc<T>((size_t)kTriSplit * nB * nB);
    GtiS = dalloc<T>(N * R2);
    GiS = dalloc<T>(N * R2);
    invLS = dalloc<T>(2 * kLuMaxKB * kLuMaxKB);
    gringS = dalloc<int>(2 * (4 * kLuMaxKB + 4));
    const int nblk32 = (nB + 31) / 32;
    ibufS = dalloc<int>((size_t)2 * nB + 4 * kLuMaxKB + 8 + 2 * nblk32);
    luS.perm = ibufS;
    luS.ipiv = ibufS + nB;
    luS.gather = ibufS + 2 * nB;
    luS.gcount = luS.gather + 4 * kLuMaxKB;
    luS.info = luS.gcount + 1;
    luS.ticket = luS.info + 1;
    luS.ready = luS.ticket + 4;
    spec_sing = dalloc<int>(2);
    luS.latch = dalloc<int>((nB + kLuMaxKB - 1) / kLuMaxKB + 2);
    if (lp_cfg) {
      alloc_lp(lpS);
      lpS.perm = luS.perm;
      lpS.info = luS.info;
      lpS.tmp = TriTmpS;
    }
    int plo = 0, phi = 0;
    CPF_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&plo, &phi));
    CPF_CUDA_CHECK(cudaStreamCreateWithPriority(&sS, cudaStreamNonBlocking, phi));
    CPF_CUDA_CHECK(cudaStreamCreateWithPriority(&sS2, cudaStreamNonBlocking, phi));
    CPF_CUDA_CHECK(cudaEventCreateWithFlags(&evS0, cudaEventDisableTiming));
    CPF_CUDA_CHECK(cudaEventCreateWithFlags(&evS1, cudaEventDisableTiming));
  }
  void swap_spec() {
    std::swap(Phi, PhiS);
    std::swap(PhiInv, PhiInvS);
    std::swap(TriTmp, TriTmpS);
    std::swap(TriPart, TriPartS);
    std::swap(Gti, GtiS);
    std::swap(Gi, GiS);
    std::swap(invL, invLS);
    std::swap(gring, gringS);
    std::swap(lu, luS);
    std::swap(lp, lpS);
    std::swap(s, sS);
    std::swap(s2, sS2);
    std::swap(s4, sS4);
  }

  // one-time digit-plane images of the bound tensor (both passes), stream-ordered after the upload.
  // Accuracy guard (tensor_pass_oz.cuh): if any row of either pass's view of Y is outside the int8
  // split's envelope, the engine drops the int8 passes for this tensor and stays on fp64.
  bool oz_y_rejected = false;
  // Host upload of a large real tensor in slices of the last mode, with the pass-B image built
  // behind it: a pass-B tile row (i1, c) is complete once slice c has arrived, so its row exponents
  // and digit planes are computed on s3 while the next slices cross PCIe (the pass-A rows span all
  // c and wait for the whole tensor).  Same kernels on tile ranges: identical image bytes.
  // Returns false (nothing done) when the plan does not apply.
  bool upload_with_split(const void* p) {
    if constexpr (sizeof(T) != 8) return false;
    else {
      bool force = false;
      if (const char* e = knob("CPF_UPLOAD_SPLIT")) {
        if (e[0] == '0') return false;
        force = true;  // tests: at any size
      }
      if (!use_oz || Cloc < 16 || (!force && Jloc < ((int64_t)1 << 27))) return false;
      const double* Yd = reinterpret_cast<const double*>(Yown);
      int* ybad = reinterpret_cast<int*>(red);  // scratch
      CPF_CUDA_CHECK(cudaMemsetAsync(ybad, 0, sizeof(int), s));
      const int nchunk = 8;
      const int64_t per = (Cloc + nchunk - 1) / nchunk, slice = Lrows;
      cudaEvent_t ev = nullptr, evEnd = nullptr;
      CPF_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      CPF_CUDA_CHECK(cudaEventCreateWithFlags(&evEnd, cudaEventDisableTiming));
      for (int64_t c0 = 0; c0 < Cloc; c0 += per) {
        const int64_t c1 = std::min(Cloc, c0 + per);
        CPF_CUDA_CHECK(cudaMemcpyAsync(Yown + c0 * slice, static_cast<const T*>(p) + c0 * slice,
                                       (size_t)((c1 - c0) * slice) * sizeof(T), cudaMemcpyHostToDevice, s));
        CPF_CUDA_CHECK(cudaEventRecord(ev, s));
        CPF_CUDA_CHECK(cudaStreamWaitEvent(s3, ev, 0));
        // pass-B tiles t = c * nb + b of the slices [c0, c1)
        k_oz_rowexp<1><<<nsm_ * 2, 256, 0, s3>>>(Yd, ob, ozFrowB, ybad, c0 * ob.nb, c1 * ob.nb);
        k_oz_split_y<1><<<nsm_ * 4, 256, 0, s3>>>(Yd, ob, ozFrowB, ozYB, c0 * ob.nb, c1 * ob.nb);
        CPF_CUDA_CHECK(cudaGetLastError());
      }
      CPF_CUDA_CHECK(cudaEventRecord(evEnd, s3));
      CPF_CUDA_CHECK(cudaStreamWaitEvent(s, evEnd, 0));
      cudaEventDestroy(ev);
      cudaEventDestroy(evEnd);
      Y = Yown;
      oz_split(/*pass_b_done=*/true);
      return true;
    }
  }
  void oz_split(bool pass_b_done = false) {
    NvtxRange nvtx_("cpf.oz_split (int8 digit-plane images)");
    if (!use_oz || Jloc == 0) return;
    if constexpr (sizeof(T) == 8) {
      const double* Yd = reinterpret_cast<const double*>(Y);
      int* ybad = reinterpret_cast<int*>(red);  // scratch
      if (!pass_b_done) CPF_CUDA_CHECK(cudaMemsetAsync(ybad, 0, sizeof(int), s));
      k_oz_rowexp<0><<<nsm_ * 8, 256, 0, s>>>(Yd, oa, ozFrowA, ybad);
      if (!pass_b_done) k_oz_rowexp<1><<<nsm_ * 8, 256, 0, s>>>(Yd, ob, ozFrowB, ybad);
      CPF_CUDA_CHECK(cudaGetLastError());
      int nbad = 0;
      CPF_CUDA_CHECK(cudaMemcpyAsync(&nbad, ybad, sizeof(int), cudaMemcpyDeviceToHost, s));
      CPF_CUDA_CHECK(cudaStreamSynchronize(s));
      if (nbad > 0) {
        oz_y_rejected = true;
        use_oz = false;
        big_free(ozYA);
        big_free(ozYB);
        ozYA = ozYB = nullptr;
        kLuReserveSms = 24;
        if (const char* e = knob("CPF_LU_RESERVE")) kLuReserveSms = atoi(e);
        if (use_dmma && !knob("CPF_SPEC")) use_spec = false;  // fp64 DMMA passes: branch off (plan_spec)
        return;
      }
      k_oz_split_y<0><<<nsm_ * 16, 256, 0, s>>>(Yd, oa, ozFrowA, ozYA);
      if (!pass_b_done) k_oz_split_y<1><<<nsm_ * 16, 256, 0, s>>>(Yd, ob, ozFrowB, ozYB);
      CPF_CUDA_CHECK(cudaGetLastError());
    }
  }

  void plan_dmma(int nsm) {
    use_dmma = false;
    if constexpr (sizeof(T) != 8) return;
    else {
      if (I1 < 256 || I1 % 2 != 0 || Cloc < 1) return;
      if (const char* e = knob("CPF_NO_DMMA")) if (e[0] == '1') return;
      dm_nt = (R + 7) / 8;
      if (dm_nt == 7) dm_nt = 8;
      int ws = 8 * dm_nt;
      while (ws % 16 != 4) ++ws;
      auto fill = [&](DmmaGeom& g) {
        g.I1 = I1; g.Lmid = Lmid; g.C = Cloc; g.WS = ws;
        g.tiles = (int)((I1 + kDmmaRows - 1) / kDmmaRows);
        g.CK = kDmmaCK;
        g.stage_elems = ((size_t)g.CK * (kDmmaSLp + ws) + 15) / 16 * 16;
      };
      fill(da);
      fill(db);
      const size_t sb = da.stage_elems * sizeof(double);
      const size_t m1b = 0;  // M_1 accumulates in global (L2-resident) memory
      const size_t redb = (size_t)8 * 8 * dm_nt * sizeof(double);
      const size_t budget = (size_t)220 * 1024 - 128;
      if (m1b + redb + 2 * sb > budget) return;
      da.NST = (int)std::min<size_t>(6, (budget - m1b - redb) / sb);
      db.NST = (int)std::min<size_t>(6, (budget - redb) / sb);
      da_smem = 128 + (size_t)da.NST * sb + m1b + redb;
      db_smem = 128 + (size_t)db.NST * sb + redb;
      int64_t groups = std::max<int64_t>(1, ((int64_t)nsm + da.tiles - 1) / da.tiles);
      groups = std::min<int64_t>(groups, Lmid);
      da.m_per_cta = (Lmid + groups - 1) / groups;
      da_groups = (int)((Lmid + da.m_per_cta - 1) / da.m_per_cta);
      int64_t per_c = std::max<int64_t>(1, 2 * (int64_t)nsm / std::max<int64_t>(1, Cloc * db.tiles));
      per_c = std::min<int64_t>(per_c, std::max<int64_t>(1, Lmid / 64));
      db.m_per_cta = (Lmid + per_c - 1) / per_c;
      db_chunks = (int)((Lmid + db.m_per_cta - 1) / db.m_per_cta);
      WNd = dalloc<double>((size_t)Cloc * ws + 8);
      KMd = dalloc<double>((size_t)Lmid * ws + 8);
      if (zpart) cudaFreeAsync(zpart, s);
      if (m1part) cudaFreeAsync(m1part, s);
      if (bpart) cudaFreeAsync(bpart, s);
      zpart = dalloc<T>((size_t)da.tiles * Lmid * RP);
      m1part = dalloc<T>((size_t)std::max(da_groups, 1) * I1 * RP + (size_t)Cloc * db_chunks * db.tiles * RP);
      bpart = dalloc<T>((size_t)std::max<int64_t>(Cloc, 1) * db_chunks * db.tiles * RP);
      dispatch_nt([&](auto ntc) { this->template set_dmma_attrs<decltype(ntc)::value>(); });
      use_dmma = true;
    }
  }

  void plan_v2(int nsm) {
    const bool cplx = sizeof(T) == 16;
    use_v2 = cplx || (I1 % 2 == 0);
    if (!use_v2) return;
    rpt = (!cplx && RP <= 24) ? 2 : 1;
    const int nthr = 256;
    const size_t es = sizeof(T);
    auto base = [&](PassGeom& g) {
      g.I1 = I1; g.Lmid = Lmid; g.C = Cloc; g.RPT = rpt;
      const int64_t tilmax = (int64_t)nthr * rpt;
      if (I1 <= tilmax) {
        g.full = 1;
        g.TI = (int)((I1 + rpt - 1) / rpt);
        g.TM = std::max(1, nthr / g.TI);
        g.tiles = 1;
      } else {
        g.full = 0;
        g.TI = nthr;
        g.TM = 1;
        g.tiles = (int)((I1 + tilmax - 1) / tilmax);
      }
    };
    auto round_up = [](size_t v, size_t m) { return (v + m - 1) / m * m; };
    const size_t align_e = 128 / es;
    // ---- pass A
    base(ga);
    {
      const int64_t tilmax = (int64_t)nthr * rpt;
      ga.SL = ga.full ? I1 * ga.TM : tilmax;
      const size_t side = (size_t)RP * nthr * es * (1 + rpt);  // zs + m1 slots
      const size_t budget = (size_t)220 * 1024 - 256 - side;
      // c per stage: ~32 KB stages, at least 2 stages within the budget
      int64_t ck = std::min<int64_t>(32, 32768 / std::max<int64_t>(1, ga.SL * (int64_t)es));
      const int64_t ckmax = (int64_t)(budget / 2) / (int64_t)((ga.SL + RP) * es) - 1;
      ck = std::min(ck, ckmax);
      ck &= ~(int64_t)1;
      if (ck < 2 || side > (size_t)180 * 1024) {
        use_v2 = false;  // shape outside the staged kernel's smem envelope: LDG path
        return;
      }
      ga.CK = (int)ck;
      ga.stage_elems = round_up((size_t)ga.CK * ga.SL + (size_t)ga.CK * RP + 2, align_e);
      ga.NST = (int)std::max<size_t>(2, std::min<size_t>(8, budget / (ga.stage_elems * es)));
      ga_smem = 128 + (size_t)ga.NST * ga.stage_elems * es + side;
      int64_t groups = std::max<int64_t>(1, (2 * (int64_t)nsm + ga.tiles - 1) / ga.tiles);
      int64_t mper = (Lmid + groups - 1) / groups;
      mper = ((mper + ga.TM - 1) / ga.TM) * ga.TM;
      ga.m_per_cta = mper;
      ga_groups = (int)((Lmid + mper - 1) / mper);
    }
    // ---- pass B
    base(gb);
    {
      const int64_t tilmax = (int64_t)nthr * rpt;
      gb.SL = gb.full ? I1 : tilmax;
      int ck = (int)std::max<int64_t>(2, std::min<int64_t>(64, 32768 / std::max<int64_t>(1, gb.SL * (int64_t)es)));
      ck &= ~1;
      gb.CK = std::max(2, ck);
      gb.stage_elems = round_up((size_t)gb.CK * gb.SL + (size_t)gb.CK * RP + 2, align_e);
      gb.NST = (int)std::max<size_t>(2, std::min<size_t>(8, (140 * 1024) / (gb.stage_elems * es)));
      gb_smem = 128 + (size_t)gb.NST * gb.stage_elems * es + (size_t)RP * 8 * es;
      int64_t per_c = std::max<int64_t>(1, 2 * (int64_t)nsm / std::max<int64_t>(1, Cloc * gb.tiles));
      per_c = std::min<int64_t>(per_c, std::max<int64_t>(1, Lmid / gb.CK));
      int64_t mper = (Lmid + per_c - 1) / per_c;
      mper = ((mper + gb.CK - 1) / gb.CK) * gb.CK;
      gb.m_per_cta = mper;
      gb_chunks = (int)((Lmid + mper - 1) / mper);
    }
    if (zpart) cudaFreeAsync(zpart, s);
    if (m1part) cudaFreeAsync(m1part, s);
    if (bpart) cudaFreeAsync(bpart, s);
    zpart = dalloc<T>((size_t)ga.tiles * Lmid * RP);
    m1part = dalloc<T>((size_t)ga_groups * I1 * RP);
    bpart = dalloc<T>((size_t)std::max<int64_t>(Cloc, 1) * gb_chunks * gb.tiles * RP);
  }

  // ------------------------------------------------------------------------------------------
  // launch helpers
  template <class K, class... Args>
  void launch(K kern, dim3 g, dim3 b, size_t smem, Args... args) {
    if (g.x == 0 || g.y == 0 || g.z == 0) return;
    if (use_pdl && pdl_now) {  // programmatic dependent launch (pdl_wait, cpf_common.cuh)
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = g;
      cfg.blockDim = b;
      cfg.dynamicSmemBytes = smem;
      cfg.stream = ls;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      CPF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, args...));
    } else {
      kern<<<g, b, smem, ls>>>(args...);
    }
    ++nlaunch;
    CPF_CUDA_CHECK(cudaGetLastError());
  }
  static unsigned nblocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

  int cur_phase = -1;
  cudaEvent_t cur_ev = nullptr;
  void ph_begin(int ph) {
    if (!prof) return;
    cudaEvent_t a;
    CPF_CUDA_CHECK(cudaEventCreate(&a));
    CPF_CUDA_CHECK(cudaEventRecord(a, ls));
    cur_phase = ph;
    cur_ev = a;
  }
  void ph_end() {
    if (!prof || cur_phase < 0) return;
    cudaEvent_t b;
    CPF_CUDA_CHECK(cudaEventCreate(&b));
    CPF_CUDA_CHECK(cudaEventRecord(b, ls));
    evs.push_back({cur_phase, cur_ev, b});
    cur_phase = -1;
  }

  // ------------------------------------------------------------------------------------------
  // tensor passes
  // ------------------------------------------------------------------------------------------
  template <int RPc>
  void set_pass_attrs_t() {
    CPF_CUDA_CHECK(cudaFuncSetAttribute(k_pass_a<T, RPc>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pa_smem));
    if (use_v2) {
      if (rpt == 2) {
        if constexpr (sizeof(T) == 8) {
          CPF_CUDA_CHECK(cudaFuncSetAttribute(k_pass_a2<T, RPc, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ga_smem));
          CPF_CUDA_CHECK(cudaFuncSetAttribute(k_pass_b2<T, RPc, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gb_smem));
        }
      } else {
        CPF_CUDA_CHECK(cudaFuncSetAttribute(k_pass_a2<T, RPc, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ga_smem));
        CPF_CUDA_CHECK(cudaFuncSetAttribute(k_pass_b2<T, RPc, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gb_smem));
      }
    }
  }
  void set_pass_attrs() { dispatch_rp([&](auto rpc) { this->template set_pass_attrs_t<decltype(rpc)::value>(); }); }

  template <int V> struct IC { static constexpr int value = V; };
  template <class F>
  void dispatch_rp(F&& f) {
    switch (RP) {
      case 2: f(IC<2>{}); break;
      case 4: f(IC<4>{}); break;
      case 6: f(IC<6>{}); break;
      case 8: f(IC<8>{}); break;
      case 10: f(IC<10>{}); break;
      case 12: f(IC<12>{}); break;
      case 16: f(IC<16>{}); break;
      case 20: f(IC<20>{}); break;
      case 24: f(IC<24>{}); break;
      case 32: f(IC<32>{}); break;
      case 40: f(IC<40>{}); break;
      case 48: f(IC<48>{}); break;
      case 64: f(IC<64>{}); break;
      default: throw ApiError(CPF_E_UNSUPPORTED, "unsupported padded rank");
    }
  }

  // conj row-major operand copies for factors F (stacked)
  void prep_operands(const T* F, bool need_wn, int gate) {
    launch(k_conj_rowmajor<T>, nblocks(I1 * RP, 256), 256, 0, F + offs[0], I1, (int64_t)0, I1, R, RP, A1c, (const LmDeviceState*)st, (const DevFlags*)fl, gate, 1);
    if (N == 3) {
      launch(k_conj_rowmajor<T>, nblocks(Lmid * RP, 256), 256, 0, F + offs[1], Lmid, (int64_t)0, Lmid, R, RP, KMc, (const LmDeviceState*)st, (const DevFlags*)fl, gate, 1);
    } else {
      launch(k_krmid<T>, nblocks(Lmid * RP, 256), 256, 0, (const T*)F, mg, Lmid, R, RP, KMc, (const LmDeviceState*)st, (const DevFlags*)fl, gate, 1);
    }
    if (need_wn && Cloc > 0)
      launch(k_conj_rowmajor<T>, nblocks(Cloc * RP, 256), 256, 0, F + offs[N - 1], Cloc, slab_lo, IN, R, RP, WNc, (const LmDeviceState*)st, (const DevFlags*)fl, gate, 1);
  }

  int* oz_bad_ptr(int pass) {
    return reinterpret_cast<int*>(reinterpret_cast<char*>(fl) + offsetof(DevFlags, oz_bad)) + pass * kOzGuardCols;
  }

  // Pass A at factors F -> out modes 1..N-1 of Mout (stacked), allreduced.
  // Int8 (Ozaki) passes: the operand split also checks the accuracy envelope; the int8 kernels are
  // gated on it and the fp64 pass below runs instead when the operand is outside it.
  void pass_a(const T* F, T* Mout, int gate) {
    NvtxRange nvtx_("cpf.pass_a");
    prep_operands(F, true, gate);
    ph_begin(kPhPassA);
    bool oz = false;
    if constexpr (sizeof(T) == 8) {
      if (Cloc > 0 && use_oz) {
        oz = true;
        const LmDeviceState* cst = st;
        const DevFlags* cfl = fl;
        const int go = gate | kGateIfOzOk, gf = gate | kGateIfOzBad;
        launch(k_oz_split_b, dim3(R), 256, 0, (const double*)WNc, Cloc, R, RP, ozBA, ozFr, oz_bad_ptr(0), cst, cfl,
               gate);
        // beside a speculated core system, pass A leaves the LU its SMs like pass B does
        const int nch = std::max(1, (use_spec ? nsm_ - kSpecReserveSms : nsm_) / oa.nb);
        const OzOut oo{(const double*)A1c, (const double*)KMc, RP, nch, (Lmid + nch - 1) / nch, ozM1, ozZ};
        // beside a speculated core system the pass runs on the low-priority stream (like pass B in
        // the fork): on the LU's own priority level its resident persistent grid held back the
        // branch's trailing updates until it retired
        const bool side = use_spec && spec_a_side && ls == s && gate == kRunning;
        if (side) {
          CPF_CUDA_CHECK(cudaEventRecord(evF, s));
          CPF_CUDA_CHECK(cudaStreamWaitEvent(s3, evF, 0));
          ls = s3;
        }
        launch(k_oz_pass<0>, dim3((unsigned)(oa.nb * nch)), kOzThreads, kOzSmem, (const uint8_t*)ozYA,
               (const int*)ozFrowA, (const uint8_t*)ozBA, (const int*)ozFr, oa, oo, cst, cfl, go);
        if (side) {
          ls = s;
          CPF_CUDA_CHECK(cudaEventRecord(evG, s3));
          CPF_CUDA_CHECK(cudaStreamWaitEvent(s, evG, 0));
        }
        ph_end();
        launch(k_m1_reduce<T>, nblocks(I1 * R, 32), 256, 0, (const T*)ozM1, nch, I1, R, RP, pa_out, cst, cfl, go);
        launch(k_z_reduce<T>, nblocks(Lmid * R, 256), 256, 0, (const T*)ozZ, oa.nb, Lmid, R, RP, pa_out + I1 * R,
               cst, cfl, go);
        launch(k_oz_note_fallback, 1, 1, 0, fl, cst, gf);
        pass_a_fp64(F, gf);
      }
    }
    if (!oz) pass_a_fp64(F, gate);
    if (comm) comm->allreduce_sum((double*)pa_out, (size_t)(I1 + Lmid) * R * (sizeof(T) / sizeof(double)), s);
    // scatter: M_1 = pa_out[0 : I1 R]; N==3: M_2 = Z; N>=4: M_2..M_{N-1} from Z (at F)
    launch(k_copy<T>, nblocks(I1 * R, 256), 256, 0, (const T*)pa_out, Mout + offs[0], I1 * R, (const LmDeviceState*)st, (const DevFlags*)fl, gate);
    if (N == 3) {
      launch(k_copy<T>, nblocks(Lmid * R, 256), 256, 0, (const T*)(pa_out + I1 * R), Mout + offs[1], Lmid * R, (const LmDeviceState*)st, (const DevFlags*)fl, gate);
    } else if (N >= 4) {
      for (int k = 0; k < N - 2; ++k)
        launch(k_mid_mttkrp<T>, nblocks(mg.dims[k] * R, 128), 128, 0, (const T*)(pa_out + I1 * R), Lmid, F, mg, k, R,
               Mout + offs[k + 1], (const LmDeviceState*)st, (const DevFlags*)fl, gate);
    }
  }

  // fp64 pass A (DMMA / staged DFMA / plain) -> pa_out partial sums of this slab
  void pass_a_fp64(const T* F, int gate) {
    if constexpr (sizeof(T) == 8) {
      if (Cloc > 0 && use_dmma) {
        const LmDeviceState* cst = st;
        const DevFlags* cfl = fl;
        launch(k_conj_rowmajor<T>, nblocks(Cloc * da.WS, 256), 256, 0, (const T*)(F + offs[N - 1]), Cloc, slab_lo, IN, R,
               da.WS, (T*)WNd, cst, cfl, gate, 1);
        dispatch_nt([&](auto ntc) {
          constexpr int NTc = decltype(ntc)::value;
          launch(k_pass_dmma<NTc, 0, kDmmaCK>, dim3(da.tiles, da_groups), dim3(kConsumers + 32), da_smem, (const double*)Y, da,
                 (const double*)WNd, (const double*)A1c, (const double*)KMc, RP, R, (double*)zpart, (double*)m1part,
                 cst, cfl, gate);
        });
        ph_end();
        launch(k_m1_reduce<T>, nblocks(I1 * R, 32), 256, 0, (const T*)m1part, da_groups, I1, R, RP, pa_out, cst, cfl,
               gate);
        launch(k_z_reduce<T>, nblocks(Lmid * R, 256), 256, 0, (const T*)zpart, da.tiles, Lmid, R, RP, pa_out + I1 * R,
               cst, cfl, gate);
        return;
      }
    }
    if (Cloc > 0 && use_v2) {
      dispatch_rp([&](auto rpc) {
        constexpr int RPc = decltype(rpc)::value;
        if (rpt == 2) {
          if constexpr (sizeof(T) == 8)
            launch(k_pass_a2<T, RPc, 2>, dim3(ga.tiles, ga_groups), dim3(kConsumers + 32), ga_smem, Y, ga, (const T*)WNc,
                   (const T*)A1c, (const T*)KMc, zpart, m1part, (const LmDeviceState*)st, (const DevFlags*)fl, gate);
        } else {
          launch(k_pass_a2<T, RPc, 1>, dim3(ga.tiles, ga_groups), dim3(kConsumers + 32), ga_smem, Y, ga, (const T*)WNc,
                 (const T*)A1c, (const T*)KMc, zpart, m1part, (const LmDeviceState*)st, (const DevFlags*)fl, gate);
        }
      });
      ph_end();
      launch(k_m1_reduce<T>, nblocks(I1 * R, 32), 256, 0, (const T*)m1part, ga_groups, I1, R, RP, pa_out,
             (const LmDeviceState*)st, (const DevFlags*)fl, gate);
      launch(k_z_reduce<T>, nblocks(Lmid * R, 256), 256, 0, (const T*)zpart, ga.tiles, Lmid, R, RP, pa_out + I1 * R,
             (const LmDeviceState*)st, (const DevFlags*)fl, gate);
    } else if (Cloc > 0) {
      dispatch_rp([&](auto rpc) {
        constexpr int RPc = decltype(rpc)::value;
        launch(k_pass_a<T, RPc>, dim3(pa_tiles, pa_groups), dim3(pa_threads), pa_smem, Y, I1, Lmid, Cloc,
               (const T*)WNc, (const T*)A1c, (const T*)KMc, pa_TI, pa_TM, pa_mper, zpart, m1part, (const LmDeviceState*)st, (const DevFlags*)fl, gate);
      });
      ph_end();
      launch(k_pass_a_reduce<T>, nblocks((I1 + Lmid) * R, 256), 256, 0, (const T*)m1part, pa_groups,
             (const T*)zpart, pa_tiles, I1, Lmid, R, RP, pa_out, pa_out + I1 * R, (const LmDeviceState*)st, (const DevFlags*)fl, gate);
    } else {
      ph_end();
      CPF_CUDA_CHECK(cudaMemsetAsync(pa_out, 0, sizeof(T) * (I1 + Lmid) * R, s));
    }
  }

  // Pass B at factors F -> mode N of Mout (allgathered).  Int8 passes: guarded like pass A.
  void pass_b(const T* F, T* Mout, int gate) {
    NvtxRange nvtx_("cpf.pass_b");
    prep_operands(F, false, gate);
    ph_begin(kPhPassB);
    struct Red { const T* src; int nparts; int gate; };
    Red reds[2];
    int nred = 0;
    bool oz = false;
    if constexpr (sizeof(T) == 8) {
      if (Cloc > 0 && use_oz) {
        oz = true;
        const int go = gate | kGateIfOzOk | kGateOzPass, gf = gate | kGateIfOzBad | kGateOzPass;
        // overlapped with the next LU (ls != s): leave kLuReserveSms SMs to the panel clusters
        const int grid = ls != s ? std::max(1, nsm_ - kLuReserveSms) : nsm_;
        launch(k_oz_split_b, dim3(R), 256, 0, (const double*)KMc, Lmid, R, RP, ozBB, ozFr + kOzN, oz_bad_ptr(1),
               (const LmDeviceState*)st, (const DevFlags*)fl, gate);
        const int nch = std::max(1, grid / ob.nb);
        const OzOut oo{(const double*)A1c, nullptr, RP, nch, (Cloc + nch - 1) / nch, nullptr, ozBp};
        launch(k_oz_pass<1>, dim3((unsigned)(ob.nb * nch)), kOzThreads, kOzSmem, (const uint8_t*)ozYB,
               (const int*)ozFrowB, (const uint8_t*)ozBB, (const int*)(ozFr + kOzN), ob, oo, (const LmDeviceState*)st,
               (const DevFlags*)fl, go);
        ph_end();
        launch(k_oz_note_fallback, 1, 1, 0, fl, (const LmDeviceState*)st, gf);
        reds[nred++] = Red{(const T*)ozBp, ob.nb, go};
        reds[nred++] = Red{(const T*)bpart, pass_b_fp64(F, gf), gf};
      }
    }
    if (!oz) {
      reds[nred++] = Red{(const T*)bpart, pass_b_fp64(F, gate), gate};
      ph_end();
    }
    // M_N rows of this slab from the partial sums
    auto mn_rows = [&](T* dst, int64_t ldm) {
      for (int i = 0; i < nred; ++i)
        launch(k_pass_b_reduce<T>, nblocks(Cloc * R, 256), 256, 0, reds[i].src, Cloc, reds[i].nparts, R, RP, ldm, dst,
               (const LmDeviceState*)st, (const DevFlags*)fl, reds[i].gate);
    };
    if (!comm) {
      mn_rows(Mout + offs[N - 1], IN);
    } else {
      CPF_CUDA_CHECK(cudaMemsetAsync(pb_out, 0, sizeof(T) * Cpad * R, ls));
      if (Cloc > 0) mn_rows(pb_out, Cpad);
      const size_t cnt = (size_t)Cpad * R * (sizeof(T) / sizeof(double));
      comm->allgather((const double*)pb_out, (double*)pb_all, cnt, ls);
      // pb_all[rank][c + Cpad r] -> Mout_N[(rank*Cpad + c) + IN r]
      for (int q = 0; q < world; ++q) {
        const int64_t lo = std::min<int64_t>(IN, (int64_t)q * Cpad);
        const int64_t cnt_rows = std::min<int64_t>(IN, lo + Cpad) - lo;
        if (cnt_rows <= 0) continue;
        launch(k_copy2d<T>, nblocks(cnt_rows * R, 256), 256, 0, (const T*)(pb_all + (size_t)q * Cpad * R), Cpad,
               Mout + offs[N - 1] + lo, IN, cnt_rows, (int64_t)R, (const LmDeviceState*)st, (const DevFlags*)fl, gate);
      }
    }
  }

  // fp64 pass B (DMMA / staged DFMA / plain) -> bpart; returns the number of partials per row
  int pass_b_fp64(const T* F, int gate) {
    if (Cloc <= 0) return 1;
    if constexpr (sizeof(T) == 8) {
      if (use_dmma) {
        const LmDeviceState* cst = st;
        const DevFlags* cfl = fl;
        if (N == 3)
          launch(k_conj_rowmajor<T>, nblocks(Lmid * db.WS, 256), 256, 0, (const T*)(F + offs[1]), Lmid, (int64_t)0, Lmid,
                 R, db.WS, (T*)KMd, cst, cfl, gate, 1);
        else
          launch(k_krmid<T>, nblocks(Lmid * db.WS, 256), 256, 0, F, mg, Lmid, R, db.WS, (T*)KMd, cst, cfl, gate, 1);
        dispatch_nt([&](auto ntc) {
          constexpr int NTc = decltype(ntc)::value;
          if (ls != s && persistent_b) {
            // overlapped with the next LU: persistent grid that leaves SMs for the panel cluster
            const int64_t items = (int64_t)db.tiles * Cloc * db_chunks;
            const int ctas = (int)std::min<int64_t>(items, std::max(1, nsm_ - kLuReserveSms));
            launch(k_pass_b_dmma_pers<NTc, kDmmaCK>, dim3(ctas), dim3(kConsumers + 32), db_smem, (const double*)Y, db,
                   (const double*)KMd, (const double*)A1c, RP, R, (int)Cloc, db_chunks, (double*)bpart, cst, cfl, gate);
          } else {
            launch(k_pass_dmma<NTc, 1, kDmmaCK>, dim3(db.tiles, (unsigned)Cloc, db_chunks), dim3(kConsumers + 32), db_smem,
                   (const double*)Y, db, (const double*)KMd, (const double*)A1c, (const double*)KMc, RP, R, (double*)zpart,
                   (double*)bpart, cst, cfl, gate);
          }
        });
        return db_chunks * db.tiles;
      }
    }
    if (use_v2) {
      dispatch_rp([&](auto rpc) {
        constexpr int RPc = decltype(rpc)::value;
        if (rpt == 2) {
          if constexpr (sizeof(T) == 8)
            launch(k_pass_b2<T, RPc, 2>, dim3((unsigned)Cloc, gb_chunks, gb.tiles), dim3(kConsumers + 32), gb_smem, Y, gb,
                   (const T*)A1c, (const T*)KMc, bpart, (const LmDeviceState*)st, (const DevFlags*)fl, gate);
        } else {
          launch(k_pass_b2<T, RPc, 1>, dim3((unsigned)Cloc, gb_chunks, gb.tiles), dim3(kConsumers + 32), gb_smem, Y, gb,
                 (const T*)A1c, (const T*)KMc, bpart, (const LmDeviceState*)st, (const DevFlags*)fl, gate);
        }
      });
      return gb_chunks * gb.tiles;
    }
    dispatch_rp([&](auto rpc) {
      constexpr int RPc = decltype(rpc)::value;
      const size_t smem = sizeof(T) * RPc * ((pb_threads + 31) / 32);
      launch(k_pass_b<T, RPc>, dim3((unsigned)Cloc, pb_chunks, pb_tiles), dim3(pb_threads), smem, Y, I1, Lmid,
             Cloc, (const T*)A1c, (const T*)KMc, pb_TI, pb_TM, pb_mper, bpart, (const LmDeviceState*)st, (const DevFlags*)fl, gate);
    });
    return pb_chunks * pb_tiles;
  }

  // ||Y - X(F)||^2 computed directly (guard band, preamble, relative_error API) -> *out (device)
  void direct_resid(const T* F, double* out, int gate) {
    const LmDeviceState* cst = st;
    const DevFlags* cfl = fl;
    launch(k_conj_rowmajor<T>, nblocks(I1 * RP, 256), 256, 0, F + offs[0], I1, (int64_t)0, I1, R, RP, A1r, cst, cfl, gate, 0);
    if (N == 3)
      launch(k_conj_rowmajor<T>, nblocks(Lmid * RP, 256), 256, 0, F + offs[1], Lmid, (int64_t)0, Lmid, R, RP, KMr, cst,
             cfl, gate, 0);
    else
      launch(k_krmid<T>, nblocks(Lmid * RP, 256), 256, 0, F, mg, Lmid, R, RP, KMr, cst, cfl, gate, 0);
    if (Cloc > 0) {
      launch(k_conj_rowmajor<T>, nblocks(Cloc * RP, 256), 256, 0, F + offs[N - 1], Cloc, slab_lo, IN, R, RP, WNr, cst,
             cfl, gate, 0);
      const int nb = (int)std::min<int64_t>(1024, std::max<int64_t>(1, nblocks(Lrows, 256)));
      dispatch_rp([&](auto rpc) {
        constexpr int RPc = decltype(rpc)::value;
        launch(k_direct_resid<T, RPc>, nb, 256, sizeof(T) * kPassCK * RPc, Y, I1, Lmid, Cloc, (const T*)WNr,
               (const T*)A1r, (const T*)KMr, red, cst, cfl, gate);
      });
      launch(k_sum_partials, 1, 1024, 0, (const double*)red, nb, out, cst, cfl, gate);
    } else {
      launch(k_axpby<double>, 1, 1, 0, (const double*)out, 0.0, (const double*)nullptr, 0.0, out, (int64_t)1, cst, cfl,
             gate);
    }
    if (comm) comm->allreduce_sum(out, 1, s);
  }

  // ------------------------------------------------------------------------------------------
  // building blocks
  // ------------------------------------------------------------------------------------------
  void cross_gram(const T* X, const T* Yv, T* out, int gate) {
    launch(k_cross_gram<T>, dim3(R * R, N), 128, 0, X, Yv, md, out, (const LmDeviceState*)st, (const DevFlags*)fl, gate);
  }
  void cache_from_grams(const T* C, int gate) {
    launch(k_hadamards<T>, nblocks(R * R, 128), 128, 0, C, N, R, Gx, Gp, Gf, (const LmDeviceState*)st,
           (const DevFlags*)fl, gate);
    launch(k_kernel_flag<T>, 1, 256, 0, (const T*)Gp, N, R, st, (const DevFlags*)fl, gate, kinv_ok);
  }
  void tall(const TallArgs& a, int gate) {
    int64_t maxrows = 0;
    for (int n = 0; n < N; ++n) maxrows = std::max(maxrows, dims[n] * R);
    launch(k_tall<T>, dim3(nblocks(maxrows, 128), N), 128, 2 * R * R * sizeof(T), a, md, (const LmDeviceState*)st,
           (const DevFlags*)fl, gate);
  }
  void axpby(const T* x, double al, const T* y, double be, T* out, int gate) {
    launch(k_axpby<T>, nblocks(RT, 256), 256, 0, x, al, y, be, out, RT, (const LmDeviceState*)st, (const DevFlags*)fl,
           gate);
  }
  void small(int op, const T* P0, const T* P1, T* out, int gate) {
    launch(k_small<T>, N, 128, 2 * R * R * sizeof(T), op, P0, P1, (const T*)Gx, (const T*)Gti, (const T*)Gp, N, R, out,
           (const LmDeviceState*)st, (const DevFlags*)fl, gate);
  }
  // gradient G = M - A Gamma^T (solver.py:251-256)
  void gradient(int gate) {
    TallArgs a{};
    a.X1 = A; a.S1 = Gx; a.t1 = 1; a.s1stride = (int64_t)R * R;
    a.X4 = M; a.coef4 = 1.0; a.neg1 = 1;
    a.out = G;
    tall(a, gate);
  }
  void normalize(const T* X, T* out, int gate, int mode) {
    launch(k_colnorms<T>, dim3(R, N), 256, 0, X, md, norms, (const LmDeviceState*)st, (const DevFlags*)fl, gate);
    launch(k_normalize<T>, R, 256, 0, X, md, (const double*)norms, out, st, (const DevFlags*)fl, gate, mode);
  }

  // ---- LU of Phi and the B-application
  // trailing update of panel (k0, kb) restricted to columns [c0, c1): U12 there, then A22 -= L21 U12
  void lu_update_cols(int k0, int kb, int c0, int c1, const T* invl, cudaStream_t strm, int gr) {
    if (c1 <= c0) return;
    const int w = c1 - c0, rows = nB - k0 - kb;
    k_u12<T, kLuMaxKB><<<nblocks(w, 64), 256, 0, strm>>>(Phi, c1, nB, k0, kb, invl, (const LmDeviceState*)st, gr, c0);
    ++nlaunch;
    CPF_CUDA_CHECK(cudaGetLastError());
    if (rows <= 0) return;
    if constexpr (sizeof(T) == 8)
      k_gemm_dmma<<<dim3(nblocks(rows, 64), nblocks(w, 64)), 128, 0, strm>>>(Phi, nB, k0 + kb, c0, k0, rows, w, kb,
                                                                            (const LmDeviceState*)st, gr);
    else
      k_gemm_sub<T><<<dim3(nblocks(rows, 64), nblocks(w, 64)), 256, 0, strm>>>(Phi, nB, k0 + kb, c0, k0, rows, w, kb,
                                                                              (const LmDeviceState*)st, gr);
    ++nlaunch;
    CPF_CUDA_CHECK(cudaGetLastError());
  }
  void lu_gather(int slot, int ca0, int ca1, int cb0, int cb1, int do_perm, cudaStream_t strm, int gr) {
    const int cols = std::max(0, ca1 - ca0) + std::max(0, cb1 - cb0);
    const int cb = 256 / (2 * kLuMaxKB);
    int* g = gring + slot * (4 * kLuMaxKB + 4);
    k_row_gather2<T><<<std::max(1u, nblocks(cols, cb)), 256, 256 * sizeof(T), strm>>>(
        Phi, nB, g, g + 4 * kLuMaxKB, lu.perm, ca0, ca1, cb0, cb1, do_perm, (const LmDeviceState*)st, gr);
    ++nlaunch;
    CPF_CUDA_CHECK(cudaGetLastError());
  }

  void lu_factor(int gate_running, bool with_inverse = false) {
    NvtxRange nvtx_("cpf.lu");
    ph_begin(kPhLU);
    tri_in_lu = false;
    if (lp_cfg) {
      lu_factor_lp(gate_running);
      if (!spec_capture) launch(k_lu_info_to_err, 1, 1, 0, (const int*)lu.info, st);
      ph_end();
      return;
    }
    launch(k_lu_init, nblocks(nB, 256), 256, 0, lu.perm, nB, lu.info, (const LmDeviceState*)st,
           gate_running == 3 ? lu.latch : (int*)nullptr, gate_running);
    if (lu3_rpt) {
      // Look-ahead right-looking LU.  Panel k+1's columns are the "next block" of step k: the
      // panel kernel itself applies step k's interchange and update to them while loading
      // (PanelPrev, lu3.cuh), so consecutive panels follow each other on stream s with no
      // kernels in between.  Stream s2 applies panel k to everything else (left columns' swaps,
      // perm, columns >= k0 + 2 KB) concurrently with panel k+1.  Gather lists and inv(L11) are
      // double-buffered across steps; panel k waits for s2's step k-2 (which updated its block
      // and last read the slot panel k overwrites).
      const int KB = kLuMaxKB;
      const int np = (nB + KB - 1) / KB;
      CPF_CUDA_CHECK(cudaEventRecord(evJ, s));
      CPF_CUDA_CHECK(cudaStreamWaitEvent(s2, evJ, 0));
      for (int k = 0; k < np; ++k) {
        const int k0 = k * KB, kb = std::min(KB, nB - k0), m = nB - k0;
        const int slot = k & 1;
        LuWork wk = lu;
        wk.gather = gring + slot * (4 * KB + 4);
        wk.gcount = wk.gather + 4 * KB;
        T* invl = invL + (size_t)slot * KB * KB;
        PanelPrev<T> pv{-1, 0, nullptr, nullptr, nullptr};
        if (k > 0 && lu_fuse) {
          const int ps = slot ^ 1;
          pv.kp0 = k0 - KB;
          pv.kbp = KB;
          pv.gather = gring + ps * (4 * KB + 4);
          pv.gcount = pv.gather + 4 * KB;
          pv.invL = invL + (size_t)ps * KB * KB;
        }
        if (k >= 2 && lu_fuse) CPF_CUDA_CHECK(cudaStreamWaitEvent(s, evB2[slot], 0));
        const int cl = (m + lu3_thr * lu3_rpt - 1) / (lu3_thr * lu3_rpt);
        if (use_lu4) launch_panel4(k0, kb, (m + kLu4Rpt * kLu4Thr - 1) / (kLu4Rpt * kLu4Thr), gate_running, wk, invl, pv);
        else if (lu3_thr == 128) launch_panel3<1, 128>(k0, kb, cl, gate_running, wk, invl, pv);
        else if constexpr (sizeof(T) == 8) launch_panel3<2, 256>(k0, kb, cl, gate_running, wk, invl, pv);
        else launch_panel3<1, 256>(k0, kb, cl, gate_running, wk, invl, pv);
        CPF_CUDA_CHECK(cudaEventRecord(evP, s));
        const int nb0 = k0 + kb, nb1 = std::min(nB, k0 + 2 * kb);
        if (!lu_fuse) {
          // unfused: the next block's interchange + update as kernels on s, after s2's step k-1
          if (k > 0) CPF_CUDA_CHECK(cudaStreamWaitEvent(s, evB, 0));
          lu_gather(slot, nb0, nb1, 0, 0, 0, s, gate_running);
          lu_update_cols(k0, kb, nb0, nb1, invl, s, gate_running);
        }
        // s2: left columns + the rest + perm, after panel k
        CPF_CUDA_CHECK(cudaStreamWaitEvent(s2, evP, 0));
        lu_gather(slot, 0, k0, nb1, nB, 1, s2, gate_running);
        lu_update_cols(k0, kb, nb1, nB, invl, s2, gate_running);
        CPF_CUDA_CHECK(cudaEventRecord(evB2[slot], s2));
        CPF_CUDA_CHECK(cudaEventRecord(evB, s2));
        if (with_inverse && tri_prog) {
          // s2's step k finalised the leading 32 (k + 1) rows/columns of L and U: the merges of the
          // triangular inverse that live inside it run on s4, beside the remaining panels
          CPF_CUDA_CHECK(cudaStreamWaitEvent(s4, evB, 0));
          tri_progress(k, np, gate_running);
        }
      }
      CPF_CUDA_CHECK(cudaStreamWaitEvent(s, evB, 0));
      if (with_inverse && tri_prog) {
        CPF_CUDA_CHECK(cudaEventRecord(evT2, s4));
        CPF_CUDA_CHECK(cudaStreamWaitEvent(s, evT2, 0));
        tri_in_lu = true;
      }
      if (!spec_capture) launch(k_lu_info_to_err, 1, 1, 0, (const int*)lu.info, st);
      ph_end();
      return;
    }
    const int kbmax = lu_kb;
    for (int k0 = 0; k0 < nB; k0 += kbmax) {
      const int kb = std::min(kbmax, nB - k0);
      const int m = nB - k0;
      {
        int cl = lu_cl;
        const int rpc = (m + cl - 1) / cl;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cl);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = panel_smem_bytes<T>(rpc, kb, cl);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cl;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CPF_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_panel_lu<T>, Phi, nB, nB, k0, kb, rpc, lu,
                                          (const LmDeviceState*)st, gate_running));
        ++nlaunch;
      }
      {
        const int cb = 256 / (2 * kLuMaxKB);
        const int ncols = nB - kb;
        launch(k_row_gather<T>, std::max(1u, nblocks(ncols, cb)), 256, 256 * sizeof(T), Phi, nB, nB, k0, kb, lu,
               (const LmDeviceState*)st, gate_running);
      }
      const int rest = nB - k0 - kb;
      if (rest > 0) {
        launch(k_trsm_llnu<T, kLuMaxKB>, nblocks(rest, 64), 64, 0, Phi, nB, nB, k0, kb, (const LmDeviceState*)st,
               gate_running);
        launch(k_gemm_sub<T>, dim3(nblocks(rest, 64), nblocks(rest, 64)), 256, 0, Phi, nB, k0 + kb, k0 + kb, k0,
               rest, rest, kb, (const LmDeviceState*)st, gate_running);
      }
    }
    launch(k_lu_info_to_err, 1, 1, 0, (const int*)lu.info, st);
    ph_end();
  }
  // f = B w  (flm-b: Phi^{-1} w; flm-a: K Phi^{-1} w)
  // inv(L), inv(U) of the factored Phi (tri_inv.cuh), packed like the factors
  // split-K factor of a triangular-inverse level (levels with few output tiles and long K)
  int tri_split(int sz) const {
    int k = kTriSplit;
    if (const char* e = knob("CPF_TRI_SPLIT")) k = std::max(1, std::min(kTriSplit, atoi(e)));
    // not in the pair form of the band 512 < n_B <= 1024 (config 2: its parity margin prefers
    // sequential sums, see tri_rows; 472 it/s either way there)
    return (sz >= 256 && (nB > 1024 || nB <= 512)) ? k : 1;
  }
  static constexpr int kTriSplit = 4;
  T* TriPart = nullptr;   // split-K partials: kTriSplit x nB x nB
  T* TriPartS = nullptr;  // the speculative branch's
  // Block step k of the inverse (tri_inv.cuh k_tri_row) on stream strm: the diagonal inverse of
  // block k, the long products against the leading inverse (split-K with a fixed-order reduce from
  // 256 leading rows up), then the 32-deep products with the diagonal inverses.  Inside the
  // look-ahead LU it is launched on s4 right after s2's step k, which finalised blocks 0..k of L
  // and U -- only the last block's step is left when the factorisation ends.
  void tri_row_product(int r0, int bs, int base, int tstep, int gate_running, cudaStream_t strm) {
    const LmDeviceState* cst = st;
    const int lead = r0 - base;
    if (lead <= 0) return;
    const int ks = tri_split(lead);
    const unsigned ty = (unsigned)((bs + 63) / 64);
    T* part = ks > 1 ? TriPart : (T*)nullptr;
    k_tri_row<T, 0><<<dim3((lead + 63) / 64, ty, 2 * ks), 256, 0, strm>>>((const T*)Phi, PhiInv, TriTmp, nB, r0, bs, base, cst,
                                                                         gate_running, ks, part, tstep);
    ++nlaunch;
    if (ks > 1) {
      const dim3 rgrid(std::max(1, std::min(64, (int)nblocks((int64_t)lead * bs, 256))), 2);
      k_tri_row_reduce<T><<<rgrid, 256, 0, strm>>>(TriTmp, (const T*)TriPart, ks, nB, r0, bs, base, cst, gate_running, tstep);
      ++nlaunch;
    }
    k_tri_row<T, 1><<<dim3((lead + 63) / 64, ty, 2), 256, 0, strm>>>((const T*)Phi, PhiInv, TriTmp, nB, r0, bs, base, cst,
                                                                    gate_running, 1, (T*)nullptr, tstep);
    ++nlaunch;
  }
  // rows per group of the two-level schedule (32: every block is its own group).  Groups of 128
  // make the long products four times rarer; measured at config 4 they still lose to the pair form
  // (182 vs 188 it/s), so the knob only serves experiments and tests
  int tri_group() const {
    if (const char* e = knob("CPF_TRI_GROUP")) return std::max(32, atoi(e) / 32 * 32);
    return 32;
  }
  void tri_row_step(int k, int gate_running, cudaStream_t strm) {
    const LmDeviceState* cst = st;
    const int np = (nB + 31) / 32;
    const int r0 = k * 32, bs = std::min(32, nB - r0);
    const int cap = tri_cap(), G = tri_group();
    const int base = (r0 / cap) * cap;      // start of the inverse this block belongs to
    const int g0 = (r0 / G) * G;            // start of its group
    k_tri_inv_diag<T><<<1, 64, 0, strm>>>((const T*)Phi, nB, PhiInv, cst, gate_running, k, k);
    ++nlaunch;
    tri_row_product(r0, bs, g0, k, gate_running, strm);  // inside the group
    const int gend = std::min({nB, g0 + G, base + cap});
    if (r0 + bs >= gend || k == np - 1) tri_row_product(g0, r0 + bs - g0, base, k, gate_running, strm);
    CPF_CUDA_CHECK(cudaGetLastError());
  }
  // which form: rows for the small systems, pairs above (tri_inv.cuh header)
  bool tri_rows() const {
    if (const char* e = knob("CPF_TRI_ROWS")) return e[0] == '1';
    // up to n_B = 512.  Between 512 and 1024 (config 2: 900) the row form needs split-K to keep up
    // with the panels, and split-K sums move the ill-conditioned config-2 trajectory away from the
    // reference's (final factors 1.9e-9 with it, 5e-10 without but 423 it/s); the pair form without
    // split-K gives 6.6e-10 at 472 it/s
    return nB <= 512;
  }
  void tri_progress(int k, int np, int gate_running) {
    if (tri_rows()) tri_row_step(k, gate_running, s4);
    else tri_pair_progress(k, np, gate_running);
  }
  // Pair form (n_B > 1024), progressive: after the LU's step k the blocks 0..k of L and U are final.
  // Launch on s4 the diagonal inverse of block k and, level by level, every merge whose pair ends
  // at block k (the last block closes the ragged pairs).  Same kernels and operation order per
  // output element as the batched launches of tri_invert -> bitwise identical inverse.
  void tri_pair_progress(int k, int np, int gate_running) {
    const LmDeviceState* cst = st;
    k_tri_inv_diag<T><<<1, 64, 0, s4>>>((const T*)Phi, nB, PhiInv, cst, gate_running, k, k);
    ++nlaunch;
    const bool last = k == np - 1;
    for (int sz = 32; sz < tri_cap(); sz *= 2) {
      const int w = sz / 32;  // blocks per half
      if (!last && (k + 1) % (2 * w) != 0) break;  // higher levels end at the same block or later
      const int pair = k / (2 * w);
      if ((2 * pair + 1) * sz >= nB) continue;  // single (ragged) half: nothing to merge
      const int ks = tri_split(sz);
      const dim3 grid((sz + 63) / 64, (sz + 63) / 64, 2 * ks);
      const dim3 rgrid(std::max(1, std::min(256, (int)nblocks((int64_t)sz * sz, 256))), 2);
      T* part = ks > 1 ? TriPart : (T*)nullptr;
      k_tri_level<T, 0><<<grid, 256, 0, s4>>>((const T*)Phi, PhiInv, TriTmp, nB, sz, cst, gate_running, ks, part, pair, k);
      ++nlaunch;
      if (ks > 1) {
        k_tri_reduce<T, 0><<<rgrid, 256, 0, s4>>>(PhiInv, TriTmp, (const T*)TriPart, ks, nB, sz, cst, gate_running, pair, k);
        ++nlaunch;
      }
      k_tri_level<T, 1><<<grid, 256, 0, s4>>>((const T*)Phi, PhiInv, TriTmp, nB, sz, cst, gate_running, ks, part, pair, k);
      ++nlaunch;
      if (ks > 1) {
        k_tri_reduce<T, 1><<<rgrid, 256, 0, s4>>>(PhiInv, TriTmp, (const T*)TriPart, ks, nB, sz, cst, gate_running, pair, k);
        ++nlaunch;
      }
    }
    CPF_CUDA_CHECK(cudaGetLastError());
  }
  void tri_invert(int gate_running) {
    NvtxRange nvtx_("cpf.tri_inverse");
    ph_begin(kPhLU);
    if (tri_rows()) {
      const int np = (nB + 31) / 32;
      for (int k = 0; k < np; ++k) tri_row_step(k, gate_running, ls);
      ph_end();
      return;
    }
    const int nblk = (nB + 31) / 32;
    launch(k_tri_inv_diag<T>, nblk, 64, 0, (const T*)Phi, nB, PhiInv, (const LmDeviceState*)st, gate_running, 0, 200);
    for (int sz = 32; sz < tri_cap(); sz *= 2) {
      const int npairs = (nB + 2 * sz - 1) / (2 * sz);
      const int ks = tri_split(sz);
      const dim3 grid((sz + 63) / 64, (sz + 63) / 64, 2 * npairs * ks);
      const dim3 rgrid(std::max(1, std::min(256, (int)nblocks((int64_t)sz * sz, 256))), 2 * npairs);
      launch(k_tri_level<T, 0>, grid, 256, 0, (const T*)Phi, PhiInv, TriTmp, nB, sz, (const LmDeviceState*)st,
             gate_running, ks, ks > 1 ? TriPart : (T*)nullptr, 0, 200);
      if (ks > 1)
        launch(k_tri_reduce<T, 0>, rgrid, 256, 0, PhiInv, TriTmp, (const T*)TriPart, ks, nB, sz, (const LmDeviceState*)st,
               gate_running, 0, 200);
      launch(k_tri_level<T, 1>, grid, 256, 0, (const T*)Phi, PhiInv, TriTmp, nB, sz, (const LmDeviceState*)st,
             gate_running, ks, ks > 1 ? TriPart : (T*)nullptr, 0, 200);
      if (ks > 1)
        launch(k_tri_reduce<T, 1>, rgrid, 256, 0, PhiInv, TriTmp, (const T*)TriPart, ks, nB, sz, (const LmDeviceState*)st,
               gate_running, 0, 200);
    }
    ph_end();
  }


  void apply_b(const T* w, T* f, int gate_running) {
    ph_begin(kPhSolve);
    launch(k_perm_gather<T>, nblocks(nB, 256), 256, 0, w, (const int*)lu.perm, nB, xvec, (const LmDeviceState*)st,
           gate_running);
    if (use_inv) {
      const dim3 grid((nB + kTmvRows - 1) / kTmvRows, (nB + kTmvCols - 1) / kTmvCols);
      const int nsl = (int)grid.y;
      launch(k_tri_mv<T, true>, grid, 256, 0, (const T*)PhiInv, nB, (const T*)xvec, tmv_part, (const LmDeviceState*)st,
             gate_running);
      launch(k_tri_mv_sum<T, true>, nblocks(nB, 256), 256, 0, (const T*)tmv_part, nsl, nB, (const T*)xvec, yvec,
             (const LmDeviceState*)st, gate_running);
      launch(k_tri_mv<T, false>, grid, 256, 0, (const T*)PhiInv, nB, (const T*)yvec, tmv_part, (const LmDeviceState*)st,
             gate_running);
      launch(k_tri_mv_sum<T, false>, nblocks(nB, 256), 256, 0, (const T*)tmv_part, nsl, nB, (const T*)yvec, xvec,
             (const LmDeviceState*)st, gate_running);
      launch(k_apply_k<T>, nblocks(nB, 256), 256, 0, (const T*)xvec, N, R, (const T*)Gp, f, (const LmDeviceState*)st,
             gate_running);
      ph_end();
      return;
    }
    if (use_blkinv) {
      const LmDeviceState* cst = st;
      const int DB = blk_db, nb = (nB + DB - 1) / DB;
      auto step = [&](auto lower, int b) {
        constexpr bool LOWER = decltype(lower)::value;
        const int r0 = b * DB, r1 = std::min(nB, r0 + DB);
        const int c0 = LOWER ? 0 : r1, c1 = LOWER ? r0 : nB;
        const unsigned rt = nblocks(r1 - r0, kTmvRows), rs = nblocks(r1 - r0, 256);
        if (c1 > c0) {  // right-hand side minus the off-diagonal block row times the solved part
          const unsigned nsl = nblocks(c1 - c0, kTmvCols);
          launch(k_blk_mv<T, 0>, dim3(rt, nsl), 256, 0, (const T*)Phi, nB, r0, r1, c0, c1, (const T*)xvec, tmv_part, cst,
                 gate_running);
          launch(k_blk_sum<T, 0>, rs, 256, 0, (const T*)tmv_part, (int)nsl, nB, r0, r1, xvec, cst, gate_running);
        }
        const unsigned nsd = nblocks(r1 - r0, kTmvCols);
        launch(k_blk_mv<T, LOWER ? 1 : 2>, dim3(rt, nsd), 256, 0, (const T*)PhiInv, nB, r0, r1, r0, r1, (const T*)xvec,
               tmv_part, cst, gate_running);
        launch(k_blk_sum<T, LOWER ? 1 : 2>, rs, 256, 0, (const T*)tmv_part, (int)nsd, nB, r0, r1, xvec, cst, gate_running);
      };
      for (int b = 0; b < nb; ++b) step(std::true_type{}, b);
      for (int b = nb - 1; b >= 0; --b) step(std::false_type{}, b);
      launch(k_apply_k<T>, nblocks(nB, 256), 256, 0, (const T*)xvec, N, R, (const T*)Gp, f, cst, gate_running);
      ph_end();
      return;
    }
    const int nblk = (nB + 31) / 32;
    // ready flags are cleared in-stream (graph-replay safe: no host-side epoch)
    CPF_CUDA_CHECK(cudaMemsetAsync(lu.ticket, 0, sizeof(int) * 2, s));
    CPF_CUDA_CHECK(cudaMemsetAsync(lu.ready, 0, sizeof(int) * 2 * nblk, s));
    launch(k_trsv<T, true>, nblk, 128, 0, (const T*)Phi, nB, nB, xvec, lu.ticket, lu.ready, 1,
           (const LmDeviceState*)st, gate_running);
    launch(k_trsv<T, false>, nblk, 128, 0, (const T*)Phi, nB, nB, xvec, lu.ticket + 1, lu.ready + nblk, 1,
           (const LmDeviceState*)st, gate_running);
    launch(k_apply_k<T>, nblocks(nB, 256), 256, 0, (const T*)xvec, N, R, (const T*)Gp, f, (const LmDeviceState*)st,
           gate_running);
    ph_end();
  }

  // fLM candidate at (A, cache, M, G) with the state's mu -> Cand  (solver.py:189-226)
  // Damped Gamma inverses for the state's mu, Phi and its LU: everything of the step that does
  // not depend on Y or the MTTKRPs (it only needs the Grams and mu)
  // mode 0: the state's mu; 1: speculative rejection branch (buffers swapped in, mu * growth,
  // errors deferred); 2: the fork's core system when a rejection branch was speculated (skipped
  // after a rejection)
  void prepare_core(int gate, int mode = 0) {
    NvtxRange nvtx_("cpf.core_system (phi + lu + inverse)");
    const int gr = mode == 2 ? 2 : mode == 1 ? 3 : (gate == kRunning ? 1 : 0);
    if (mode == 1) {  // mu * growth snapshot: k_spec_begin on the main stream (iteration())
      launch(k_damped_inverses<T>, 2 * N, 128, 2 * R * R * sizeof(T), (const T*)Gx, N, R, Gti, Gi, st,
             (const DevFlags*)fl, gate, (const int*)nullptr, (const double*)(dscal + 8), spec_sing);
    } else {
      launch(k_damped_inverses<T>, 2 * N, 128, 2 * R * R * sizeof(T), (const T*)Gx, N, R, Gti, Gi, st,
             (const DevFlags*)fl, mode == 2 ? (int)kOnCoreNeeded : gate, (const int*)kinv_ok, (const double*)nullptr,
             (int*)nullptr);
    }
    launch(k_phi_assemble<T>, nblocks((int64_t)nB * nB, 256), 256, 0, Phi, N, R, (const T*)Cg, (const T*)Gi,
           (const T*)Gp, (const T*)Gf, (const LmDeviceState*)st, gr);
    if (test_singular) launch(k_test_zero_col<T>, 1, 256, 0, Phi, nB, (const LmDeviceState*)st, mode == 1 ? 2 : 1);
    mark(5);
    lu_factor(gr, use_inv || use_blkinv);
    mark(6);
    if ((use_inv || use_blkinv) && !tri_in_lu) tri_invert(gr);
    mark(7);
  }

  void candidate(int refine_steps, int gate, bool core_ready = false) {
    NvtxRange nvtx_("cpf.candidate");
    const int gr = gate == kRunning ? 1 : 0;
    if (!core_ready) prepare_core(gate);
    // damped factors D = M Gti
    { TallArgs a{}; a.X1 = M; a.S1 = Gti; a.s1stride = (int64_t)R * R; a.out = D; tall(a, gate); }
    // w = vec(A^H D - C Gamma^T Gti)
    cross_gram(A, D, W1, gate);
    small(kOpW, W1, Cg, wvec, gate);
    apply_b(wvec, fvec, gr);
    // update: Cand = D + A (I - (F + Gamma^T) Gti)
    small(kOpE, fvec, nullptr, Sm, gate);
    { TallArgs a{}; a.X1 = A; a.S1 = Sm; a.s1stride = (int64_t)R * R; a.X4 = D; a.coef4 = 1.0; a.out = Cand; tall(a, gate); }
    if (refine_steps > 0) {
      axpby(Cand, 1.0, A, -1.0, V1, gate);  // delta
      for (int it = 0; it < refine_steps; ++it) {
        // (H + mu I) delta  (hessian.py:311-326)
        cross_gram(A, V1, W1, gate);
        small(kOpS, W1, nullptr, Sm, gate);
        {
          TallArgs a{};
          a.X1 = V1; a.S1 = Gx; a.t1 = 1; a.s1stride = (int64_t)R * R;
          a.X3 = V1; a.coef3_mu = 1;
          a.X2 = A; a.S2 = Sm; a.s2stride = (int64_t)R * R;
          a.out = V2;
          tall(a, gate);
        }
        axpby(G, 1.0, V2, -1.0, V3, gate);  // resid = g - Hd
        // (H + mu I)^{-1} resid  (hessian.py:329-348)
        { TallArgs a{}; a.X1 = V3; a.S1 = Gti; a.s1stride = (int64_t)R * R; a.out = V4; tall(a, gate); }
        cross_gram(A, V4, wvec, gate);
        apply_b(wvec, fvec, gr);
        small(kOpYG, fvec, nullptr, Sm, gate);
        { TallArgs a{}; a.X1 = A; a.S1 = Sm; a.s1stride = (int64_t)R * R; a.neg1 = 1; a.X4 = V4; a.coef4 = 1.0; a.out = V2; tall(a, gate); }
        axpby(V1, 1.0, V2, 1.0, V1, gate);  // delta += ...
      }
      axpby(A, 1.0, V1, 1.0, Cand, gate);  // model_from_vector(base + delta)
    }
  }

  // cache (Grams, Hadamards, K flag), MTTKRPs and gradient at the current factors A
  void build_cache_and_mttkrps(int gate) {
    cross_gram(A, A, Cg, gate);
    cache_from_grams(Cg, gate);
    pass_a(A, M, gate);
    pass_b(A, M, gate);
    gradient(gate);
  }

  double host_yx_from(const T* Mx, const T* F) {
    launch(k_redot<T>, 1, 1024, 0, F + offs[0], Mx + offs[0], I1 * R, 0, dscal + 0, (const LmDeviceState*)st,
           (const DevFlags*)fl, (int)kAlways);
    double v;
    CPF_CUDA_CHECK(cudaMemcpyAsync(&v, dscal + 0, sizeof(double), cudaMemcpyDeviceToHost, s));
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    return v;
  }

  double ynorm_sq() {
    const int nb = 1024;
    if (Jloc > 0) {
      launch(k_sumsq_partial<T>, nb, 256, 0, Y, Jloc, red);
      launch(k_sum_partials, 1, 1024, 0, (const double*)red, nb, dscal + 1, (const LmDeviceState*)nullptr, (const DevFlags*)nullptr, 0);
    } else {
      CPF_CUDA_CHECK(cudaMemsetAsync(dscal + 1, 0, sizeof(double), s));
    }
    if (comm) comm->allreduce_sum(dscal + 1, 1, s);
    double v;
    CPF_CUDA_CHECK(cudaMemcpyAsync(&v, dscal + 1, sizeof(double), cudaMemcpyDeviceToHost, s));
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    return v;
  }

  void require_ready() {
    if (!have_tensor) throw ApiError(CPF_E_STATE, "no tensor bound");
    if (!have_factors) throw ApiError(CPF_E_STATE, "no factors bound");
  }

  void reset_state(int variant, double mu, double tol, int max_iters) {
    std::memset(hst, 0, sizeof(LmDeviceState));
    hst->mu = mu;
    hst->growth = 2.0;
    hst->variant = variant;
    hst->tol = tol;
    hst->max_iters = max_iters;
    CPF_CUDA_CHECK(cudaMemcpyAsync(st, hst, sizeof(LmDeviceState), cudaMemcpyHostToDevice, s));
    CPF_CUDA_CHECK(cudaMemsetAsync(fl, 0, sizeof(DevFlags), s));
  }
  void pull_state() {
    CPF_CUDA_CHECK(cudaMemcpyAsync(hst, st, sizeof(LmDeviceState), cudaMemcpyDeviceToHost, s));
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
  }
  void fill_status(cpf_status* o) {
    if (!o) return;
    o->stopped = hst->stopped;
    o->err_code = hst->err_code;
    o->err_iter = hst->err_iter;
    o->iter = hst->iter;
    o->last_accepted = hst->accepted;
    o->err_column = 0;
    o->relerr = hst->err;
    o->mu = hst->mu;
    o->ynorm = hst->ynorm;
  }

  // ------------------------------------------------------------------------------------------
  // EngineBase
  // ------------------------------------------------------------------------------------------
  void slab(int64_t* lo, int64_t* hi) const override { *lo = slab_lo; *hi = slab_hi; }
  void* stream() override { return (void*)s; }

  void set_tensor(const void* p, int64_t n, int where) override {
    NvtxRange nvtx_("cpf.set_tensor (upload)");
    if (n != Jloc) throw ApiError(CPF_E_ARG, "tensor slab size mismatch: expected " + std::to_string(Jloc));
    CPF_CUDA_CHECK(cudaSetDevice(dev));
    if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }  // Y pointer is baked into the graph
    if (where == 1) {
      if (Yown) { big_free(Yown); Yown = nullptr; }
      Y = static_cast<const T*>(p);
    } else {
      if (!Yown) Yown = static_cast<T*>(big_alloc((size_t)std::max<int64_t>(Jloc, 1) * sizeof(T), false));
      if (upload_with_split(p)) {
        have_tensor = true;
        ysq_cached = -1.0;
        return;
      }
      if (Jloc > 0) CPF_CUDA_CHECK(cudaMemcpyAsync(Yown, p, Jloc * sizeof(T), cudaMemcpyHostToDevice, s));
      Y = Yown;
    }
    oz_split();
    have_tensor = true;
    ysq_cached = -1.0;
  }
  // CPTN file -> this rank's slab in device memory, double-buffered through pinned staging
  void load_cptn(const char* path, int64_t payload_off) override {
    NvtxRange nvtx_("cpf.load_cptn");
    CPF_CUDA_CHECK(cudaSetDevice(dev));
    if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) throw ApiError(CPF_E_ARG, std::string("cannot open ") + path);
    struct FdGuard { int fd; ~FdGuard() { ::close(fd); } } guard{fd};
    struct stat sb;
    if (fstat(fd, &sb) != 0) throw ApiError(CPF_E_ARG, std::string("cannot stat ") + path);
    const int64_t es = (int64_t)sizeof(T);
    const int64_t count = Lrows * IN;
    const int64_t have = ((int64_t)sb.st_size - payload_off) / es;
    if ((int64_t)sb.st_size < payload_off || have != count || ((int64_t)sb.st_size - payload_off) % es != 0)
      throw ApiError(CPF_E_FORMAT, "expected " + std::to_string(count) + " scalars, found " + std::to_string(have));
    posix_fadvise(fd, 0, 0, POSIX_FADV_SEQUENTIAL);
    if (!Yown) Yown = static_cast<T*>(big_alloc((size_t)std::max<int64_t>(Jloc, 1) * sizeof(T), false));
    const int64_t bytes = Jloc * es;
    const int64_t start = payload_off + slab_lo * Lrows * es;
    const int64_t chunk = std::min<int64_t>(bytes, (int64_t)64 << 20);
    void* stage[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    struct Staging {
      void** b; cudaEvent_t* e;
      ~Staging() { for (int i = 0; i < 2; ++i) { if (b[i]) cudaFreeHost(b[i]); if (e[i]) cudaEventDestroy(e[i]); } }
    } sg{stage, done};
    for (int i = 0; i < 2 && chunk > 0; ++i) {
      CPF_CUDA_CHECK(cudaMallocHost(&stage[i], (size_t)chunk));
      CPF_CUDA_CHECK(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
    int k = 0;
    for (int64_t off = 0; off < bytes; off += chunk, ++k) {
      const int b = k & 1;
      const int64_t n = std::min(chunk, bytes - off);
      if (k >= 2) CPF_CUDA_CHECK(cudaEventSynchronize(done[b]));  // staging buffer free again
      int64_t got = 0;
      while (got < n) {
        const ssize_t r = ::pread(fd, static_cast<char*>(stage[b]) + got, (size_t)(n - got), (off_t)(start + off + got));
        if (r <= 0) throw ApiError(CPF_E_FORMAT, std::string("short read in ") + path);
        got += r;
      }
      CPF_CUDA_CHECK(cudaMemcpyAsync(reinterpret_cast<char*>(Yown) + off, stage[b], (size_t)n, cudaMemcpyHostToDevice, s));
      CPF_CUDA_CHECK(cudaEventRecord(done[b], s));
    }
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    Y = Yown;
    oz_split();
    have_tensor = true;
    ysq_cached = -1.0;
  }
  void set_factors(const void* p) override {
    CPF_CUDA_CHECK(cudaMemcpyAsync(A, p, RT * sizeof(T), cudaMemcpyHostToDevice, s));
    have_factors = true;
    have_hist = false;
  }
  void get_factors(void* p) override {
    CPF_CUDA_CHECK(cudaMemcpyAsync(p, A, RT * sizeof(T), cudaMemcpyDeviceToHost, s));
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
  }

  void fit_begin(int variant, double tau, double tol, int max_iters, cpf_status* o) override {
    NvtxRange nvtx_("cpf.fit_begin (preamble)");
    require_ready();
    if (variant < 0 || variant > 2) throw ApiError(CPF_E_ARG, "unknown variant");
    reset_state(variant, 0.0, tol, max_iters);
    if (trace_cap < max_iters) {
      if (dtrace) CPF_CUDA_CHECK(cudaFreeAsync(dtrace, s));
      dtrace = dalloc<IterRecordDev>(std::max(max_iters, 1));
      trace_cap = max_iters;
    }
    // model = normalize_equal_energy(init)  (solver.py:321)
    normalize(A, A, kAlways, 0);
    pull_state();
    if (hst->err_code == kErrZeroColumn) throw ApiError(CPF_E_ZERODIV, "component has a zero-norm vector");
    // ||Y||; zero tensor -> ZeroDivisionError (solver.py:322-324)
    const double ysq = ynorm_sq();
    const double ynorm = std::sqrt(ysq);
    if (ynorm == 0.0) throw ApiError(CPF_E_ZERODIV, "cannot fit a zero tensor");
    // mu0 = tau * max(1, max Re diag C^(N)) of normalize_unit_modes(model) (solver.py:326-327, 229-235)
    std::vector<double> hn((size_t)N * R);
    launch(k_colnorms<T>, dim3(R, N), 256, 0, (const T*)A, md, norms, (const LmDeviceState*)st, (const DevFlags*)fl,
           (int)kAlways);
    CPF_CUDA_CHECK(cudaMemcpyAsync(hn.data(), norms, sizeof(double) * N * R, cudaMemcpyDeviceToHost, s));
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    double dmax = -INFINITY;
    for (int r = 0; r < R; ++r) {
      double sc = 1.0;
      for (int n = 0; n < N - 1; ++n) sc = sc * hn[(size_t)n * R + r];
      const double v = hn[(size_t)(N - 1) * R + r] * sc;
      dmax = std::max(dmax, v * v);
    }
    const double mu0 = tau * std::max(1.0, dmax);
    // cache, MTTKRPs, err (solver.py:329-332); error via ||Y||^2 - 2 Re<Y,X> + ||X||^2
    build_cache_and_mttkrps(kAlways);
    launch(k_xnorm2<T>, 1, 256, 0, (const T*)Cg, N, R, dscal + 2, (const LmDeviceState*)st, (const DevFlags*)fl,
           (int)kAlways);
    direct_resid(A, dscal + 5, kAlways);
    double res;
    CPF_CUDA_CHECK(cudaMemcpyAsync(&res, dscal + 5, sizeof(double), cudaMemcpyDeviceToHost, s));
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    const double err = std::sqrt(res) / ynorm;
    hst->err_direct = 1;
    hst->mu = mu0;
    hst->growth = 2.0;
    hst->err = err;
    hst->err_sq = (err * ynorm) * (err * ynorm);
    hst->ynorm = ynorm;
    hst->ynorm_sq = ysq;
    hst->variant = variant;
    hst->tol = tol;
    hst->max_iters = max_iters;
    hst->stopped = max_iters <= 0 ? kStopMaxIters : 0;
    // When one direct-residual pass (2 J R flops) costs < 5% of the iteration's LU ((2/3) n_B^3),
    // evaluate every trial fit directly from Y as well: removes the identity's ~eps/relerr^2
    // cancellation error at no measurable cost (config 1 regime).
    {
      const double cw = sizeof(T) == 16 ? 4.0 : 1.0;
      // global J, not Jloc * world: identical on every rank of a ragged split (the choice decides
      // which collectives the iteration issues)
      const double pass_flops = 2.0 * cw * (double)Lrows * IN * R;
      const double lu_flops = (2.0 / 3.0) * cw * (double)nB * nB * nB;
      hst->force_direct = pass_flops < 0.05 * lu_flops ? 1 : 0;
      if (const char* e = knob("CPF_FORCE_DIRECT")) hst->force_direct = (e[0] == '1');
    }
    hst->rej_grow = 0;
    hst->test_negdenom_iter = 0;
    if (const char* e = knob("CPF_TEST_NEGDENOM")) hst->test_negdenom_iter = atoi(e);  // test hook
    hst->test_singular_iter = 0;
    if (const char* e = knob("CPF_TEST_SINGULAR")) hst->test_singular_iter = atoi(e);  // test hook
    if (test_singular != (hst->test_singular_iter != 0) && gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }
    test_singular = hst->test_singular_iter != 0;
    // keep use_kinv computed by the cache kernels
    LmDeviceState tmp;
    CPF_CUDA_CHECK(cudaMemcpyAsync(&tmp, st, sizeof(tmp), cudaMemcpyDeviceToHost, s));
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    hst->use_kinv = tmp.use_kinv;
    CPF_CUDA_CHECK(cudaMemcpyAsync(st, hst, sizeof(LmDeviceState), cudaMemcpyHostToDevice, s));
    if (!rotated()) prepare_core(kRunning);  // else Phi(mu_0, cache_0) is factored by the first unit's fork
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    fill_status(o);
  }

  static constexpr int kStopMaxIters = 4;

  // One replay unit, in one of two orders.
  //   rotated (the FMA-pass configurations): fork -> step.  The unit starts at the fork that follows
  //     the previous decision (first iteration: only the core system) and ends with this
  //     iteration's decision and commit.  The step's rejection branch Phi(cache_t, mu_t * growth_t)
  //     -- known as soon as the previous decision is -- is launched BEFORE the fork, so it has
  //     the whole unit (fork + candidate + pass A): a rejection right after an accepted step no
  //     longer waits for most of the speculated factorisation, and a fit does not end with a
  //     fork nobody needs.
  //   classic (int8 passes, config 4): step -> fork, the branch beside candidate + pass A only.
  //     Measured there: two factorisations beside pass B share its 40 SMs (173 it/s), and with
  //     the branch after the fork the unit ends with the drain of an abandoned branch's ~250
  //     gated kernels, which the classic order hides inside the fork (163 vs 185 it/s).
  //   fork   accepted previous step: pass B (M_N of the new model) + gradient on s3, beside the
  //          core system Phi(mu_t, cache_t), its LU and inverse on s (independent of Y);
  //          after a rho <= 0 rejection nothing (the speculated system is copied in)
  //   step   candidate -> normalise -> pass A -> trial fit -> decide -> commit
  bool rotated() const {
    if (const char* e = knob("CPF_ROTATED")) return e[0] == '1';
    return !use_oz;
  }
  void spec_launch(int g) {
    // the previous step was rejected: its core system is the speculated one
    const int gp = kOnRejectPrev;
    launch(k_copy<T>, nblocks((int64_t)nB * nB, 256), 256, 0, (const T*)PhiInvS, PhiInv, (int64_t)nB * nB,
           (const LmDeviceState*)st, (const DevFlags*)fl, gp);
    launch(k_copy<int>, nblocks(nB, 256), 256, 0, (const int*)luS.perm, lu.perm, (int64_t)nB,
           (const LmDeviceState*)st, (const DevFlags*)fl, gp);
    launch(k_copy<T>, nblocks((int64_t)N * R * R, 256), 256, 0, (const T*)GtiS, Gti, (int64_t)N * R * R,
           (const LmDeviceState*)st, (const DevFlags*)fl, gp);
    launch(k_copy<T>, nblocks((int64_t)N * R * R, 256), 256, 0, (const T*)GiS, Gi, (int64_t)N * R * R,
           (const LmDeviceState*)st, (const DevFlags*)fl, gp);
    launch(k_spec_errors, 1, 1, 0, st, (const DevFlags*)fl, (const int*)spec_sing, (const int*)luS.info);
    // its mu is snapshotted on s (ordered before this iteration's k_decide), the branch itself only
    // reads dscal[8]
    launch(k_spec_begin, 1, 1, 0, st, dscal + 8, spec_sing);
    CPF_CUDA_CHECK(cudaEventRecord(evS0, s));
    CPF_CUDA_CHECK(cudaStreamWaitEvent(sS, evS0, 0));
    const bool pdl_prev = pdl_now;
    pdl_now = false;
    spec_capture = true;
    swap_spec();
    ls = s;
    prepare_core(g, 1);
    CPF_CUDA_CHECK(cudaEventRecord(evS1, s));
    swap_spec();
    ls = s;
    spec_capture = false;
    pdl_now = pdl_prev;
  }
  void fork_core(int g) {
    const int ga = kOnAccept;
    pdl_now = false;
    if (serial) {  // diagnostic (CPF_SERIAL=1): no overlap, phases time standalone
      pass_b(A, M, ga);
      gradient(ga);
      prepare_core(g, use_spec ? 2 : 0);
    } else {
      CPF_CUDA_CHECK(cudaEventRecord(evF, s));
      CPF_CUDA_CHECK(cudaStreamWaitEvent(s3, evF, 0));
      ls = s3;
      pass_b(A, M, ga);
      gradient(ga);
      ls = s;
      CPF_CUDA_CHECK(cudaEventRecord(evG, s3));
      prepare_core(g, use_spec ? 2 : 0);
      CPF_CUDA_CHECK(cudaStreamWaitEvent(s, evG, 0));
    }
    launch(k_clear_pending, 1, 1, 0, fl);
    pdl_now = true;
  }

  void iteration() {
    NvtxRange nvtx_("cpf.iteration (eager or captured)");
    const int g = kRunning;
    pdl_now = true;
    mark(0);
    if (rotated()) {
      if (use_spec) spec_launch(g);
      fork_core(g);
    } else if (use_spec) {
      spec_launch(g);
    }
    mark(1);
    candidate(2, g, /*core_ready=*/true);  // Phi(mu_t, cache_t): factored in the fork or speculated
    mark(2);
    // delta' = cand - model (solver.py:348)
    axpby(Cand, 1.0, A, -1.0, V1, g);
    // normalised candidate: trial fit and, if accepted, the new model (solver.py:362)
    normalize(Cand, Ac, g, 1);
    cross_gram(Ac, Ac, Ccg, g);
    launch(k_xnorm2<T>, 1, 256, 0, (const T*)Ccg, N, R, dscal + 2, (const LmDeviceState*)st, (const DevFlags*)fl, g);
    pass_a(Ac, Mc, g);
    launch(k_redot<T>, 1, 1024, 0, (const T*)(Ac + offs[0]), (const T*)(Mc + offs[0]), I1 * R, 0, dscal + 0,
           (const LmDeviceState*)st, (const DevFlags*)fl, g);
    launch(k_redot<T>, 1, 1024, 0, (const T*)V1, (const T*)G, RT, 1, dscal + 3, (const LmDeviceState*)st,
           (const DevFlags*)fl, g);
    launch(k_precheck, 1, 1, 0, (const LmDeviceState*)st, fl, (const double*)dscal);
    direct_resid(Ac, dscal + 4, kOnDirect);
    direct_resid(A, dscal + 5, kOnCurDirect);
    launch(k_decide, 1, 1, 0, st, fl, dtrace, (const double*)dscal);
    mark(3);
    // commit an accepted candidate (solver.py:361-367): model, cache, MTTKRPs; M_N and the gradient
    // follow in the next unit's fork
    const int ga = kOnAccept;
    launch(k_copy<T>, nblocks(RT, 256), 256, 0, (const T*)Ac, A, RT, (const LmDeviceState*)st, (const DevFlags*)fl, ga);
    launch(k_copy<T>, nblocks((int64_t)N * R * R, 256), 256, 0, (const T*)Ccg, Cg, (int64_t)N * R * R,
           (const LmDeviceState*)st, (const DevFlags*)fl, ga);
    cache_from_grams(Cg, ga);
    launch(k_copy<T>, nblocks(offs[N - 1], 256), 256, 0, (const T*)Mc, M, offs[N - 1], (const LmDeviceState*)st,
           (const DevFlags*)fl, ga);
    pdl_now = false;
    mark(4);
    if (!rotated()) fork_core(g);
    if (use_spec) CPF_CUDA_CHECK(cudaStreamWaitEvent(s, evS1, 0));
    mark(8);
  }

  void capture_iteration() {
    cudaGraph_t g = nullptr;
    const int64_t before = nlaunch;
    CPF_CUDA_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try {
      capturing = true;
      iteration();
      capturing = false;
    } catch (...) {
      capturing = false;
      cudaStreamEndCapture(s, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    CPF_CUDA_CHECK(cudaStreamEndCapture(s, &g));
    CPF_CUDA_CHECK(cudaGraphInstantiate(&gexec, g, 0));
    cudaGraphDestroy(g);
    graph_nodes = nlaunch - before;
    nlaunch = before;
  }

  void fit_step(int n, cpf_status* o) override {
    NvtxRange nvtx_("cpf.fit_step");
    pull_state();
    const char* env = knob("CPF_NO_GRAPH");
    const bool use_graph = graph_ok && !prof && !(env && env[0] == '1');
    if (use_graph && !gexec) capture_iteration();
    int k = 0;
    while (k < n && hst->stopped == 0) {
      const int batch = use_graph && !gmarks ? std::min(kPoll, n - k) : 1;
      for (int b = 0; b < batch; ++b) {
        if (use_graph) {
          CPF_CUDA_CHECK(cudaGraphLaunch(gexec, s));
          nlaunch += graph_nodes;
        } else {
          iteration();
        }
      }
      k += batch;
      pull_state();
      if (use_graph && gmarks && gmark[0] && gmark[4] && gmark[8]) {
        // sections: [rotated: branch launch + fork | else branch launch] | candidate | normalise +
        // pass A + decide | commit | [classic: fork] + join of the branch
        float t[5];
        for (int i = 0; i < 4; ++i) CPF_CUDA_CHECK(cudaEventElapsedTime(&t[i], gmark[i], gmark[i + 1]));
        CPF_CUDA_CHECK(cudaEventElapsedTime(&t[4], gmark[4], gmark[8]));
        fprintf(stderr, "[cpf graph iter] %.3f %.3f %.3f %.3f %.3f", t[0], t[1], t[2], t[3], t[4]);
        if (gmark[5] && gmark[6] && gmark[7]) {  // inside the fork: core prep | LU | inverse
          float u[3];
          CPF_CUDA_CHECK(cudaEventElapsedTime(&u[0], gmark[rotated() ? 0 : 4], gmark[5]));
          CPF_CUDA_CHECK(cudaEventElapsedTime(&u[1], gmark[5], gmark[6]));
          CPF_CUDA_CHECK(cudaEventElapsedTime(&u[2], gmark[6], gmark[7]));
          fprintf(stderr, "  | core prep %.3f LU %.3f inverse %.3f", u[0], u[1], u[2]);
        }
        fprintf(stderr, "\n");
      }
    }
    fill_status(o);
  }
  int trace(cpf_iter_record* out, int cap) override {
    pull_state();
    const int cnt = std::min(cap, hst->iter);
    std::vector<IterRecordDev> h(std::max(cnt, 1));
    if (cnt > 0) {
      CPF_CUDA_CHECK(cudaMemcpyAsync(h.data(), dtrace, sizeof(IterRecordDev) * cnt, cudaMemcpyDeviceToHost, s));
      CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    }
    for (int i = 0; i < cnt; ++i) {
      out[i].iter = h[i].iter;
      out[i].accepted = h[i].accepted;
      out[i].relerr = h[i].relerr;
      out[i].mu = h[i].mu;
    }
    return cnt;
  }
  void mttkrp(int mode, void* out) override {
    require_ready();
    reset_state(0, 0.0, 0.0, 0);
    pass_a(A, M, kAlways);
    pass_b(A, M, kAlways);
    if (mode == 0) {
      CPF_CUDA_CHECK(cudaMemcpyAsync(out, M, RT * sizeof(T), cudaMemcpyDeviceToHost, s));
    } else {
      if (mode < 1 || mode > N) throw ApiError(CPF_E_ARG, "mode out of range");
      CPF_CUDA_CHECK(cudaMemcpyAsync(out, M + offs[mode - 1], dims[mode - 1] * R * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
  }
  double relative_error() override {
    require_ready();
    reset_state(0, 0.0, 0.0, 0);
    const double ysq = ynorm_sq();
    if (ysq == 0.0) throw ApiError(CPF_E_ZERODIV, "relative error undefined for a zero tensor");
    direct_resid(A, dscal + 5, kAlways);
    double res;
    CPF_CUDA_CHECK(cudaMemcpyAsync(&res, dscal + 5, sizeof(double), cudaMemcpyDeviceToHost, s));
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    return std::sqrt(res) / std::sqrt(ysq);
  }
  int flm_step(double mu, int variant, int refine, void* out) override {
    require_ready();
    reset_state(variant, mu, 0.0, 1);
    build_cache_and_mttkrps(kAlways);
    candidate(refine, kAlways);
    pull_state();
    if (hst->err_code) return hst->err_code;
    CPF_CUDA_CHECK(cudaMemcpyAsync(out, Cand, RT * sizeof(T), cudaMemcpyDeviceToHost, s));
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    return 0;
  }
  void profile(int on) override {
    prof = on != 0;
    if (prof) for (auto& v : ph_max) v = 0.0;
  }
  void phase_max(double* ms, int n) override {
    for (int i = 0; i < n && i < kNumPhases; ++i) ms[i] = ph_max[i];
  }
  void phase_times(double* ms, int64_t* cnt, int n) override {
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    for (auto& e : evs) {
      float t = 0.f;
      CPF_CUDA_CHECK(cudaEventElapsedTime(&t, e.a, e.b));
      ph_ms[e.ph] += t;
      ph_cnt[e.ph] += 1;
      ph_max[e.ph] = std::max(ph_max[e.ph], (double)t);
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    evs.clear();
    const bool verbose = knob("CPF_MARKS") && knob("CPF_MARKS")[0] == '2';
    for (size_t i = 0; i + 1 < marks.size(); ++i) {
      const int a = marks[i].first, b = marks[i + 1].first;
      if (b == a + 1 && a < 4) {
        float t = 0.f;
        CPF_CUDA_CHECK(cudaEventElapsedTime(&t, marks[i].second, marks[i + 1].second));
        mark_ms[a] += t;
        if (verbose) fprintf(stderr, "%s%.3f%s", a == 0 ? "[cpf iter] " : " ", t, a == 3 ? "\n" : "");
      }
    }
    for (auto& m : marks) cudaEventDestroy(m.second);
    marks.clear();
    if (const char* e = knob("CPF_MARKS"))
      if (e[0] == '1')
        fprintf(stderr, "[cpf marks] branch launch (+ fork, rotated) %.3f  candidate %.3f  passA+decide %.3f  commit %.3f ms (totals)\n",
                mark_ms[0], mark_ms[1], mark_ms[2], mark_ms[3]);
    for (int i = 0; i < n && i < kNumPhases; ++i) {
      ms[i] = ph_ms[i];
      cnt[i] = ph_cnt[i];
    }
  }
  int64_t launches() const override { return nlaunch; }
  int pass_impl() const override { return use_oz ? CPF_PASS_OZAKI : use_dmma ? CPF_PASS_DMMA : CPF_PASS_FMA; }
  void pass_guard(int64_t* fallbacks, int* rejected) override {
    int n = 0;
    CPF_CUDA_CHECK(cudaMemcpyAsync(&n, reinterpret_cast<const char*>(fl) + offsetof(DevFlags, oz_fallbacks), sizeof(int),
                                   cudaMemcpyDeviceToHost, s));
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    if (fallbacks) *fallbacks = n;
    if (rejected) *rejected = oz_y_rejected ? 1 : 0;
  }

  // Partial Gram block  Ya_(n) Yb_(n)^H  (Ina x Inb) -> out (device, column-major, ld Ina)
  void gram_block(const T* Ya, const T* Yb, int64_t P, int64_t Ina, int64_t Inb, int64_t Q, T* out) {
    const int64_t K = P * Q;
    const int ta = (int)((Ina + 31) / 32), tb = (int)((Inb + 31) / 32);
    int nsplit = (int)std::max<int64_t>(1, std::min<int64_t>((K + 4095) / 4096, (148 * 8) / std::max(1, ta * tb) + 1));
    const int64_t kchunk = ((K + nsplit - 1) / nsplit + 31) / 32 * 32;
    nsplit = (int)((K + kchunk - 1) / kchunk);
    T* part = nullptr;
    CPF_CUDA_CHECK(cudaMallocAsync(&part, sizeof(T) * (size_t)nsplit * Ina * Inb, s));
    launch(k_unfold_gram<T>, dim3(ta * tb, nsplit), 256, 0, Ya, Yb, P, Ina, Inb, Q, kchunk, part);
    launch(k_gram_reduce<T>, nblocks(Ina * Inb, 256), 256, 0, (const T*)part, nsplit, Ina * Inb, out);
    CPF_CUDA_CHECK(cudaFreeAsync(part, s));
  }

  // G_n = Y_(n) Y_(n)^H on the device.  Modes n < N: every rank's slab gives a partial sum over
  // its columns, allreduced.  Mode N of a sharded tensor: the rows of Y_(N) are split across
  // ranks, so rank p forms its block row G[slab_p, :] against every rank's slab (each slab
  // broadcast in turn from its owner) and the block rows are summed across ranks.
  void unfolding_gram(int mode, void* out) override {
    NvtxRange nvtx_("cpf.unfolding_gram");
    if (!have_tensor) throw ApiError(CPF_E_STATE, "no tensor bound");
    if (mode < 1 || mode > N) throw ApiError(CPF_E_ARG, "mode out of range");
    const int n = mode - 1;
    const size_t words = sizeof(T) / sizeof(double);
    if (mode == N && comm && world > 1) {
      T* G = nullptr;
      T* Yq = nullptr;
      T* blk = nullptr;
      CPF_CUDA_CHECK(cudaMallocAsync(&G, sizeof(T) * (size_t)IN * IN, s));
      CPF_CUDA_CHECK(cudaMemsetAsync(G, 0, sizeof(T) * (size_t)IN * IN, s));
      CPF_CUDA_CHECK(cudaMallocAsync(&Yq, sizeof(T) * (size_t)std::max<int64_t>(1, Lrows * Cpad), s));
      CPF_CUDA_CHECK(cudaMallocAsync(&blk, sizeof(T) * (size_t)std::max<int64_t>(1, Cpad * Cpad), s));
      for (int q = 0; q < world; ++q) {
        const int64_t lo = std::min<int64_t>(IN, (int64_t)q * Cpad);
        const int64_t cnt = std::min<int64_t>(IN, lo + Cpad) - lo;
        if (cnt <= 0) continue;
        comm->broadcast(q == wrank ? (const double*)Y : nullptr, (double*)Yq, (size_t)(Lrows * cnt) * words, q, s);
        if (Cloc <= 0) continue;
        gram_block(Y, Yq, Lrows, Cloc, cnt, 1, blk);
        launch(k_copy2d<T>, nblocks(Cloc * cnt, 256), 256, 0, (const T*)blk, Cloc, G + slab_lo + IN * lo, IN, Cloc, cnt,
               (const LmDeviceState*)st, (const DevFlags*)fl, (int)kAlways);
      }
      comm->allreduce_sum((double*)G, (size_t)IN * IN * words, s);
      CPF_CUDA_CHECK(cudaMemcpyAsync(out, G, sizeof(T) * IN * IN, cudaMemcpyDeviceToHost, s));
      CPF_CUDA_CHECK(cudaStreamSynchronize(s));
      cudaFreeAsync(G, s);
      cudaFreeAsync(Yq, s);
      cudaFreeAsync(blk, s);
      CPF_CUDA_CHECK(cudaStreamSynchronize(s));
      return;
    }
    int64_t P = 1, Q = 1;
    for (int k = 0; k < n; ++k) P *= dims[k];
    for (int k = n + 1; k < N; ++k) Q *= (k == N - 1) ? Cloc : dims[k];
    const int64_t In = (n == N - 1) ? Cloc : dims[n];
    T* G = nullptr;
    CPF_CUDA_CHECK(cudaMallocAsync(&G, sizeof(T) * (size_t)In * In, s));
    if (Jloc > 0) gram_block(Y, Y, P, In, In, Q, G);
    else CPF_CUDA_CHECK(cudaMemsetAsync(G, 0, sizeof(T) * (size_t)In * In, s));
    if (comm && mode < N) comm->allreduce_sum((double*)G, (size_t)In * In * words, s);
    CPF_CUDA_CHECK(cudaMemcpyAsync(out, G, sizeof(T) * In * In, cudaMemcpyDeviceToHost, s));
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    cudaFreeAsync(G, s);
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
  }

  // ------------------------------------------------------------------------------------------
  // ALS / ALS with line search (solver.py:294-316, kruskal.py:245-293) on the engine's kernels:
  // one MTTKRP per mode per sweep through pass A (modes 1..N-1) / pass B (mode N) at the
  // partially updated factors, the Gram cache, pinv_psd by Jacobi (als.cuh), A_n = M_n pinv^T.
  // ------------------------------------------------------------------------------------------
  T* Hist = nullptr;   // previous iterate (history of the line search)
  T* Pinv = nullptr;   // R x R
  bool have_hist = false, pinv_attr = false;
  double ysq_cached = -1.0;

  void als_alloc() {
    if (R > kPinvMaxR) throw ApiError(CPF_E_UNSUPPORTED, "ALS: rank > 64 is outside the pinv_psd kernel");
    if (!Hist) Hist = dalloc<T>(RT);
    if (!Pinv) Pinv = dalloc<T>((size_t)R * R);
    if (!pinv_attr) {
      CPF_CUDA_CHECK(cudaFuncSetAttribute(k_pinv_psd<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)pinv_smem_bytes<T>(kPinvMaxR)));
      pinv_attr = true;
    }
  }
  // one ALS sweep of F in place (kruskal.py:257-265)
  void als_sweep(T* F) {
    for (int n = 0; n < N; ++n) {
      if (n < N - 1) pass_a(F, M, kAlways);
      else pass_b(F, M, kAlways);
      cross_gram(F, F, Cg, kAlways);
      cache_from_grams(Cg, kAlways);
      launch(k_pinv_psd<T>, 1, 256, pinv_smem_bytes<T>(R), (const T*)(Gx + (size_t)n * R * R), R, Pinv);
      launch(k_als_factor<T>, nblocks(dims[n] * R, 128), 128, (size_t)R * R * sizeof(T), (const T*)(M + offs[n]),
             (const T*)Pinv, dims[n], R, F + offs[n]);
    }
  }
  double relerr_of(const T* F) {
    if (ysq_cached < 0.0) ysq_cached = ynorm_sq();
    if (ysq_cached == 0.0) throw ApiError(CPF_E_ZERODIV, "relative error undefined for a zero tensor");
    direct_resid(F, dscal + 5, kAlways);
    double res;
    CPF_CUDA_CHECK(cudaMemcpyAsync(&res, dscal + 5, sizeof(double), cudaMemcpyDeviceToHost, s));
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    return std::sqrt(res) / std::sqrt(ysq_cached);
  }
  // One ALS (line_search = 0) or ALS-ls step of the bound factors A at iteration t; the history is
  // the iterate before the previous call (none right after set_factors) or set_history's.
  double als_step(int line_search, int t) override {
    NvtxRange nvtx_("cpf.als_step");
    require_ready();
    als_alloc();
    reset_state(0, 0.0, 0.0, 0);
    CPF_CUDA_CHECK(cudaMemcpyAsync(Cand, A, RT * sizeof(T), cudaMemcpyDeviceToDevice, s));
    als_sweep(Cand);
    const T* best = Cand;
    double err = -1.0;
    if (line_search && have_hist) {  // kruskal.py:279-292
      err = relerr_of(Cand);
      const double steps[2] = {1.1, std::pow((double)t, 1.0 / 3.0)};
      T* bufs[2] = {V1, V2};
      for (int k = 0; k < 2; ++k) {
        launch(k_als_extrap<T>, nblocks(RT, 256), 256, 0, (const T*)Hist, (const T*)Cand, steps[k], RT, bufs[k]);
        const double e2 = relerr_of(bufs[k]);
        if (e2 < err) { best = bufs[k]; err = e2; }
      }
    }
    CPF_CUDA_CHECK(cudaMemcpyAsync(Hist, A, RT * sizeof(T), cudaMemcpyDeviceToDevice, s));
    have_hist = true;
    CPF_CUDA_CHECK(cudaMemcpyAsync(A, best, RT * sizeof(T), cudaMemcpyDeviceToDevice, s));
    if (err < 0.0) err = relerr_of(A);
    return err;
  }
  // fast_damped_inverse (hessian.py:232-277) at the bound factors: gamma_tilde_n = (Gamma_n + mu I)^-1
  // (N R x R) and the core grid D (nB x nB), through the engine's Gram cache, LU and substitution
  // on the identity (fdi.cuh).  use_kinv: -1 auto (kernel_is_invertible), 0 K-free, 1 K^{-1}.  Returns a
  // CPF_ERR_* code (0 = ok).  Needs factors only (no tensor).
  int fast_damped_inverse(double mu, int use_kinv, void* gt_out, void* d_out) override {
    NvtxRange nvtx_("cpf.fast_damped_inverse");
    if (!have_factors) throw ApiError(CPF_E_STATE, "no factors bound");
    if (!(mu > 0.0)) throw ApiError(CPF_E_ARG, "mu must be positive");
    if (N < 2) throw ApiError(CPF_E_ARG, "kernel inverse needs at least two modes");
    reset_state(use_kinv < 0 ? 0 : (use_kinv ? 2 : 1), mu, 0.0, 1);
    cross_gram(A, A, Cg, kAlways);
    cache_from_grams(Cg, kAlways);
    int kok = 0;
    CPF_CUDA_CHECK(cudaMemcpyAsync(&kok, kinv_ok, sizeof(int), cudaMemcpyDeviceToHost, s));
    pull_state();
    if (use_kinv == 1 && !kok) return CPF_ERR_KINV_SINGULAR;
    const int kinv = hst->use_kinv;
    launch(k_damped_inverses<T>, 2 * N, 128, 2 * R * R * sizeof(T), (const T*)Gx, N, R, Gti, Gi, st, (const DevFlags*)fl,
           (int)kAlways, (const int*)nullptr, (const double*)nullptr, (int*)nullptr);
    pull_state();
    if (hst->err_code) return CPF_ERR_SINGULAR;  // np.linalg.inv(g + mu I) failed
    launch(k_fdi_assemble<T>, nblocks((int64_t)nB * nB, 256), 256, 0, Phi, N, R, (const T*)Cg, (const T*)Gx,
           (const T*)Gp, (const T*)Gf, mu, kinv);
    lu_factor(0);
    pull_state();
    if (hst->err_code) return kinv ? CPF_ERR_SINGULAR : CPF_ERR_SBCK_SINGULAR;
    if (!TriTmp) TriTmp = dalloc<T>((size_t)nB * nB);
    launch(k_perm_ident<T>, nblocks((int64_t)nB * nB, 256), 256, 0, (const int*)lu.perm, nB, TriTmp);
    launch(k_trsm_ident<T, true>, nblocks(nB, 16), 256, 0, (const T*)Phi, nB, TriTmp);
    launch(k_trsm_ident<T, false>, nblocks(nB, 16), 256, 0, (const T*)Phi, nB, TriTmp);
    const T* Dres = TriTmp;
    if (!kinv) {
      launch(k_fdi_gtk<T>, nblocks((int64_t)nB * nB, 256), 256, 0, (const T*)TriTmp, N, R, (const T*)Gi, (const T*)Gp,
             Phi);
      Dres = Phi;
    }
    CPF_CUDA_CHECK(cudaMemcpyAsync(gt_out, Gi, sizeof(T) * N * R * R, cudaMemcpyDeviceToHost, s));
    CPF_CUDA_CHECK(cudaMemcpyAsync(d_out, Dres, sizeof(T) * nB * nB, cudaMemcpyDeviceToHost, s));
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    return 0;
  }
  void set_history(const void* p) override {
    als_alloc();
    if (!p) { have_hist = false; return; }
    CPF_CUDA_CHECK(cudaMemcpyAsync(Hist, p, RT * sizeof(T), cudaMemcpyHostToDevice, s));
    CPF_CUDA_CHECK(cudaStreamSynchronize(s));
    have_hist = true;
  }
};

}  // namespace cpf

// ============================================================================================
// C ABI (include/cpfast_b200.h)
// ============================================================================================
struct cpf_engine {
  std::unique_ptr<cpf::EngineBase> impl;
  std::string err;
};

namespace {
thread_local std::string g_create_error;

template <class F>
int guarded(cpf_engine* e, F&& f) {
  try {
    f();
    return CPF_OK;
  } catch (const ApiError& x) {
    if (e) e->err = x.what();
    else g_create_error = x.what();
    return x.code;
  } catch (const CudaError& x) {
    if (e) e->err = x.what();
    else g_create_error = x.what();
    return CPF_E_CUDA;
  } catch (const std::exception& x) {
    if (e) e->err = x.what();
    else g_create_error = x.what();
    return CPF_E_CUDA;
  }
}
}  // namespace

extern "C" {

int cpf_abi_version(void) { return CPF_ABI_VERSION; }

int cpf_pool_reserve(int device, int64_t bytes) {
  if (cudaSetDevice(device) != cudaSuccess) return CPF_E_CUDA;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return CPF_E_CUDA;
  uint64_t thr = ~0ull;
  cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  void* p = nullptr;
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return CPF_E_CUDA;
  cudaError_t e = cudaMallocAsync(&p, (size_t)std::max<int64_t>(bytes, 1), st);
  if (e == cudaSuccess) e = cudaFreeAsync(p, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (e != cudaSuccess) { cudaGetLastError(); return CPF_E_CUDA; }
  return CPF_OK;
}

int cpf_device_count(int* n) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  if (n) *n = c;
  return CPF_OK;
}

int cpf_nccl_unique_id(void* out128) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return CPF_E_NCCL;
  std::memcpy(out128, &id, sizeof(id));
  return CPF_OK;
}

int cpf_engine_create(cpf_engine** out, int device, int kind, int order, const int64_t* dims, int rank,
                      int world_rank, int world_size, const void* nccl_uid128) {
  if (!out) return CPF_E_ARG;
  *out = nullptr;
  auto* e = new cpf_engine();
  int rc = guarded(nullptr, [&] {
    if (kind == CPF_REAL)
      e->impl.reset(new cpf::Engine<double>(device, order, dims, rank, world_rank, world_size, nccl_uid128));
    else if (kind == CPF_COMPLEX)
      e->impl.reset(new cpf::Engine<cplx>(device, order, dims, rank, world_rank, world_size, nccl_uid128));
    else
      throw ApiError(CPF_E_KIND, "unknown scalar kind");
  });
  if (rc != CPF_OK) {
    e->err = g_create_error;
    *out = e;  // caller reads the message then destroys
    return rc;
  }
  *out = e;
  return CPF_OK;
}

int cpf_loopback_group_create(int world, void** out) {
  if (!out) return CPF_E_ARG;
  *out = nullptr;
  try {
    *out = new cpf::LoopbackGroup(world);
    return CPF_OK;
  } catch (const ApiError& x) {
    g_create_error = x.what();
    return x.code;
  } catch (const std::exception& x) {
    g_create_error = x.what();
    return CPF_E_CUDA;
  }
}

void cpf_loopback_group_destroy(void* group) { delete static_cast<cpf::LoopbackGroup*>(group); }

int cpf_engine_create_loopback(cpf_engine** out, int device, int kind, int order, const int64_t* dims, int rank,
                               int world_rank, void* group) {
  if (!out || !group) return CPF_E_ARG;
  *out = nullptr;
  auto* g = static_cast<cpf::LoopbackGroup*>(group);
  auto* e = new cpf_engine();
  int rc = guarded(nullptr, [&] {
    if (kind == CPF_REAL)
      e->impl.reset(new cpf::Engine<double>(device, order, dims, rank, world_rank, g->world, nullptr, g));
    else if (kind == CPF_COMPLEX)
      e->impl.reset(new cpf::Engine<cplx>(device, order, dims, rank, world_rank, g->world, nullptr, g));
    else
      throw ApiError(CPF_E_KIND, "unknown scalar kind");
  });
  if (rc != CPF_OK) e->err = g_create_error;
  *out = e;
  return rc;
}

void cpf_engine_destroy(cpf_engine* e) { delete e; }

const char* cpf_engine_last_error(const cpf_engine* e) {
  return e ? e->err.c_str() : g_create_error.c_str();
}

int cpf_engine_slab(const cpf_engine* e, int64_t* lo, int64_t* hi) {
  if (!e || !e->impl) return CPF_E_STATE;
  e->impl->slab(lo, hi);
  return CPF_OK;
}

void* cpf_engine_stream(cpf_engine* e) { return (e && e->impl) ? e->impl->stream() : nullptr; }

int cpf_engine_set_tensor(cpf_engine* e, const void* data, int64_t nelem, int where) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] { e->impl->set_tensor(data, nelem, where); });
}

int cpf_engine_load_cptn(cpf_engine* e, const char* path, int64_t payload_offset) {
  if (!e || !e->impl || !path) return CPF_E_STATE;
  return guarded(e, [&] { e->impl->load_cptn(path, payload_offset); });
}

int cpf_engine_set_factors(cpf_engine* e, const void* stacked) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] { e->impl->set_factors(stacked); });
}

int cpf_engine_get_factors(cpf_engine* e, void* stacked) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] { e->impl->get_factors(stacked); });
}

int cpf_engine_fit_begin(cpf_engine* e, int variant, double tau, double tol, int max_iters, cpf_status* st) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] { e->impl->fit_begin(variant, tau, tol, max_iters, st); });
}

int cpf_engine_fit_step(cpf_engine* e, int n_iters, cpf_status* st) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] { e->impl->fit_step(n_iters, st); });
}

int cpf_engine_trace(cpf_engine* e, cpf_iter_record* out, int cap, int* n) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] { *n = e->impl->trace(out, cap); });
}

int cpf_engine_mttkrp(cpf_engine* e, int mode, void* out) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] { e->impl->mttkrp(mode, out); });
}

int cpf_pinv_psd(int device, int kind, int R, const void* gram, void* out) {
  if (R < 1 || R > kPinvMaxR || !gram || !out) return CPF_E_ARG;
  if (kind != CPF_REAL && kind != CPF_COMPLEX) return CPF_E_KIND;
  const size_t es = kind == CPF_COMPLEX ? 16 : 8;
  const size_t bytes = es * (size_t)R * R;
  void *dg = nullptr, *dout = nullptr;
  cudaError_t rc = cudaSetDevice(device);
  if (rc == cudaSuccess) rc = cudaMalloc(&dg, bytes);
  if (rc == cudaSuccess) rc = cudaMalloc(&dout, bytes);
  if (rc == cudaSuccess) rc = cudaMemcpy(dg, gram, bytes, cudaMemcpyHostToDevice);
  if (rc == cudaSuccess) {
    if (kind == CPF_COMPLEX) {
      rc = cudaFuncSetAttribute(k_pinv_psd<cplx>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)pinv_smem_bytes<cplx>(kPinvMaxR));
      if (rc == cudaSuccess) k_pinv_psd<cplx><<<1, 256, pinv_smem_bytes<cplx>(R)>>>((const cplx*)dg, R, (cplx*)dout);
    } else {
      rc = cudaFuncSetAttribute(k_pinv_psd<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)pinv_smem_bytes<double>(kPinvMaxR));
      if (rc == cudaSuccess) k_pinv_psd<double><<<1, 256, pinv_smem_bytes<double>(R)>>>((const double*)dg, R, (double*)dout);
    }
    if (rc == cudaSuccess) rc = cudaGetLastError();
  }
  if (rc == cudaSuccess) rc = cudaMemcpy(out, dout, bytes, cudaMemcpyDeviceToHost);
  if (dg) cudaFree(dg);
  if (dout) cudaFree(dout);
  return rc == cudaSuccess ? CPF_OK : CPF_E_CUDA;
}

int cpf_engine_als_step(cpf_engine* e, int line_search, int t, double* relerr) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] {
    const double v = e->impl->als_step(line_search, t);
    if (relerr) *relerr = v;
  });
}

int cpf_engine_fast_damped_inverse(cpf_engine* e, double mu, int use_kernel_inverse, void* gamma_tilde, void* core,
                                   int* err_code) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] { *err_code = e->impl->fast_damped_inverse(mu, use_kernel_inverse, gamma_tilde, core); });
}

int cpf_engine_set_history(cpf_engine* e, const void* stacked) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] { e->impl->set_history(stacked); });
}

int cpf_engine_relative_error(cpf_engine* e, double* out) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] { *out = e->impl->relative_error(); });
}

int cpf_engine_flm_step(cpf_engine* e, double mu, int variant, int refine_steps, void* cand, int* err_code) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] { *err_code = e->impl->flm_step(mu, variant, refine_steps, cand); });
}

int cpf_engine_profile(cpf_engine* e, int enable) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] { e->impl->profile(enable); });
}

int cpf_engine_phase_times(cpf_engine* e, double* ms_out, int64_t* counts_out, int nphases) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] { e->impl->phase_times(ms_out, counts_out, nphases); });
}

int cpf_engine_phase_max(cpf_engine* e, double* ms_out, int nphases) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] { e->impl->phase_max(ms_out, nphases); });
}

int64_t cpf_engine_launch_count(const cpf_engine* e) { return (e && e->impl) ? e->impl->launches() : 0; }
int cpf_engine_pass_impl(const cpf_engine* e) { return (e && e->impl) ? e->impl->pass_impl() : -1; }

int cpf_engine_pass_guard(cpf_engine* e, int64_t* fallbacks, int* tensor_rejected) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] { e->impl->pass_guard(fallbacks, tensor_rejected); });
}

int cpf_engine_unfolding_gram(cpf_engine* e, int mode, void* out) {
  if (!e || !e->impl) return CPF_E_STATE;
  return guarded(e, [&] { e->impl->unfolding_gram(mode, out); });
}

}  // extern "C"

// diagnostic: on != 0 resets and enables the LU timeline, on == 0 disables it and copies it out
extern "C" int cpf_debug_lu_trace(int on, unsigned long long* out) {
  static unsigned long long init[3 * 512 * 2];
  if (on) {
    for (int i = 0; i < 3 * 512; ++i) { init[2 * i] = ~0ull; init[2 * i + 1] = 0ull; }
    if (cudaMemcpyToSymbol(cpf::g_lu_trace, init, sizeof(init)) != cudaSuccess) return -4;
  } else if (out) {
    if (cudaDeviceSynchronize() != cudaSuccess) return -4;
    if (cudaMemcpyFromSymbol(out, cpf::g_lu_trace, sizeof(init)) != cudaSuccess) return -4;
    if (cudaMemcpyFromSymbol(out + 3 * 512 * 2, cpf::g_lu_clk, sizeof(unsigned long long) * 1024) != cudaSuccess)
      return -4;
  }
  return cudaMemcpyToSymbol(cpf::g_lu_trace_on, &on, sizeof(int)) == cudaSuccess ? 0 : -4;
}

extern "C" int cpf_debug_panel_cycles(long long* out12) {
  if (cudaMemcpyFromSymbol(out12 + 8, cpf::g_panel_seg, sizeof(long long) * 12) != cudaSuccess) return -4;
  return cudaMemcpyFromSymbol(out12, cpf::g_panel_cycles, sizeof(long long) * 8) == cudaSuccess ? 0 : -4;
}
