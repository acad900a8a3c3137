// Common device helpers for the B200 fast damped Gauss-Newton (fLM) CP engine.
//
// Scalar kinds: the reference runs one code path over float64 and complex128
// (cpfast/solver.py:1-12, cpfast/kruskal.py:1-7).  Here every kernel is a
// template over T in {double, cplx}; conjugation is a no-op for double, so the
// placements (Hermitian Grams, conj Khatri-Rao in MTTKRP, Gamma^T = conj Gamma)
// are written once, as in the reference.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <cmath>

// Engine knobs: CPF_* environment variables for diagnostics, tests and A/B experiments (the full
// list is DESIGN.md §11).  They are read only when CPF_DEBUG=1, so a production process ignores
// stray CPF_* variables and always runs the planned paths.
inline const char* knob(const char* name) {
  const char* d = std::getenv("CPF_DEBUG");
  return (d && d[0] == '1') ? std::getenv(name) : nullptr;
}

struct __align__(16) cplx {
  double x, y;
};

// ------------------------------------------------------------------------------------------
// Scalar algebra (double and complex128)
// ------------------------------------------------------------------------------------------
template <class T> struct ScalarTraits;
template <> struct ScalarTraits<double> { static constexpr bool kComplex = false; static constexpr int kWords = 1; };
template <> struct ScalarTraits<cplx>   { static constexpr bool kComplex = true;  static constexpr int kWords = 2; };

__host__ __device__ __forceinline__ double sc_zero(double) { return 0.0; }
__host__ __device__ __forceinline__ cplx sc_zero(cplx) { return cplx{0.0, 0.0}; }
template <class T> __host__ __device__ __forceinline__ T zero_of() { return sc_zero(T{}); }
template <class T> __host__ __device__ __forceinline__ T from_real(double a);
template <> __host__ __device__ __forceinline__ double from_real<double>(double a) { return a; }
template <> __host__ __device__ __forceinline__ cplx from_real<cplx>(double a) { return cplx{a, 0.0}; }

__host__ __device__ __forceinline__ double cj(double a) { return a; }
__host__ __device__ __forceinline__ cplx cj(cplx a) { return cplx{a.x, -a.y}; }
__host__ __device__ __forceinline__ double re(double a) { return a; }
__host__ __device__ __forceinline__ double re(cplx a) { return a.x; }
__host__ __device__ __forceinline__ double im(double) { return 0.0; }
__host__ __device__ __forceinline__ double im(cplx a) { return a.y; }

__host__ __device__ __forceinline__ double add(double a, double b) { return a + b; }
__host__ __device__ __forceinline__ cplx add(cplx a, cplx b) { return cplx{a.x + b.x, a.y + b.y}; }
__host__ __device__ __forceinline__ double sub(double a, double b) { return a - b; }
__host__ __device__ __forceinline__ cplx sub(cplx a, cplx b) { return cplx{a.x - b.x, a.y - b.y}; }
__host__ __device__ __forceinline__ double neg(double a) { return -a; }
__host__ __device__ __forceinline__ cplx neg(cplx a) { return cplx{-a.x, -a.y}; }
__host__ __device__ __forceinline__ double mul(double a, double b) { return a * b; }
__host__ __device__ __forceinline__ cplx mul(cplx a, cplx b) {
  return cplx{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
__host__ __device__ __forceinline__ double scale(double a, double s) { return a * s; }
__host__ __device__ __forceinline__ cplx scale(cplx a, double s) { return cplx{a.x * s, a.y * s}; }
// a / b with the straightforward formula (reference divisions are by phases / pivots)
__host__ __device__ __forceinline__ double dvd(double a, double b) { return a / b; }
__host__ __device__ __forceinline__ cplx dvd(cplx a, cplx b) {
  // Smith's algorithm, robust to scaling
  if (fabs(b.x) >= fabs(b.y)) {
    double r = b.y / b.x, d = b.x + b.y * r;
    return cplx{(a.x + a.y * r) / d, (a.y - a.x * r) / d};
  } else {
    double r = b.x / b.y, d = b.y + b.x * r;
    return cplx{(a.x * r + a.y) / d, (a.y * r - a.x) / d};
  }
}
// 1/a via the hardware-seeded IEEE reciprocal (__drcp_rn): avoids the long div.rn.f64 sequence
__device__ __forceinline__ double rcp_of(double a) { return __drcp_rn(a); }
__device__ __forceinline__ cplx rcp_of(cplx a) {
  const double s = __drcp_rn(a.x * a.x + a.y * a.y);
  return cplx{a.x * s, -a.y * s};
}
// modulus |a| (np.abs): hypot for complex
__host__ __device__ __forceinline__ double modulus(double a) { return fabs(a); }
__host__ __device__ __forceinline__ double modulus(cplx a) { return hypot(a.x, a.y); }
// |a|^2
__host__ __device__ __forceinline__ double abs2(double a) { return a * a; }
__host__ __device__ __forceinline__ double abs2(cplx a) { return a.x * a.x + a.y * a.y; }
// LAPACK i?amax magnitude: |x| real, |re|+|im| complex (dcabs1)
__host__ __device__ __forceinline__ double pivmag(double a) { return fabs(a); }
__host__ __device__ __forceinline__ double pivmag(cplx a) { return fabs(a.x) + fabs(a.y); }

// streaming / read-only loads
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ cplx ld_stream(const cplx* p) {
  double2 v = __ldcs(reinterpret_cast<const double2*>(p));
  return cplx{v.x, v.y};
}
__device__ __forceinline__ double ld_ro(const double* p) { return __ldg(p); }
__device__ __forceinline__ cplx ld_ro(const cplx* p) {
  double2 v = __ldg(reinterpret_cast<const double2*>(p));
  return cplx{v.x, v.y};
}
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ int ld_cg(const int* p) { return __ldcg(p); }
__device__ __forceinline__ cplx ld_cg(const cplx* p) {
  double2 v = __ldcg(reinterpret_cast<const double2*>(p));
  return cplx{v.x, v.y};
}

// acc += a * b
__device__ __forceinline__ void fma_acc(double& acc, double a, double b) { acc = fma(a, b, acc); }
__device__ __forceinline__ void fma_acc(cplx& acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
__device__ __forceinline__ void fma_cacc(double& acc, double a, double b) { acc = fma(a, b, acc); }
__device__ __forceinline__ void fma_cacc(cplx& acc, cplx a, cplx b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}
// acc -= a * b
__device__ __forceinline__ void fms_acc(double& acc, double a, double b) { acc = fma(-a, b, acc); }
__device__ __forceinline__ void fms_acc(cplx& acc, cplx a, cplx b) {
  acc.x = fma(-a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(-a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}

// ------------------------------------------------------------------------------------------
// Shuffles / reductions (deterministic fixed trees)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ double shfl_down(double v, int o) { return __shfl_down_sync(0xffffffffu, v, o); }
__device__ __forceinline__ cplx shfl_down(cplx v, int o) {
  return cplx{__shfl_down_sync(0xffffffffu, v.x, o), __shfl_down_sync(0xffffffffu, v.y, o)};
}
__device__ __forceinline__ double shfl_idx(double v, int l) { return __shfl_sync(0xffffffffu, v, l); }
__device__ __forceinline__ cplx shfl_idx(cplx v, int l) {
  return cplx{__shfl_sync(0xffffffffu, v.x, l), __shfl_sync(0xffffffffu, v.y, l)};
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = add(v, shfl_down(v, o));
  return v;
}

// Block-wide sum; result valid in thread 0.  `scratch` must hold blockDim/32 T.
template <class T>
__device__ __forceinline__ T block_sum(T v, T* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  T r = zero_of<T>();
  if (wid == 0) {
    r = lane < nw ? scratch[lane] : zero_of<T>();
    r = warp_sum(r);
  }
  return r;
}

// ------------------------------------------------------------------------------------------
// Engine status codes (mirrors include/cpfast_b200.h)
// ------------------------------------------------------------------------------------------
enum : int {
  kErrNone = 0,
  kErrSingular = 1,        // exactly zero pivot: numpy LinAlgError("Singular matrix")
  kErrKernelSingular = 2,  // flm-b with non-invertible K (solver.py:146-147)
  kErrPhi1Singular = 3,    // flm-a: I + Psi K singular (hessian.py:210-211)
  kErrZeroColumn = 4,      // normalize_equal_energy zero-norm vector (kruskal.py:184-185)
  kErrNonFinite = 5,
};

// Device-resident LM state: the whole accept/reject control lives on the GPU so that an
// iteration is a fixed launch sequence (graph-capturable); the host only polls it.
struct LmDeviceState {
  double mu, growth;
  double err, err_sq;        // current model (solver.py:331-332)
  double ynorm, ynorm_sq;
  double cand_err, cand_sq;  // candidate (solver.py:354-355)
  double yx_re, xx;          // Re<Y,X_cand>, ||X_cand||^2
  double denom, rho;
  double tol;
  double deltas[10];         // ring of the last 10 |err - cand_err| (solver.py:367,373)
  int ndeltas;
  int iter;                  // last completed iteration t
  int accepted;              // decision of the last iteration
  int stopped;               // 0 running, 1 tol, 2 mu_overflow, 3 error, 4 max_iters
  int err_code;              // kErr* of the error stop
  int err_iter;
  int use_kinv;              // flm-b (1) / flm-a (0) for the current cache
  int variant;               // 0 auto, 1 flm-a, 2 flm-b
  int max_iters;
  int cand_zero;             // normalised candidate had a zero-norm column (raise on accept)
  int err_direct;            // err/err_sq come from a direct residual (not the identity)
  int force_direct;          // evaluate every trial fit directly (cheap-pass / LU-bound regime)
  int rej_grow;              // last decision took the rho <= 0 branch (mu *= growth): the only
                             // case whose next core system is Phi(Grams_t, mu_t * growth_t), i.e.
                             // the speculated one.  A rho > 0 rejection (cand_err >= err) shrinks
                             // mu instead and needs a freshly factored core system.
  int test_negdenom_iter;    // test hook (CPF_TEST_NEGDENOM=t): negate the gain-ratio denominator
                             // at iteration t to force a rho > 0 / not-improved rejection
  int test_singular_iter;   // test hook (CPF_TEST_SINGULAR=t): zero a column of the core system that
                            // iteration t factors (fault injection: a zero pivot, solver.py:349-352)
  int spec_iter;            // st->iter when this iteration's speculative rejection branch started
  int accept_iter;          // t when decision t was an acceptance (else -1): ONE word, so a reader
                            // on another SM sees the decision and its iteration together
};

// Gate of the core-system kernels (Phi, LU, inverse): gate_running 0 = always, 1 = while the fit
// runs, 2 = while it runs unless the last decision was a rho <= 0 rejection (the main core system
// when that rejection branch was factored speculatively, engine.cu prepare_core)
__device__ __forceinline__ int ld_volatile_int(const int* p) { return *(const volatile int*)p; }
// 3 = the speculative rejection branch: as 1, and abandoned as soon as this iteration's decision is
// an acceptance (the branch is then never used; its remaining kernels return at once and leave the
// SMs to the accepted step's fork)
__device__ __forceinline__ bool lu_gated(const LmDeviceState* st, int gate_running) {
  return st && gate_running &&
         (st->stopped || st->err_code || (gate_running == 2 && st->rej_grow) ||
          (gate_running == 3 && ld_volatile_int(&st->accept_iter) == st->spec_iter + 1));
}
// Kernels whose CTAs synchronise with each other (cluster panels, look-back substitutions, the
// persistent LU) must take the same branch in every CTA; the acceptance of the running step can
// land between two CTAs' reads, so they never abandon the speculative branch mid-way.
__device__ __forceinline__ bool lu_gated_sync(const LmDeviceState* st, int gate_running) {
  return lu_gated(st, gate_running == 3 ? 1 : gate_running);
}

struct IterRecordDev {
  double relerr, mu;
  int iter, accepted;
};

#define CPF_CUDA_CHECK(expr)                                        \
  do {                                                              \
    cudaError_t _e = (expr);                                        \
    if (_e != cudaSuccess) throw CudaError(_e, #expr, __FILE__, __LINE__); \
  } while (0)

// ------------------------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, 1-D) + mbarrier pipeline helpers (sm_90+/sm_100a)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Programmatic dependent launch.  Kernels of the iteration graph are launched with programmatic
// stream serialization: kernel n+1 may be scheduled while kernel n still runs.  Every kernel starts
// here: wait until the predecessor grid has completed and its memory is visible, then let the
// successor be scheduled (its CTAs park in their own wait).  Launch latency of a chain of small
// dependent kernels overlaps the previous kernel instead of adding to it.  No-op for a normally
// launched kernel.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// named barrier over the first `nthreads` threads (consumer warps only)
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// DSMEM: address of `p` (this CTA's shared memory) in CTA `rank` of the cluster, and stores to it
__device__ __forceinline__ uint32_t mapa_u32(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void st_cluster(uint32_t addr, cplx v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
}
// 16-byte remote store that completes 16 tx-bytes on the destination CTA's mbarrier (st.async):
// the receiver learns the data has landed by waiting on its own local mbarrier, no cluster barrier.
__device__ __forceinline__ void st_async16(uint32_t raddr, double x, double y, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(raddr), "d"(x),
               "d"(y), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_cluster(uint32_t addr, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
