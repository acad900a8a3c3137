/*
 * cpfast_b200.h -- C ABI of the B200-native fast damped Gauss-Newton (fLM) CP engine.
 *
 * The reference (`cpfast`, pure Python/NumPy) has no FFI: its boundary is the Python API
 *   cpfast.fit(y: DenseTensor, config: FitConfig) -> FitResult          (pkg/src/cpfast/solver.py:278-291)
 *   cpfast.fit_complex(y, config) -> FitResult                           (pkg/src/cpfast/complexcp.py:51-54)
 *   cpfast.solver.flm_step(y, model, mu, variant, cache, mttkrps, refine_steps)  (solver.py:189-226)
 *   cpfast.kruskal.mttkrp(y, model, n)                                   (kruskal.py:126-135)
 *   cpfast.kruskal.relative_error(y, model)                              (kruskal.py:163-167)
 * This header is the native boundary those entry points are re-implemented over.  A binding is a
 * thin ctypes / cffi / pybind layer (paper_1205_2584_b200/_native.py is the in-tree one; see
 * INTEGRATION.md).  All pointers are plain; no torch types cross the boundary.
 *
 * Conventions (identical to the reference):
 *   - tensors are column-major (mode-1 index fastest), float64 or interleaved complex128;
 *   - factors are I_n x R column-major and are passed "stacked": the concatenation of the
 *     column-major vectorisations of A^(1..N) (kruskal.py:70-82);
 *   - modes are 1-based where a mode index is taken.
 * Every call is ordered on the engine's CUDA stream; calls returning host data synchronise it.
 * Multi-GPU: one engine per process/GPU; the tensor is slab-sharded along mode N
 * (cpf_engine_slab) and the engines exchange MTTKRP partials with NCCL.
 */
#ifndef CPFAST_B200_H_
#define CPFAST_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CPF_ABI_VERSION 1

/* return codes */
#define CPF_OK 0
#define CPF_E_ARG (-1)         /* ValueError: bad shape / rank / variant (solver.py:72-76, kruskal.py:132-133) */
#define CPF_E_KIND (-2)        /* TypeError / ScalarKindError (tensor.py:21-33, complexcp.py:18-22) */
#define CPF_E_CUDA (-4)        /* CUDA runtime failure */
#define CPF_E_NCCL (-5)        /* NCCL failure */
#define CPF_E_ZERODIV (-6)     /* ZeroDivisionError: zero tensor / zero-norm component (solver.py:323-324, kruskal.py:184-185) */
#define CPF_E_UNSUPPORTED (-7) /* shape outside the engine's envelope (order > 8, NR^2 too large, ...) */
#define CPF_E_STATE (-8)       /* call out of order (no tensor / factors bound) */
#define CPF_E_FORMAT (-9)      /* cptn.FormatError(ValueError): malformed tensor file (cptn.py:24-59) */

/* scalar kinds */
#define CPF_REAL 0     /* float64 */
#define CPF_COMPLEX 1  /* complex128, interleaved (re, im) */

/* variants (solver.py:44 VARIANTS, LM family only) */
#define CPF_VARIANT_AUTO 0
#define CPF_VARIANT_FLM_A 1
#define CPF_VARIANT_FLM_B 2

/* stop codes (FitResult.stop_reason, solver.py:378-383, 349-352) */
#define CPF_RUNNING 0
#define CPF_STOP_TOL 1
#define CPF_STOP_MU_OVERFLOW 2
#define CPF_STOP_ERROR 3
#define CPF_STOP_MAX_ITERS 4

/* in-loop error codes (become "error at iteration t: <msg>", solver.py:349-352) */
#define CPF_ERR_NONE 0
#define CPF_ERR_SINGULAR 1         /* LinAlgError("Singular matrix") */
#define CPF_ERR_KERNEL_SINGULAR 2  /* SingularKernelError("flm-b requested but K is singular") */
#define CPF_ERR_PHI1_SINGULAR 3    /* SingularKernelError("I + Psi K numerically singular: Singular matrix") */
#define CPF_ERR_ZERO_COLUMN 4      /* ZeroDivisionError while normalising an accepted candidate */
#define CPF_ERR_NONFINITE 5
#define CPF_ERR_KINV_SINGULAR 6    /* SingularKernelError("a pairwise Gamma entry vanishes; K is singular") (hessian.py:97-107) */
#define CPF_ERR_SBCK_SINGULAR 7    /* SingularKernelError("Sb + Chat K numerically singular: Singular matrix") (hessian.py:266-267) */

typedef struct cpf_engine cpf_engine;

/* IterRecord (solver.py:79-84) */
typedef struct {
  int32_t iter;
  int32_t accepted;
  double relerr;
  double mu;
} cpf_iter_record;

typedef struct {
  int32_t stopped;   /* CPF_RUNNING or CPF_STOP_* */
  int32_t err_code;  /* CPF_ERR_* when stopped == CPF_STOP_ERROR */
  int32_t err_iter;  /* iteration t of the error stop */
  int32_t iter;      /* last completed iteration */
  int32_t last_accepted;
  int32_t err_column;
  double relerr;     /* current relative error */
  double mu;         /* current damping */
  double ynorm;
} cpf_status;

int cpf_abi_version(void);
int cpf_device_count(int* n);
/* Grow the device's stream-ordered memory pool (which engines allocate from and return to) to at
 * least `bytes`, so a following engine's allocations are reuses instead of fresh mappings
 * (process setup, like context creation; no reference counterpart). */
int cpf_pool_reserve(int device, int64_t bytes);
/* 128-byte NCCL unique id for a multi-GPU engine group (rank 0 creates, all ranks receive). */
int cpf_nccl_unique_id(void* out128);

/* Create an engine for an order-`order` tensor with global `dims`, CP rank `rank`, scalar
 * `kind`.  world_size > 1 shards mode N across ranks and requires nccl_uid128. */
int cpf_engine_create(cpf_engine** out, int device, int kind, int order, const int64_t* dims, int rank,
                      int world_rank, int world_size, const void* nccl_uid128);
void cpf_engine_destroy(cpf_engine* e);
/* TEST TRANSPORT (no reference counterpart): a loopback group of `world` engines in ONE process on
 * one device, each driven by its own host thread, whose collectives (the same allreduce /
 * allgather / broadcast the NCCL path issues) exchange through device buffers ordered by CUDA
 * events and a host barrier -- no kernel waits on another rank's kernel.  It runs the multi-rank
 * data path (slab bounds, ragged slabs, packed allreduce, allgather reorder, sharded mode-N Gram)
 * without a multi-GPU box.  Loopback engines launch eagerly (no CUDA graph). */
int cpf_loopback_group_create(int world, void** group);
void cpf_loopback_group_destroy(void* group);
int cpf_engine_create_loopback(cpf_engine** out, int device, int kind, int order, const int64_t* dims, int rank,
                               int world_rank, void* group);
const char* cpf_engine_last_error(const cpf_engine* e);
/* Local slab [lo, hi) of mode N owned by this rank. */
int cpf_engine_slab(const cpf_engine* e, int64_t* lo, int64_t* hi);
/* The engine's CUDA stream (cudaStream_t) for event-based timing by the caller. */
void* cpf_engine_stream(cpf_engine* e);

/* Bind the local slab (column-major, prod(dims[0:N-1]) * (hi-lo) elements).
 * where = 0: host memory, copied (pinned or pageable); where = 1: device memory, borrowed. */
int cpf_engine_set_tensor(cpf_engine* e, const void* data, int64_t nelem, int where);
/* Stream this engine's slab of a CPTN tensor file (cptn.py:1-7 layout: 16-byte header, N x u64
 * dims, then the scalars column-major) straight into device memory: the slab of the last mode is
 * one contiguous byte range of the payload, read with pread into two pinned staging buffers and
 * copied asynchronously -- no host copy of the tensor.  Replaces cptn.read_tensor (cptn.py:37-59)
 * + DenseTensor upload on the fit path (cli.py:115-118).  `payload_offset` = header + dims bytes
 * (the caller validated magic / version / kind / dims); a payload whose size is not the dims'
 * product fails with CPF_E_FORMAT and the reference's message. */
int cpf_engine_load_cptn(cpf_engine* e, const char* path, int64_t payload_offset);
/* Factors, stacked (kruskal.py:70-72).  Host memory; full (replicated) factors on every rank. */
int cpf_engine_set_factors(cpf_engine* e, const void* stacked);
int cpf_engine_get_factors(cpf_engine* e, void* stacked);

/* fit (solver.py:319-384): begin = preamble (normalise the bound factors, ||Y||, mu0, cache,
 * MTTKRPs, initial error); step = up to n_iters LM iterations (stops early at a stop condition). */
int cpf_engine_fit_begin(cpf_engine* e, int variant, double tau, double tol, int max_iters, cpf_status* st);
int cpf_engine_fit_step(cpf_engine* e, int n_iters, cpf_status* st);
int cpf_engine_trace(cpf_engine* e, cpf_iter_record* out, int cap, int* n);

/* Building blocks at the bound factors, no normalisation (kruskal.py / solver.py semantics). */
int cpf_engine_mttkrp(cpf_engine* e, int mode, void* out);            /* mode 1..N; 0 = all, stacked */
int cpf_engine_relative_error(cpf_engine* e, double* out);            /* ||Y-X||/||Y|| */
int cpf_engine_flm_step(cpf_engine* e, double mu, int variant, int refine_steps, void* cand_stacked,
                        int* err_code);

/* ALS baselines (solver.py:294-316 _fit_als; kruskal.py:257-293 als_step / als_line_search_step).
 * One step of the bound factors at iteration t (1-based): a sweep in ascending mode order, each
 * mode A_n = M_n pinv_psd(Gamma^(n))^T at the partially updated factors (one tensor read per
 * mode).  line_search != 0 (variant "als-ls") then scores A_prev + s (A_als - A_prev) for
 * s in {1.1, t^(1/3)} against the sweep by relative error and keeps the best (strictly smaller
 * wins, the sweep on ties).  The history A_prev is the iterate the previous call started from --
 * none right after cpf_engine_set_factors, so the first step is a plain sweep as in the reference
 * -- or the one given to cpf_engine_set_history (NULL clears it).  *relerr = ||Y - X|| / ||Y|| of
 * the new factors (the value _fit_als records).  Rank <= 64. */
int cpf_engine_als_step(cpf_engine* e, int line_search, int t, double* relerr);
int cpf_engine_set_history(cpf_engine* e, const void* stacked);
/* fast_damped_inverse(cache, factors, mu, use_kernel_inverse) (hessian.py:232-277) at the bound
 * factors (no tensor needed): gamma_tilde = N blocks (Gamma^(n) + mu I)^{-1} (R x R, column-major,
 * stacked) and the core grid D (N R^2 x N R^2, column-major; block (n, m) is S[n][m]), computed
 * from the same O(1)-conditioned systems as the reference (K^{-1} path: inv(Sb K~ Sb +
 * blkdiag((Gamma_n + mu I) kron C_n)); K-free path: blkdiag(Gt kron I) K inv(Sb + Chat K)) with the
 * engine's LU and triangular inverses.  use_kernel_inverse: -1 = auto (kernel_is_invertible),
 * 0 = K-free, 1 = K^{-1}.  mu <= 0 is CPF_E_ARG.  *err_code = CPF_ERR_KINV_SINGULAR (K^{-1}
 * requested, K singular), CPF_ERR_SBCK_SINGULAR (K-free system singular), CPF_ERR_SINGULAR
 * (np.linalg.inv failure) or 0. */
int cpf_engine_fast_damped_inverse(cpf_engine* e, double mu, int use_kernel_inverse, void* gamma_tilde, void* core,
                                   int* err_code);
/* pinv_psd(gamma) (kruskal.py:245-254) of a Hermitian PSD R x R matrix (column-major, lower
 * triangle read) on `device`: Jacobi eigen-decomposition, eigenvalues <= eps R max(w) dropped.
 * Host buffers in and out; R <= 64. */
int cpf_pinv_psd(int device, int kind, int R, const void* gram, void* out);

/* Per-phase device time accumulated with CUDA events on the engine stream (profiling on/off).
 * Phases: 0 pass A, 1 pass B, 2 LU factor, 3 solves, 4 other; counts = launches per phase. */
int cpf_engine_profile(cpf_engine* e, int enable);
int cpf_engine_phase_times(cpf_engine* e, double* ms_out, int64_t* counts_out, int nphases);
/* Longest single instance of each phase since profiling was last switched on (after a
 * cpf_engine_phase_times call): a complete factorisation / pass, where the per-phase totals also
 * hold instances whose kernels were gated off (rejected step, abandoned speculative branch). */
int cpf_engine_phase_max(cpf_engine* e, double* ms_out, int nphases);
/* G_n = Y_(n) Y_(n)^H (I_n x I_n, column-major) of the bound tensor, for the SVD initialisation
 * (kruskal.py:227-242).  Sharded tensors: every mode (mode N by broadcasting each slab in turn;
 * every rank returns the full matrix). */
int cpf_engine_unfolding_gram(cpf_engine* e, int mode, void* out);
/* Number of kernels this engine has launched (for the bench's gpu_launches count). */
int64_t cpf_engine_launch_count(const cpf_engine* e);
/* Tensor-pass implementation the engine planned for its tensor (diagnostic, no reference
 * counterpart): fp64/complex FMA passes, fp64 tensor-core DMMA passes, or the int8 tcgen05 passes
 * on exact digit splits (Ozaki scheme). */
#define CPF_PASS_FMA 0
#define CPF_PASS_DMMA 1
#define CPF_PASS_OZAKI 2
int cpf_engine_pass_impl(const cpf_engine* e);
/* Accuracy guard of the int8 passes (diagnostic, no reference counterpart): number of tensor-pass
 * launches since the last fit_begin whose K x R operand was outside the int8 split's accuracy
 * envelope and that therefore ran in fp64 (*out); and whether the bound tensor itself was outside
 * it (*tensor_rejected = 1: the engine planned fp64 passes for the whole tensor). */
int cpf_engine_pass_guard(cpf_engine* e, int64_t* fallbacks, int* tensor_rejected);

#ifdef __cplusplus
}
#endif
#endif /* CPFAST_B200_H_ */
