// Dense LU with partial pivoting (getrf) and the triangular solves (getrs) for the fLM core
// system Phi (phi.cuh).  The reference forms B = inv(Phi) with LAPACK getrf+getri
// (hessian.py:207) or solve(I + Psi K, I) (hessian.py:209); here Phi is factored once per
// iteration and B w is applied three times by forward/back substitution.
//
// Blocked right-looking algorithm, panel width KB:
//   1. k_panel_lu   -- one thread-block CLUSTER owns the whole m x KB panel in distributed shared
//                      memory.  Pivot search per column is a block reduction + one cluster
//                      barrier: each CTA publishes its best candidate row into every CTA's smem
//                      slot (double-buffered by column parity), so the chosen pivot row is
//                      already local everywhere.  Rows are pivoted logically (retired), then
//                      written back once in LAPACK order; the panel's row interchange is emitted
//                      as a short gather list (<= 2 KB touched positions).
//   2. k_row_gather -- applies that interchange to the columns outside the panel and to perm.
//   3. k_trsm_llnu  -- U12 = L11^{-1} A12.
//   4. k_gemm_sub   -- A22 -= L21 U12 (fp64 / complex128 tiled GEMM).
// Solves: x = P b (gather by perm), then k_trsv<lower, unit> and k_trsv<upper> -- single-kernel
// blocked substitution with per-block ready flags (decoupled look-back; CTAs take logical block
// ids from an atomic ticket so every awaited block is already running).
#pragma once
#include <cooperative_groups.h>
#include "cpf_common.cuh"

namespace cpf {
namespace cg = cooperative_groups;

constexpr int kLuMaxCluster = 16;
constexpr int kLuMaxKB = 32;

// round kb up so the int arrays keep 16-byte alignment of the reduction scratch
__host__ __device__ constexpr int kbMaxPad(int kb) { return (kb + 3) & ~3; }

struct LuWork {
  int* perm;       // n: final position -> original row
  int* ipiv;       // n: LAPACK-style swap sequence (0-based positions)
  int* gather;     // 2 * (2*KB): (pos, src) pairs of the current panel
  int* gcount;     // 1
  int* info;       // 1: first zero pivot (1-based), 0 = none
  int* ticket;     // 2 counters for the substitution kernels
  int* ready;      // ceil(n/32) flags
  int* latch = nullptr;  // speculative branch only: per-panel gate latch (panel_gated)
};

// Gate of the cluster panel kernels.  Their CTAs synchronise with each other (mbarriers, st.async
// into each other's shared memory), so all of them must take the same branch: a CTA that returned
// while a peer still waits for its packet hangs the cluster or faults.  The fork's factorisation
// only reads state that k_decide wrote before the fork started.  The speculative branch (gate 3)
// runs BESIDE the step's k_decide, which may set `stopped` / the acceptance at any moment -- two
// CTAs reading the state themselves can disagree (a ~1-in-100-fits hang / launch failure on the
// last iteration of a fit, found in round 2 by a stress loop).  So in the branch the state is read
// by ONE thread, ordered before the panel by the stream: k_lu_init latches it for panel 0, panel k
// latches it for panel k + 1 when it ends, an abandoned panel passes the latch on; the panel's
// CTAs read only the latch.  This is also what lets the branch's panels be abandoned at all.
__device__ __forceinline__ int spec_branch_dead(const LmDeviceState* st) {
  return (st->stopped || st->err_code || ld_volatile_int(&st->accept_iter) == st->spec_iter + 1) ? 1 : 0;
}
__device__ __forceinline__ bool panel_gated(const LmDeviceState* st, int gate_running, const LuWork& w, int k) {
  if (gate_running != 3) return lu_gated_sync(st, gate_running);
  if (w.latch[k]) {
    if (blockIdx.x == 0 && threadIdx.x == 0) w.latch[k + 1] = 1;
    return true;
  }
  return false;
}
__device__ __forceinline__ void panel_latch_next(const LmDeviceState* st, int gate_running, const LuWork& w, int k) {
  if (gate_running == 3 && blockIdx.x == 0 && threadIdx.x == 0) w.latch[k + 1] = spec_branch_dead(st);
}

__global__ void k_lu_init(int* perm, int n, int* info, const LmDeviceState* st, int* latch, int gate_running) {
  pdl_wait();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 && latch) latch[0] = spec_branch_dead(st);  // speculative branch: panel_gated
  // a gated factorisation leaves the permutation alone: after a rho <= 0 rejection it is the
  // speculated system's, copied in at the start of the replay unit
  if (lu_gated(st, gate_running)) return;
  if (i < n) perm[i] = i;
  if (i == 0) *info = 0;
}

template <class T>
__global__ void __launch_bounds__(256) k_panel_lu(T* __restrict__ A, int n, int lda, int k0, int kb, int rpc, LuWork w,
                                                  const LmDeviceState* st, int gate_running) {
  pdl_wait();
  if (lu_gated_sync(st, gate_running)) return;
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  constexpr int NW = 8;  // warps per CTA (blockDim 256)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // layout: panel [rpc x kb] T | cand_data [2][CL*NW][kb] T | top [kb][kb] T | cand_val [2][CL*NW] double |
  //         cand_row [2][CL*NW] int | retired/pos [rpc] int | pivrows [kb] int
  const int NC = CL * NW;
  T* pan = reinterpret_cast<T*>(smem_raw);
  T* cand_data = pan + (size_t)rpc * kb;
  T* top = cand_data + (size_t)2 * NC * kb;
  double* cand_val = reinterpret_cast<double*>(top + (size_t)kb * kb);
  int* cand_row = reinterpret_cast<int*>(cand_val + 2 * NC);
  int* retired = cand_row + 2 * NC;
  int* pivrows = retired + rpc;

  const int m = n - k0;
  const int row0 = rank * rpc;
  const int rows_here = max(0, min(rpc, m - row0));
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5;

  for (int e = tid; e < rpc * kb; e += nthr) {
    int i = e % rpc, q = e / rpc;
    pan[e] = (i < rows_here) ? A[(int64_t)(k0 + row0 + i) + (int64_t)lda * (k0 + q)] : zero_of<T>();
  }
  for (int i = tid; i < rpc; i += nthr) retired[i] = (i < rows_here) ? 0 : 1;
  __syncthreads();

  for (int jj = 0; jj < kb; ++jj) {
    const int par = jj & 1;
    // ---- warp-local argmax over my non-retired rows (ties -> smaller row)
    double bv = -1.0;
    int bi = -1;
    for (int i = tid; i < rows_here; i += nthr) {
      if (retired[i]) continue;
      const double v = pivmag(pan[i + rpc * jj]);
      if (v > bv) { bv = v; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi >= 0 && (bi < 0 || oi < bi))) { bv = ov; bi = oi; }
    }
    // ---- publish this warp's candidate (value, row, row data) into every CTA of the cluster
    const int slot = par * NC + rank * NW + wid;
    for (int r = 0; r < CL; ++r) {
      if (lane < kb) {
        T* rd = cluster.map_shared_rank(cand_data, r);
        rd[(size_t)slot * kb + lane] = (bi >= 0) ? pan[bi + rpc * lane] : zero_of<T>();
      }
      if (lane == 0) {
        cluster.map_shared_rank(cand_val, r)[slot] = bv;
        cluster.map_shared_rank(cand_row, r)[slot] = (bi >= 0) ? (k0 + row0 + bi) : 0x7fffffff;
      }
    }
    cluster.sync();
    // ---- winner (identical in every thread of every CTA)
    int win = par * NC;
    {
      double b = cand_val[win];
      int rw = cand_row[win];
      for (int q = 1; q < NC; ++q) {
        const double v = cand_val[par * NC + q];
        const int rr = cand_row[par * NC + q];
        if (v > b || (v == b && rr < rw)) { b = v; rw = rr; win = par * NC + q; }
      }
    }
    const int wrow = cand_row[win];
    const T* prow = cand_data + (size_t)win * kb;
    const T piv = prow[jj];
    const bool zero_piv = (pivmag(piv) == 0.0);
    if (tid == 0) pivrows[jj] = wrow;
    if (tid < kb) top[jj * kb + tid] = prow[tid];   // top block row jj (L part | U part)
    if (zero_piv && rank == 0 && tid == 0 && *w.info == 0) *w.info = k0 + jj + 1;
    const int wl = wrow - k0 - row0;
    // ---- eliminate in my rows
    for (int i = tid; i < rows_here; i += nthr) {
      if (retired[i]) continue;
      if (i == wl) { retired[i] = 1; continue; }
      if (zero_piv) continue;
      const T l = dvd(pan[i + rpc * jj], piv);
      pan[i + rpc * jj] = l;
      for (int q = jj + 1; q < kb; ++q) fms_acc(pan[i + rpc * q], l, prow[q]);
    }
  }
  __syncthreads();

  // ---- row interchange of this panel.  Any row order below the pivots is a valid P (rows move
  // with their multipliers), so: position k0+jj <- pivot row jj; the displaced non-pivot rows of
  // the top block D (ascending) take the vacated positions V of pivot rows from below (pick order).
  __shared__ int Dl[kLuMaxKB], Vl[kLuMaxKB];
  __shared__ int nd_s;
  if (wid == 0) {
    const bool live = lane < kb;
    const int toprow = k0 + lane;
    bool top_is_piv = false;
    for (int q = 0; q < kb; ++q) top_is_piv |= (pivrows[q] == toprow);
    const unsigned dmask = __ballot_sync(0xffffffffu, live && !top_is_piv);
    const unsigned vmask = __ballot_sync(0xffffffffu, live && pivrows[live ? lane : 0] >= k0 + kb);
    if (live && !top_is_piv) Dl[__popc(dmask & ((1u << lane) - 1u))] = toprow;
    if (live && pivrows[lane] >= k0 + kb) Vl[__popc(vmask & ((1u << lane) - 1u))] = pivrows[lane];
    if (lane == 0) nd_s = __popc(dmask);
  }
  __syncthreads();
  const int nd = nd_s;
  for (int i = tid; i < rows_here; i += nthr) {
    const int o = k0 + row0 + i;
    int pos = o;
    bool piv_any = false;
    for (int q = 0; q < kb; ++q)
      if (pivrows[q] == o) { pos = k0 + q; piv_any = true; }
    if (!piv_any && o < k0 + kb)
      for (int d = 0; d < nd; ++d)
        if (Dl[d] == o) pos = Vl[d];
    retired[i] = pos;
  }
  if (rank == 0 && wid == 0) {
    int g = 0;
    for (int q = 0; q < kb; ++q) {
      if (pivrows[q] != k0 + q) {
        if (lane == 0) { w.gather[2 * g] = k0 + q; w.gather[2 * g + 1] = pivrows[q]; }
        ++g;
      }
    }
    for (int d = 0; d < nd; ++d) {
      if (lane == 0) { w.gather[2 * g] = Vl[d]; w.gather[2 * g + 1] = Dl[d]; }
      ++g;
    }
    if (lane == 0) *w.gcount = g;
  }
  __syncthreads();
  for (int e = tid; e < rows_here * kb; e += nthr) {
    const int i = e % rows_here, q = e / rows_here;
    A[(int64_t)retired[i] + (int64_t)lda * (k0 + q)] = pan[i + rpc * q];
  }
  cluster.sync();  // keep DSMEM alive until every CTA is done with remote slots
}

template <class T>
size_t panel_smem_bytes(int rpc, int kb, int CL) {
  const size_t NC = (size_t)CL * 8;
  size_t b = sizeof(T) * ((size_t)rpc * kb + 2 * NC * kb + (size_t)kb * kb);
  b += sizeof(double) * 2 * NC + sizeof(int) * 2 * NC + sizeof(int) * rpc + sizeof(int) * kbMaxPad(kb);
  return (b + 15) & ~(size_t)15;
}

// Apply the panel's row gather (pos <- src) to columns [0,k0) U [k0+kb, n) and to perm.
// Block: CB columns x G entries; first read all sources, barrier, then write.
template <class T>
__global__ void k_row_gather(T* __restrict__ A, int n, int lda, int k0, int kb, LuWork w, const LmDeviceState* st,
                             int gate_running) {
  pdl_wait();
  if (lu_gated(st, gate_running)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int G = *w.gcount;
  if (G == 0) return;
  T* buf = reinterpret_cast<T*>(smem_raw);
  __shared__ int pbuf[2 * kLuMaxKB];
  const int ncols_out = n - kb;  // columns outside the panel
  const int cb = blockDim.x / (2 * kLuMaxKB);
  const int col_first = blockIdx.x * cb;
  const int e = threadIdx.x % (2 * kLuMaxKB);
  const int cl = threadIdx.x / (2 * kLuMaxKB);
  const int cidx = col_first + cl;
  // the last block also fixes perm (virtual column index ncols_out)
  const bool do_col = (cidx < ncols_out) && (e < G);
  int col = -1;
  if (cidx < ncols_out) col = (cidx < k0) ? cidx : cidx + kb;
  T v = zero_of<T>();
  if (do_col) v = A[(int64_t)w.gather[2 * e + 1] + (int64_t)lda * col];
  const bool do_perm = (blockIdx.x == 0) && (cl == 0) && (e < G);
  int pv = 0;
  if (do_perm) pv = w.perm[w.gather[2 * e + 1]];
  buf[threadIdx.x] = v;
  if (do_perm) pbuf[e] = pv;
  __syncthreads();
  if (do_col) A[(int64_t)w.gather[2 * e] + (int64_t)lda * col] = buf[threadIdx.x];
  if (do_perm) w.perm[w.gather[2 * e]] = pbuf[e];
}

// Row interchange restricted to the column ranges [ca0, ca1) U [cb0, cb1) (+ perm when do_perm):
// the look-ahead LU applies it to the next block on one stream and to everything else on another.
template <class T>
__global__ void k_row_gather2(T* __restrict__ A, int lda, const int* __restrict__ gather, const int* __restrict__ gcount,
                              int* __restrict__ perm, int ca0, int ca1, int cb0, int cb1, int do_perm,
                              const LmDeviceState* st, int gate_running) {
  pdl_wait();
  if (lu_gated(st, gate_running)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int G = *gcount;
  if (G == 0) return;
  T* buf = reinterpret_cast<T*>(smem_raw);
  __shared__ int pbuf[2 * kLuMaxKB];
  const int na = max(0, ca1 - ca0), nb = max(0, cb1 - cb0);
  const int cb = blockDim.x / (2 * kLuMaxKB);
  const int e = threadIdx.x % (2 * kLuMaxKB);
  const int cl = threadIdx.x / (2 * kLuMaxKB);
  const int cidx = blockIdx.x * cb + cl;
  int col = -1;
  if (cidx < na) col = ca0 + cidx;
  else if (cidx < na + nb) col = cb0 + (cidx - na);
  const bool do_col = (col >= 0) && (e < G);
  T v = zero_of<T>();
  if (do_col) v = A[(int64_t)gather[2 * e + 1] + (int64_t)lda * col];
  const bool dp = do_perm && (blockIdx.x == 0) && (cl == 0) && (e < G);
  int pv = 0;
  if (dp) pv = perm[gather[2 * e + 1]];
  buf[threadIdx.x] = v;
  if (dp) pbuf[e] = pv;
  __syncthreads();
  if (do_col) A[(int64_t)gather[2 * e] + (int64_t)lda * col] = buf[threadIdx.x];
  if (dp) perm[gather[2 * e]] = pbuf[e];
}

// U12 = L11^{-1} A12 (L11 unit lower, kb x kb); one thread per column of A12.
template <class T, int KB>
__global__ void k_trsm_llnu(T* __restrict__ A, int n, int lda, int k0, int kb, const LmDeviceState* st,
                            int gate_running) {
  pdl_wait();
  if (lu_gated(st, gate_running)) return;
  __shared__ T L[KB * KB];
  for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
    int i = e % kb, j = e / kb;
    L[i + KB * j] = A[(int64_t)(k0 + i) + (int64_t)lda * (k0 + j)];
  }
  __syncthreads();
  const int col = k0 + kb + blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= n) return;
  T x[KB];
  T* a = A + (int64_t)lda * col + k0;
#pragma unroll
  for (int i = 0; i < KB; ++i) x[i] = (i < kb) ? a[i] : zero_of<T>();
#pragma unroll
  for (int j = 0; j < KB; ++j) {
    if (j >= kb) break;
#pragma unroll
    for (int i = j + 1; i < KB; ++i)
      if (i < kb) fms_acc(x[i], L[i + KB * j], x[j]);
  }
#pragma unroll
  for (int i = 0; i < KB; ++i)
    if (i < kb) a[i] = x[i];
}

// C -= A * B   (column-major; C: m x nn at (r0, c0); A = L21: m x k at (r0, k0); B = U12: k x nn at (k0, c0))
// 64 x 64 tile, 256 threads, 4 x 4 outputs per thread (strided by 16 for conflict-free smem).
template <class T>
__global__ void __launch_bounds__(256) k_gemm_sub(T* __restrict__ Mx, int lda, int r0, int c0, int k0, int m, int nn,
                                                  int k, const LmDeviceState* st, int gate_running) {
  pdl_wait();
  if (lu_gated(st, gate_running)) return;
  constexpr int TM = 64, TN = 64, BK = 16;
  __shared__ T As[BK][TM + 1];
  __shared__ T Bs[BK][TN + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int bm = blockIdx.x * TM, bn = blockIdx.y * TN;
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = zero_of<T>();
  for (int kk = 0; kk < k; kk += BK) {
    // load A tile: TM x BK  (rows bm.., cols kk..)
    for (int e = threadIdx.x; e < TM * BK; e += 256) {
      int i = e % TM, q = e / TM;
      int gi = bm + i, gq = kk + q;
      As[q][i] = (gi < m && gq < k) ? Mx[(int64_t)(r0 + gi) + (int64_t)lda * (k0 + gq)] : zero_of<T>();
    }
    for (int e = threadIdx.x; e < TN * BK; e += 256) {
      int q = e % BK, j = e / BK;
      int gj = bn + j, gq = kk + q;
      Bs[q][j] = (gj < nn && gq < k) ? Mx[(int64_t)(k0 + gq) + (int64_t)lda * (c0 + gj)] : zero_of<T>();
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < BK; ++q) {
      T a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[q][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[q][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) fma_acc(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gi = bm + ty + 16 * i, gj = bn + tx + 16 * j;
      if (gi < m && gj < nn) {
        T* c = Mx + (int64_t)(r0 + gi) + (int64_t)lda * (c0 + gj);
        *c = sub(*c, acc[i][j]);
      }
    }
}

// LU info -> engine error code (flm-a singular maps to the "I + Psi K" message)
__global__ void k_lu_info_to_err(const int* info, LmDeviceState* st) {
  pdl_wait();
  if (st->stopped || st->err_code) return;
  if (*info != 0) st->err_code = st->use_kinv ? kErrSingular : kErrPhi1Singular;
}

// x[q] = b[perm[q]]
template <class T>
__global__ void k_perm_gather(const T* __restrict__ b, const int* __restrict__ perm, int n, T* __restrict__ x,
                              const LmDeviceState* st, int gate_running) {
  pdl_wait();
  if (lu_gated(st, gate_running)) return;
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) x[q] = b[perm[q]];
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// spin with relaxed loads (no L1 invalidation per poll), then one acquire load
__device__ __forceinline__ void wait_flag(const int* p, int v) {
  while (ld_relaxed_gpu(p) != v) {
  }
  (void)ld_acquire_gpu(p);
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// In-place triangular solve on x (length n) with the LU factors in A.
// LOWER: unit lower, forward.  !LOWER: upper (non-unit), backward.
// Block = 4 warps; 32 rows per logical block.  ready[] holds the epoch of the last completion.
// Every 32x32 tile a warp needs is prefetched into registers before it waits on the producing
// block's flag, so the critical path per block is: flag -> 32 shuffles+FMAs -> 32-step diagonal
// solve from registers -> flag.
template <class T>
__device__ __forceinline__ void load_tile_col(const T* __restrict__ A, int lda, int row, bool rv, int c0, int cols,
                                              T (&t)[32]) {
#pragma unroll
  for (int c = 0; c < 32; ++c) t[c] = (rv && c < cols) ? A[(int64_t)row + (int64_t)lda * (c0 + c)] : zero_of<T>();
}

template <class T, bool LOWER>
__global__ void __launch_bounds__(128) k_trsv(const T* __restrict__ A, int n, int lda, T* __restrict__ x,
                                              int* __restrict__ ticket, int* __restrict__ ready, int epoch,
                                              const LmDeviceState* st, int gate_running) {
  pdl_wait();
  if (lu_gated_sync(st, gate_running)) return;
  __shared__ int s_b;
  __shared__ T part[4][32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_b = atomicAdd(ticket, 1);
  __syncthreads();
  const int nblk = (n + 31) / 32;
  const int lb = s_b;
  const int blk = LOWER ? lb : (nblk - 1 - lb);
  const int r0 = blk * 32;
  const int rows = min(32, n - r0);
  const int row = r0 + lane;
  const bool rv = row < n;
  // prefetch (off the critical path): the diagonal tile and this block's right-hand side
  T dg[32];
  T v0 = zero_of<T>();
  if (wid == 0) {
    load_tile_col(A, lda, row, rv, r0, rows, dg);
    v0 = rv ? ld_cg(x + row) : zero_of<T>();
  }
  T acc = zero_of<T>();
  {
    T cur[32], nxt[32];
    int q = wid;
    if (q < lb) {
      const int kb0 = LOWER ? q : (nblk - 1 - q);
      load_tile_col(A, lda, row, rv, kb0 * 32, min(32, n - kb0 * 32), cur);
    }
    while (q < lb) {
      const int kblk = LOWER ? q : (nblk - 1 - q);
      const int c0 = kblk * 32;
      const int cols = min(32, n - c0);
      const int qn = q + 4;
      if (qn < lb) {
        const int kbn = LOWER ? qn : (nblk - 1 - qn);
        load_tile_col(A, lda, row, rv, kbn * 32, min(32, n - kbn * 32), nxt);
      }
      if (lane == 0) wait_flag(ready + kblk, epoch);
      __syncwarp();
      const T xv = (lane < cols) ? ld_cg(x + c0 + lane) : zero_of<T>();
#pragma unroll
      for (int c = 0; c < 32; ++c) fms_acc(acc, cur[c], shfl_idx(xv, c));
#pragma unroll
      for (int c = 0; c < 32; ++c) cur[c] = nxt[c];
      q = qn;
    }
  }
  part[wid][lane] = acc;
  __syncthreads();
  if (wid == 0) {
    T v = add(v0, add(add(part[0][lane], part[1][lane]), add(part[2][lane], part[3][lane])));
    if (LOWER) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const T yj = shfl_idx(v, j);
        if (lane > j && j < rows) fms_acc(v, dg[j], yj);
      }
    } else {
#pragma unroll
      for (int j = 31; j >= 0; --j) {
        if (lane == j && j < rows) v = dvd(v, dg[j]);
        const T yj = shfl_idx(v, j);
        if (lane < j && j < rows) fms_acc(v, dg[j], yj);
      }
    }
    if (lane < rows) x[row] = v;
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release_gpu(ready + blk, epoch);
  }
}

}  // namespace cpf
