// LU v5: the whole partial-pivoting LU of the core system Phi in ONE persistent kernel.
//
// Why: the fLM step's LU of the NR^2 x NR^2 core system (config 4: 1200 x 1200) is a chain of
// pivot decisions, bound by latency, not flops (1.15 GF).  The v4 path (lu4.cuh) factors 32-column
// panels on a 2-3 CTA cluster -- one cluster-wide pivot exchange per column (~2350 cycles) and a
// kernel launch per panel (38 launches + the trailing-update kernels).  Here:
//
//  * CTA 0 (the panel CTA) owns every row of the matrix in REGISTERS (RPT rows per thread, row
//    phys = tid + j * NT) and factors 16-column panels: per column a warp argmax, one
//    __syncthreads and a CTA argmax -- no cluster exchange.  Rows are pivoted LOGICALLY (never
//    moved while factoring): each thread tracks the LAPACK position of its rows, so the pivot
//    choice (max |a|, |re|+|im| for complex, ties to the smaller position) is exactly getrf's.
//  * CTAs 1..H (helpers) do the trailing updates: after panel k is published, every helper
//    updates its share of the rows of block k+1 (the look-ahead block the panel needs next) and
//    signals; then each helper updates the blocks it owns (block-cyclic) for all rows.  U12 of a
//    block is formed by substitution with L11 (as LAPACK's trsm), A22 -= L21 U12 on the FMA pipe.
//  * Synchronisation is by flags in global memory (release / acquire) between CTAs of this one
//    kernel -- no kernel waits on another kernel.  Every wait ends with an acquire fence (which
//    invalidates the SM's L1), and between two waits a CTA only reads data no other CTA writes
//    meanwhile, so the matrix is read with plain (L1-cacheable, freely reordered) loads.  The grid is at most the SMs the fork leaves to
//    the LU (kLuReserveSms), so every CTA is resident next to the persistent pass B.
//  * At the end the rows are gathered into LAPACK order (perm) and copied back, so Phi holds the
//    standard packed LU (unit L below, U on/above) for tri_inv.cuh and the substitutions.
#pragma once
#include "cpf_common.cuh"
#include "lu.cuh"
#include "lu3.cuh"

namespace cpf {

constexpr int kLpKB = 16;  // panel width

struct LuPersist {
  int n, np, nhelp;
  int* panel_done;   // [np]  1 once panel k is published
  int* block_ready;  // [np]  helpers done with the look-ahead rows of block k
  int* blk_done;     // [np]  1 + last step the owner applied to block k
  int* ret;          // [n]   step at which a physical row became a pivot (INT_MAX: alive)
  int* piv;          // [np * KB] pivot physical rows of each step
  int* bar;          // [4]   grid barriers of the final phase
  int* perm;         // [n]   LAPACK order: perm[q] = physical row of position q
  int* info;         // first zero pivot (1-based), 0 = none
  void* u12s;        // [np * KB * KB] U12 of each step's look-ahead block (written in the final phase)
  void* tmp;         // n x n scratch for the final gather
};

__device__ __forceinline__ int lp_ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void lp_st_rel(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void lp_red_rel(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int lp_ld_rlx(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// thread 0 polls (relaxed loads: an acquire per poll would invalidate L1 every time) until
// *p >= v, then one acquire fence; the CTA proceeds
__device__ __forceinline__ void lp_wait_geq(const int* p, int v) {
  if (threadIdx.x == 0) {
    while (lp_ld_rlx(p) < v) __nanosleep(16);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
__device__ __forceinline__ void lp_grid_barrier(int* ctr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    lp_red_rel(ctr, 1);
    while (lp_ld_rlx(ctr) < (int)gridDim.x) __nanosleep(16);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

__global__ void k_lp_init(LuPersist p) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < p.n) p.ret[i] = 0x7fffffff;
  if (i < p.np) { p.panel_done[i] = 0; p.block_ready[i] = 0; p.blk_done[i] = 0; }
  if (i < 4) p.bar[i] = 0;
  if (i == 0) *p.info = 0;
}

// U12 (kb x w) = L11^{-1} A12 by substitution (LAPACK trsm order: right-looking over the pivot
// columns).  Warp wq solves columns 2 wq, 2 wq + 1; lane = row + 16 * (column parity): each step
// broadcasts x_c with one shuffle and updates the rows below -- no block barrier, no serial
// dependent sum.  L11 unit lower and A12 / U12 in smem ([i][q], ld KB); result in place.
template <class T>
__device__ __forceinline__ void lp_trsm16(const T (*L)[kLpKB], T (*X)[kLpKB], int kb, int w) {
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int i = lane & 15, q = 2 * wq + (lane >> 4);
  if (wq < kLpKB / 2) {
    T x = X[i][q];
    for (int c = 0; c + 1 < kb; ++c) {
      const T xc = shfl_val(x, (lane & 16) + c);
      if (i > c) fms_acc(x, L[i][c], xc);
    }
    __syncwarp();
    if (q < w) X[i][q] = x;
  }
}

// Helper dynamic shared memory: a copy of the rows' retirement steps (ret).
template <class T>
__host__ __device__ constexpr size_t lp_smem_bytes(int n) {
  return (size_t)n * sizeof(int);
}

template <class T, int NT, int RPT>
__global__ void __launch_bounds__(NT, 1) k_lu_persist(T* A, LuPersist p, const LmDeviceState* st,
                                                      int gate_running) {
  pdl_wait();
  if (lu_gated_sync(st, gate_running)) return;
  constexpr int KB = kLpKB, NW = NT / 32;
  const int n = p.n, np = p.np;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  __shared__ __align__(16) T Ls[KB][KB];   // L11 of the current step (helpers)
  __shared__ __align__(16) T Us[KB][KB];   // U12 work tile
  __shared__ int piv_s[KB];
  extern __shared__ __align__(16) unsigned char lp_smem[];

  if (blockIdx.x == 0) {
    // ======================================= panel CTA =======================================
    __shared__ __align__(16) T wrow_s[2][NW][KB];
    __shared__ double wkey_v[2][NW];
    __shared__ int wkey_p[2][NW], wkey_r[2][NW];
    // diagnostic per-segment cycle totals of warp 0 (cpf_debug_lu_trace on): 0 wait, 1 load,
    // 2 my argmax + stage, 3 barrier, 4 CTA argmax + bookkeeping, 5 elimination, 6 chunk flush,
    // 7 publish
    const bool tr = g_lu_trace_on && tid == 0;
    long long tc = tr ? clock64() : 0;
    auto seg = [&](int i) {
      if (tr) { const long long t = clock64(); atomicAdd((unsigned long long*)&g_panel_cycles[i], (unsigned long long)(t - tc)); tc = t; }
    };
    int phys[RPT], pos[RPT];
    bool alive[RPT];
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      phys[j] = tid + j * NT;
      alive[j] = phys[j] < n;
      pos[j] = phys[j];
    }
#pragma unroll 1
    for (int k = 0; k < np; ++k) {
      const int k0 = k * KB, kb = min(KB, n - k0);
      lu_trace(0, k, 0);
      seg(7);
      if (k > 0) lp_wait_geq(p.block_ready + k, p.nhelp);
      seg(0);
      T a[RPT][KB];
      bool live0[RPT];
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        live0[j] = alive[j];
#pragma unroll
        for (int q = 0; q < KB; ++q)
          a[j][q] = (alive[j] && q < kb) ? (*(A + (int64_t)phys[j] + (int64_t)n * (k0 + q))) : zero_of<T>();
      }
      lu_trace(1, k, 0);
      seg(1);
      // Column loop in chunks of CH columns: inside a chunk the CH columns are unrolled, so the
      // pivot column and the elimination range are static register indices of a FRAME (frame
      // column f = panel column c4 + f); at the chunk end its CH finished columns go to global
      // memory and the frame shifts left by CH.  Small code (instruction cache), no dynamic
      // register indexing.
      constexpr int CH = 4;
#pragma unroll 1
      for (int c4 = 0; c4 < kb; c4 += CH) {
#pragma unroll
        for (int u = 0; u < CH; ++u) {
          const int jj = c4 + u;
          if (jj >= kb) break;
          const int par = jj & 1;
          double bv = 0.0;
          int bp = 0x7fffffff, bj = 0;
#pragma unroll
          for (int j = 0; j < RPT; ++j) {
            if (!alive[j]) continue;
            const double v = pivmag(a[j][u]);
            if (bp == 0x7fffffff || v > bv || (v == bv && pos[j] < bp)) { bv = v; bp = pos[j]; bj = j; }
          }
          double wv;
          int wpos, wlane;
          warp_argmax_redux(bv, bp, wv, wpos, wlane);
          if (lane == wlane) {  // one lane: a divergent switch stores just the winning row
            T* dst = &wrow_s[par][wid][0];
#pragma unroll
            for (int j = 0; j < RPT; ++j)
              if (bj == j) {
#pragma unroll
                for (int f = 0; f < KB; ++f) dst[f] = a[j][f];
                wkey_r[par][wid] = phys[j];
              }
            wkey_v[par][wid] = wv;
            wkey_p[par][wid] = wpos;
          }
          seg(2);
          __syncthreads();
          seg(3);
          double gv;
          int gpos, gw;
          {
            const double kv = lane < NW ? wkey_v[par][lane] : 0.0;
            const int kp = lane < NW ? wkey_p[par][lane] : 0x7fffffff;
            warp_argmax_redux(kv, kp, gv, gpos, gw);
          }
          const T* prow = &wrow_s[par][gw][0];
          const int gphys = wkey_r[par][gw];
          const bool zero_piv = (gv == 0.0);
          const T rcp = zero_piv ? zero_of<T>() : rcp_of(prow[u]);
          if (tid == 0) {
            piv_s[jj] = gphys;
            p.perm[k0 + jj] = gphys;
            if (zero_piv && *p.info == 0) *p.info = k0 + jj + 1;
          }
#pragma unroll
          for (int j = 0; j < RPT; ++j) {
            if (!alive[j]) continue;
            if (phys[j] == gphys) {  // the pivot row retires at LAPACK position k0 + jj
              alive[j] = false;
              pos[j] = k0 + jj;
            } else if (pos[j] == k0 + jj) {  // the row displaced by the interchange
              pos[j] = gpos;
            }
          }
          seg(4);
          T l[RPT];
#pragma unroll
          for (int j = 0; j < RPT; ++j) l[j] = (alive[j] && !zero_piv) ? mul(a[j][u], rcp) : zero_of<T>();
#pragma unroll
          for (int f = u + 1; f < KB; ++f) {
            const T pv = prow[f];
#pragma unroll
            for (int j = 0; j < RPT; ++j) fms_acc(a[j][f], l[j], pv);
          }
#pragma unroll
          for (int j = 0; j < RPT; ++j)
            if (alive[j] && !zero_piv) a[j][u] = l[j];
          seg(5);
        }
        // chunk end: the CH finished columns are final -> global; shift the frame
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
          if (live0[j]) {
#pragma unroll
            for (int f = 0; f < CH; ++f)
              if (c4 + f < kb) A[(int64_t)phys[j] + (int64_t)n * (k0 + c4 + f)] = a[j][f];
          }
#pragma unroll
          for (int f = 0; f < KB - CH; ++f) a[j][f] = a[j][f + CH];
#pragma unroll
          for (int f = KB - CH; f < KB; ++f) a[j][f] = zero_of<T>();
        }
        seg(6);
      }
      lu_trace(1, k, 1);
      // publish (the panel's columns are in place: L multipliers / pivot rows' L11 | U11)
      if (tid < kb) {
        p.piv[k * KB + tid] = piv_s[tid];
        p.ret[piv_s[tid]] = k;
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) lp_st_rel(p.panel_done + k, 1);
      lu_trace(0, k, 1);
    }
  } else {
    // ====================================== helper CTAs ======================================
    // per step: (A) this helper's slice of the rows of the look-ahead block k+1, signalled; (B) the
    // blocks c >= k+2 it owns (block-cyclic), all alive rows, U12 written into the pivot rows.
    // Alive rows: a shared-memory copy of ret, updated from each step's pivots.
    const int h = blockIdx.x - 1, H = p.nhelp;
    int* ret_s = reinterpret_cast<int*>(lp_smem);
    for (int r = tid; r < n; r += NT) ret_s[r] = 0x7fffffff;
    T* u12s = static_cast<T*>(p.u12s);
    const int r0 = (int)((int64_t)n * h / H), r1 = (int)((int64_t)n * (h + 1) / H);
    // diagnostic cycle totals of helper 0's thread 0 (g_panel_seg): 0 wait panel, 1 setup,
    // 2 wait owner, 3 U12 (A), 4 update (A), 5 fence+signal (A), 6 U12+store (B), 7 update (B),
    // 8 fence+signal (B)
    const bool tr = g_lu_trace_on && tid == 0 && h == 0;
    long long tc = tr ? clock64() : 0;
    auto seg = [&](int i) {
      if (tr) { const long long t = clock64(); atomicAdd((unsigned long long*)&g_panel_seg[i], (unsigned long long)(t - tc)); tc = t; }
    };
#pragma unroll 1
    for (int k = 0; k + 1 < np; ++k) {
      const int k0 = k * KB, kb = min(KB, n - k0);
      lp_wait_geq(p.panel_done + k, 1);
      seg(0);
      lu_trace(2, k, 0);
      if (tid < kb) {
        const int pr_ = (*(p.piv + k * KB + tid));
        piv_s[tid] = pr_;
        ret_s[pr_] = k;
      }
      __syncthreads();
      for (int e = tid; e < KB * KB; e += NT) {
        const int i = e / KB, c = e % KB;
        Ls[i][c] = (i < kb && c < kb) ? (*(A + (int64_t)piv_s[i] + (int64_t)n * (k0 + c))) : zero_of<T>();
      }
      auto form_u12 = [&](int c0, int w) {
        for (int e = tid; e < KB * KB; e += NT) {
          const int i = e / KB, q = e % KB;
          Us[i][q] = (i < kb && q < w) ? (*(A + (int64_t)piv_s[i] + (int64_t)n * (c0 + q))) : zero_of<T>();
        }
        __syncthreads();
        lp_trsm16<T>(Ls, Us, kb, w);
        __syncthreads();
      };
      {  // (A) look-ahead block k+1, rows [r0, r1): one thread per (row, column)
        const int c0 = (k + 1) * KB, w = min(KB, n - c0);
        seg(1);
        if (k > 0) lp_wait_geq(p.blk_done + k + 1, k);  // its owner applied step k-1
        seg(2);
        form_u12(c0, w);
        seg(3);
        if (h == 0)
          for (int e = tid; e < KB * KB; e += NT) u12s[(size_t)k * KB * KB + e] = (&Us[0][0])[e];
        const int nr = r1 - r0;
        for (int e = tid; e < ((nr + 31) & ~31) * KB; e += NT) {
          const int r = r0 + ((e >> 9) << 5) + (e & 31), q = (e >> 5) & (KB - 1);
          if (r >= r1 || q >= w || ret_s[r] <= k) continue;
          T* dst = A + (int64_t)r + (int64_t)n * (c0 + q);
          T v = (*(dst));
#pragma unroll
          for (int pp = 0; pp < KB; ++pp)
            if (pp < kb) fms_acc(v, (*(A + (int64_t)r + (int64_t)n * (k0 + pp))), Us[pp][q]);
          *dst = v;
        }
        seg(4);
        __threadfence();
        __syncthreads();
        if (tid == 0) lp_red_rel(p.block_ready + k + 1, 1);
        seg(5);
        lu_trace(2, k, 1);
      }
      // (B) owned blocks c >= k+2: one thread per row, all KB columns
      for (int c = k + 2 + ((h - (k + 2)) % H + H) % H; c < np; c += H) {
        const int c0 = c * KB, w = min(KB, n - c0);
        form_u12(c0, w);
        for (int e = tid; e < KB * KB; e += NT) {
          const int i = e / KB, q = e % KB;
          if (i < kb && q < w) A[(int64_t)piv_s[i] + (int64_t)n * (c0 + q)] = Us[i][q];
        }
        seg(6);
        for (int r = tid; r < n; r += NT) {
          if (ret_s[r] <= k) continue;
          T l[KB], v[KB];
#pragma unroll
          for (int pp = 0; pp < KB; ++pp) l[pp] = pp < kb ? (*(A + (int64_t)r + (int64_t)n * (k0 + pp))) : zero_of<T>();
#pragma unroll
          for (int q = 0; q < KB; ++q) v[q] = q < w ? (*(A + (int64_t)r + (int64_t)n * (c0 + q))) : zero_of<T>();
#pragma unroll
          for (int pp = 0; pp < KB; ++pp)
#pragma unroll
            for (int q = 0; q < KB; ++q) fms_acc(v[q], l[pp], Us[pp][q]);
#pragma unroll
          for (int q = 0; q < KB; ++q)
            if (q < w) A[(int64_t)r + (int64_t)n * (c0 + q)] = v[q];
        }
        seg(7);
        __threadfence();
        __syncthreads();
        if (tid == 0) lp_st_rel(p.blk_done + c, k + 1);
        seg(8);
      }
    }
  }
  // ================================ final phase: every CTA ================================
  // the look-ahead blocks' U12 into the pivot rows, then the rows into LAPACK order (perm)
  lp_grid_barrier(p.bar + 0);
  const int64_t gtid = (int64_t)blockIdx.x * NT + tid, gstride = (int64_t)gridDim.x * NT;
  const T* u12c = static_cast<const T*>(p.u12s);
  for (int64_t e = gtid; e < (int64_t)(np - 1) * KB * KB; e += gstride) {
    const int k = (int)(e / (KB * KB)), i = (int)(e % (KB * KB)) / KB, q = (int)(e % KB);
    const int c0 = (k + 1) * KB;
    if (k * KB + i < n && c0 + q < n)
      A[(int64_t)(*(p.piv + k * KB + i)) + (int64_t)n * (c0 + q)] = (*(u12c + e));
  }
  lp_grid_barrier(p.bar + 1);
  T* tmp = static_cast<T*>(p.tmp);
  for (int64_t e = gtid; e < (int64_t)n * n; e += gstride) {
    const int64_t q = e % n, c = e / n;
    tmp[e] = (*(A + (int64_t)ld_cg(p.perm + q) + (int64_t)n * c));
  }
  lp_grid_barrier(p.bar + 2);
  for (int64_t e = gtid; e < (int64_t)n * n; e += gstride) A[e] = (*(tmp + e));
}

}  // namespace cpf
