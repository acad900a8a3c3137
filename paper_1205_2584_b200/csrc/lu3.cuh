// LU v3 building blocks (see lu.cuh for the algorithm outline and the solves).
//
// k_panel_lu3: the m x KB panel lives in REGISTERS: a thread-block cluster of CL CTAs x NTHR
// threads, each thread owning RPT rows (KB values each).  Per column: warp argmax -> CTA argmax
// (one __syncthreads) -> the CTA's candidate packet (row, |pivot|, row index, 1/pivot) is pushed
// into every CTA's shared memory with st.async, each 16-byte store completing tx-bytes on the
// receiver's mbarrier -> every CTA waits on its OWN mbarrier (no cluster barrier: cluster.sync
// costs a GPU-scope fence + L1 invalidate per column) -> winner among the CL packets -> rank-1
// elimination of the thread's own rows in registers.  Pivot rows are pivoted logically (retired) and written
// once at the end; the panel's interchange is emitted as a gather list and inv(L11) is produced
// for the U12 = inv(L11) A12 update (k_u12).
// k_gemm_dmma: trailing update A22 -= L21 U12 on the fp64 tensor cores (mma.sync m8n8k4.f64,
// SASS DMMA.8x8x4): 64x64 CTA tile, 4 warps of 32x32, K = KB staged in shared memory.
#pragma once
#include <cooperative_groups.h>
#include "cpf_common.cuh"
#include "lu.cuh"

namespace cpf {

// per-phase cycle counters of the panel kernel (CTA 0, thread 0), enabled with -DCPF_PANEL_TIMING
__device__ long long g_panel_cycles[8];
__device__ long long g_panel_seg[12];
#ifdef CPF_PANEL_TIMING
#define PSEG(i, t0) do { if (threadIdx.x == 0 && blockIdx.x == 0) { const long long tn = clock64(); atomicAdd((unsigned long long*)&g_panel_seg[i], (unsigned long long)(tn - t0)); t0 = tn; } } while (0)
#else
#define PSEG(i, t0) do {} while (0)
#endif  // lu4 panel (CTA 0): load+sync, column loop, write-back+sync, total

// Diagnostic LU timeline (cpf_debug_lu_trace): per (kind, step) the first start and last end
// %globaltimer of the panel (kind 0), U12 (1) and trailing-GEMM (2) launches of one iteration.
__device__ int g_lu_trace_on;
__device__ unsigned long long g_lu_trace[3 * 512 * 2];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ unsigned long long g_lu_clk[512 * 2];  // panel CTA 0: clock64 at start / end (SM clock)
__device__ __forceinline__ void lu_trace(int kind, int step, int end) {
  if (!g_lu_trace_on || threadIdx.x != 0 || step < 0 || step >= 512) return;
  unsigned long long* e = g_lu_trace + 2 * (kind * 512 + step);
  if (end) atomicMax(e + 1, gtimer());
  else atomicMin(e, gtimer());
  if (kind == 0 && blockIdx.x == 0) g_lu_clk[2 * step + end] = (unsigned long long)clock64();
}

template <class T>
__device__ __forceinline__ T shfl_val(T v, int src);
template <>
__device__ __forceinline__ double shfl_val<double>(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
template <>
__device__ __forceinline__ cplx shfl_val<cplx>(cplx v, int src) {
  return cplx{__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src)};
}

// Candidate packet one CTA pushes into every CTA of the cluster per column: the candidate row
// (KB elements), then {|pivot|, row} and {1/pivot} -- 16-byte chunks, pushed by all NTHR threads
// of the CTA (ceil(CL * PKC / NTHR) st.async each).
template <class T, int KB>
struct PanelPacket {
  static constexpr int DC = KB * (int)sizeof(T) / 16;  // data chunks
  static constexpr int PKC = DC + 2;                   // + key chunk + reciprocal chunk
};

template <class T>
size_t panel3_smem_bytes(int CL, int KB, int nthr) {
  const size_t NW = (size_t)nthr / 32;
  const size_t NC = (size_t)CL;  // one published candidate per CTA
  const size_t pkc = (size_t)KB * sizeof(T) / 16 + 2;
  size_t b = 16 + 16 * 2 * NC * pkc + sizeof(T) * ((size_t)KB * KB + NW * KB);  // 2 mbarriers first
  b += sizeof(double) * NW + sizeof(int) * NW + sizeof(int) * 4 * KB;
  return (b + 15) & ~(size_t)15;
}

__device__ __forceinline__ double2 as_d2(double v) { return make_double2(v, 0.0); }
__device__ __forceinline__ double2 as_d2(cplx v) { return make_double2(v.x, v.y); }
template <class T>
__device__ __forceinline__ T from_d2(double2 v);
template <>
__device__ __forceinline__ double from_d2<double>(double2 v) { return v.x; }
template <>
__device__ __forceinline__ cplx from_d2<cplx>(double2 v) { return cplx{v.x, v.y}; }

// Warp argmax of non-negative doubles with ties broken by the smaller row (redux-based: 3
// warp reductions instead of a 5-round shuffle tree).  Returns the winning value/row/lane.
__device__ __forceinline__ void warp_argmax_redux(double v, int row, double& wv, int& wrow, int& wlane) {
  const unsigned hi = (unsigned)__double2hiint(v), lo = (unsigned)__double2loint(v);
  const unsigned m1 = __reduce_max_sync(0xffffffffu, hi);
  const unsigned m2 = __reduce_max_sync(0xffffffffu, hi == m1 ? lo : 0u);
  const bool cand = (hi == m1) && (lo == m2);
  const unsigned r = (unsigned)__reduce_min_sync(0xffffffffu, cand ? (unsigned)row : 0x7fffffffu);
  const unsigned bal = __ballot_sync(0xffffffffu, cand && (unsigned)row == r);
  wlane = __ffs(bal) - 1;
  wrow = (int)r;
  wv = __hiloint2double((int)m1, (int)m2);
}

// The previous panel's update of this panel's block, fused into the panel load.  With look-ahead,
// panel k+1's 32 columns are exactly the "next block" of step k; instead of a row gather, U12 and a
// GEMM launched between the two panels, panel k+1 reads its rows through step k's interchange
// (gather list of (pos, src) pairs), forms U12 = inv(L11_k) A12 of the step's kbp top rows, and
// applies A22 -= L21_k U12 to its own rows while they go into registers.  Rank 0 writes U12 back
// after the kernel's first cluster barrier (panel_prev_store), when every CTA of the cluster is
// past its loads.  The scratch aliases smem the panel uses only later (no extra footprint, so the
// panel CTAs co-schedule with the trailing-update kernels exactly as before).
template <class T>
struct PanelPrev {
  int kp0;             // previous panel's first row/column; < 0: no previous step (plain load)
  int kbp;             // its width
  const int* gather;   // its (pos, src) pairs
  const int* gcount;
  const T* invL;       // its inv(L11), KB x KB column-major
};

template <class T, int RPT, int NTHR>
__device__ __forceinline__ void panel_load(T (&a)[RPT][kLuMaxKB], const T* __restrict__ A, int lda, int k0, int kb,
                                           const int (&myrow)[RPT], const bool (&alive)[RPT], const PanelPrev<T>& pv,
                                           int* gl, T* u12, T* stage = nullptr, T* linv = nullptr) {
  constexpr int KB = kLuMaxKB;
  const int tid = threadIdx.x;
  if (pv.kp0 < 0) {
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const T* src = A + (int64_t)(k0 + myrow[j]) + (int64_t)lda * k0;
#pragma unroll
      for (int q = 0; q < KB; ++q) a[j][q] = (alive[j] && q < kb) ? src[(int64_t)lda * q] : zero_of<T>();
    }
    return;
  }
#ifdef CPF_PANEL_TIMING
  long long pt0 = clock64();
#endif
  // Global round trips are what a panel pays for under a saturated memory system (the pass that
  // runs beside the LU): the gather list is read whole (it does not wait for its count), and this
  // thread's own rows plus the first L21 chunk are requested right after the A12 rows, so they fly
  // during the U12 product; the remaining L21 chunks are prefetched one chunk ahead.
  const int G = *pv.gcount;
  for (int e = tid; e < 4 * KB; e += NTHR) gl[e] = pv.gather[e];
  if (linv)
    for (int e = tid; e < KB * KB; e += NTHR) linv[e] = pv.invL[e];
  __syncthreads();
  auto src_of = [&](int r) {
    int s = r;
    for (int g = 0; g < G; ++g)
      if (gl[2 * g] == r) s = gl[2 * g + 1];
    return s;
  };
  // A12 (the step's top rows of this block, interchanged) -> u12[i][q]; NTHR % KB == 0, so a
  // thread's elements share one row i and one gather lookup
  static_assert(NTHR % KB == 0, "panel threads");
  constexpr int NA = (KB * KB + NTHR - 1) / NTHR;
  T a12[NA];
  {
    const int i = tid % KB;
    const int64_t srow = i < pv.kbp ? src_of(pv.kp0 + i) : 0;
#pragma unroll
    for (int t = 0; t < NA; ++t) {
      const int e = tid + t * NTHR;
      const int q = e / KB;
      a12[t] = (e < KB * KB && i < pv.kbp && q < kb) ? A[srow + (int64_t)lda * (k0 + q)] : zero_of<T>();
    }
  }
  // this panel's rows (interchanged block row) and the first L21 chunk: in flight during U12
  T v[RPT][KB];
  const T* lrow[RPT];
  T l[RPT][8];
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int r = k0 + myrow[j];
    const T* src = A + (int64_t)(alive[j] ? src_of(r) : 0) + (int64_t)lda * k0;
#pragma unroll
    for (int q = 0; q < KB; ++q) v[j][q] = (alive[j] && q < kb) ? src[(int64_t)lda * q] : zero_of<T>();
    lrow[j] = A + (int64_t)(alive[j] ? r : 0) + (int64_t)lda * pv.kp0;
  }
#pragma unroll
  for (int j = 0; j < RPT; ++j)
#pragma unroll
    for (int p = 0; p < 8; ++p) l[j][p] = (alive[j] && p < pv.kbp) ? lrow[j][(int64_t)lda * p] : zero_of<T>();
#pragma unroll
  for (int t = 0; t < NA; ++t) {
    const int e = tid + t * NTHR;
    if (e < KB * KB) u12[(tid % KB) * KB + e / KB] = a12[t];
  }
  __syncthreads();
  PSEG(4, pt0);
  // U12 = inv(L11) A12 (same summation order as k_u12)
  T uv[NA];
#pragma unroll
  for (int t = 0; t < NA; ++t) {
    const int e = tid + t * NTHR;
    T acc = zero_of<T>();
    if (e < KB * KB) {
      const int i = e / KB, q = e % KB;
      if (linv) {
#pragma unroll
        for (int p = 0; p < KB; ++p)
          if (p <= i) fma_acc(acc, linv[i + KB * p], u12[p * KB + q]);
      } else {
        for (int p = 0; p <= i; ++p) fma_acc(acc, pv.invL[i + KB * p], u12[p * KB + q]);
      }
    }
    uv[t] = acc;
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < NA; ++t) {
    const int e = tid + t * NTHR;
    if (e < KB * KB) u12[e] = uv[t];
  }
  __syncthreads();
  PSEG(5, pt0);
  // rows minus L21 U12.  With a stage (the caller's per-thread smem slots, stride RPT*NTHR) the
  // frame is loaded afterwards, so the update does not add to the column loop's register
  // pressure.  All RPT rows are updated together: each U12 value read from shared memory serves
  // every row of the thread.
  {
#pragma unroll 1
    for (int p0 = 0; p0 < pv.kbp; p0 += 8) {
      T ln[RPT][8];  // next chunk, requested before this chunk's products
#pragma unroll
      for (int j = 0; j < RPT; ++j)
#pragma unroll
        for (int p = 0; p < 8; ++p)
          ln[j][p] = (alive[j] && p0 + 8 + p < pv.kbp) ? lrow[j][(int64_t)lda * (p0 + 8 + p)] : zero_of<T>();
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const T* ur = u12 + (p0 + p) * KB;
#pragma unroll
        for (int q = 0; q < KB; ++q) {
          const T u = ur[q];
#pragma unroll
          for (int j = 0; j < RPT; ++j) fms_acc(v[j][q], l[j][p], u);
        }
      }
#pragma unroll
      for (int j = 0; j < RPT; ++j)
#pragma unroll
        for (int p = 0; p < 8; ++p) l[j][p] = ln[j][p];
    }
#pragma unroll
    for (int j = 0; j < RPT; ++j)
#pragma unroll
      for (int q = 0; q < KB; ++q) {
        if (stage) stage[(size_t)q * RPT * NTHR + j * NTHR + tid] = v[j][q];
        else a[j][q] = v[j][q];
      }
  }
  PSEG(6, pt0);
  if (stage) {
#pragma unroll
    for (int j = 0; j < RPT; ++j)
#pragma unroll
      for (int q = 0; q < KB; ++q) a[j][q] = stage[(size_t)q * RPT * NTHR + j * NTHR + tid];
  }
}

// rank 0 of the cluster, after the column loop: U12 into the step's top rows of this block
template <class T, int NTHR>
__device__ __forceinline__ void panel_prev_store(T* __restrict__ A, int lda, int k0, int kb, const PanelPrev<T>& pv,
                                                 const T* u12) {
  constexpr int KB = kLuMaxKB;
  if (pv.kp0 < 0) return;
  for (int e = threadIdx.x; e < KB * KB; e += NTHR) {
    const int i = e % KB, q = e / KB;
    if (i < pv.kbp && q < kb) A[(int64_t)(pv.kp0 + i) + (int64_t)lda * (k0 + q)] = u12[i * KB + q];
  }
}

template <class T, int KB, int RPT, int NTHR>
__global__ void __launch_bounds__(NTHR, 1) k_panel_lu3(T* __restrict__ A, int n, int lda, int k0, int kb, LuWork w,
                                                       T* __restrict__ invL, const LmDeviceState* st, int gate_running,
                                                       PanelPrev<T> pv) {
  pdl_wait();
  static_assert(KB == kLuMaxKB, "panel width");
  if (panel_gated(st, gate_running, w, k0 / KB)) return;
  lu_trace(0, k0 / KB, 0);
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  constexpr int NW = NTHR / 32;
  const int NC = CL;  // one published candidate per CTA
  using PK = PanelPacket<T, KB>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* pbar = reinterpret_cast<uint64_t*>(smem_raw);    // [2] packet-arrival mbarriers (by parity)
  double2* cand_pk = reinterpret_cast<double2*>(smem_raw + 16);  // [2][NC][PKC] packets pushed by every CTA
  T* top = reinterpret_cast<T*>(cand_pk + (size_t)2 * NC * PK::PKC);  // [KB][KB] row jj = pivot row jj
  T* wrow_s = top + (size_t)KB * KB;                         // [NW][KB] staging of each warp's candidate
  double* wkey_v = reinterpret_cast<double*>(wrow_s + (size_t)NW * KB);  // [NW]
  int* wkey_r = reinterpret_cast<int*>(wkey_v + NW);               // [NW]
  int* pivrows = wkey_r + NW;                                // [KB]
  int* Dl = pivrows + KB;                                    // [KB]
  int* Vl = Dl + KB;                                         // [KB]
  int* misc = Vl + KB;                                       // [KB]

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int m = n - k0;
  const int cta_rows = NTHR * RPT;
  T a[RPT][KB];
  bool alive[RPT];
  int myrow[RPT];  // panel-relative row index
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    myrow[j] = rank * cta_rows + j * NTHR + tid;
    alive[j] = myrow[j] < m;
  }
  // PanelPrev scratch: gather list in pivrows..misc (4 KB ints), U12 in top (both used only later)
  panel_load<T, RPT, NTHR>(a, A, lda, k0, kb, myrow, alive, pv, pivrows, top);
  T cur[RPT];  // a[j][jj] of the current column, maintained by the elimination loop
#pragma unroll
  for (int j = 0; j < RPT; ++j) cur[j] = a[j][0];
  // packet exchange: every CTA pushes its candidate into every CTA with st.async; pbar[par]
  // completes when all CL packets of the column have landed (tx = CL * PKC * 16 bytes)
  if (tid == 0) {
    mbar_init(&pbar[0], 1);
    mbar_init(&pbar[1], 1);
    fence_mbar_init();
  }
  cluster.sync();  // remote CTAs may target pbar only once it is initialised
  if (rank == 0) {  // every CTA is past its loads: U12 to the previous step's top rows
    panel_prev_store<T, NTHR>(A, lda, k0, kb, pv, top);
    __syncthreads();  // top is reused for the pivot rows
  }
  const uint32_t pk_tx = (uint32_t)(NC * PK::PKC * 16);

  // Column loop NOT unrolled (I-cache); registers addressed statically by predication over q.
#ifdef CPF_PANEL_TIMING
  long long tacc[6] = {0, 0, 0, 0, 0, 0};
  long long tprev = clock64();
#define PT(i) do { long long tn = clock64(); tacc[i] += tn - tprev; tprev = tn; } while (0)
#else
#define PT(i) do {} while (0)
#endif
#pragma unroll 1
  for (int jj = 0; jj < kb; ++jj) {
    const int par = jj & 1;
    // ---- (a) my best alive row, then warp argmax (ties -> smaller row)
    double bv = 0.0;
    int bj = 0, brow = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      if (!alive[j]) continue;
      const double v = pivmag(cur[j]);
      if (brow == 0x7fffffff || v > bv) { bv = v; bj = j; brow = myrow[j]; }
    }
    double wv;
    int wrow, wlane;
    warp_argmax_redux(bv, brow, wv, wrow, wlane);
    PT(0);
    // ---- (b) the warp's best lane stages its row; lane 0 posts the warp key
    if (lane == wlane) {
      T* dst = wrow_s + wid * KB;
#pragma unroll
      for (int q = 0; q < KB; ++q) {
        T sel = a[0][q];
#pragma unroll
        for (int j = 1; j < RPT; ++j)
          if (bj == j) sel = a[j][q];
        dst[q] = sel;
      }
      wkey_v[wid] = wv;
      wkey_r[wid] = wrow;
    }
    __syncthreads();
    PT(5);
    // ---- (c) every warp: CTA argmax over the NW warp keys (same result everywhere), then the
    // CTA's threads push the packet chunks (CTA r, chunk c) lane-parallel with st.async
    {
      const double kv = lane < NW ? wkey_v[lane] : 0.0;
      const int kr = lane < NW ? wkey_r[lane] : 0x7fffffff;
      double cv;
      int crow, cw;
      warp_argmax_redux(kv, kr, cv, crow, cw);
      const double2* src = reinterpret_cast<const double2*>(wrow_s + cw * KB);
      const uint32_t slot = smem_u32(cand_pk + (size_t)(par * NC + rank) * PK::PKC);
      const uint32_t bar = smem_u32(&pbar[par]);
      for (int si = tid; si < CL * PK::PKC; si += NTHR) {
        const int r = si / PK::PKC, c = si - r * PK::PKC;
        double2 v;
        if (c < PK::DC) v = src[c];
        else if (c == PK::DC) v = make_double2(cv, __longlong_as_double((long long)crow));
        else v = as_d2(cv != 0.0 ? rcp_of(wrow_s[cw * KB + jj]) : zero_of<T>());
        uint32_t raddr, rbar;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(slot + 16u * c), "r"(r));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(bar), "r"(r));
        st_async16(raddr, v.x, v.y, rbar);
      }
    }
    if (tid == 0) mbar_expect_tx(&pbar[par], pk_tx);
    PT(1);
    mbar_wait(&pbar[par], (uint32_t)((jj >> 1) & 1));
    PT(2);
    // ---- (d) winner among the CL CTA candidates (identical everywhere)
    double gv;
    int grow, gl;
    {
      double2 kk = make_double2(0.0, __longlong_as_double(0x7fffffffLL));
      if (lane < NC) kk = cand_pk[(size_t)(par * NC + lane) * PK::PKC + PK::DC];
      warp_argmax_redux(kk.x, (int)__double_as_longlong(kk.y), gv, grow, gl);
    }
    const int cr = grow;
    const double2* wpk = cand_pk + (size_t)(par * NC + gl) * PK::PKC;
    const T* prow = reinterpret_cast<const T*>(wpk);
    const T rcp = from_d2<T>(wpk[PK::DC + 1]);
    const bool zero_piv = (gv == 0.0);
    if (tid == 0) pivrows[jj] = k0 + cr;
    if (tid < KB) top[jj * KB + tid] = prow[tid];
    if (zero_piv && rank == 0 && tid == 0 && *w.info == 0) *w.info = k0 + jj + 1;
    PT(3);
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      if (alive[j] && myrow[j] == cr) alive[j] = false;
      const bool el = alive[j] && !zero_piv;
      const T l = el ? mul(cur[j], rcp) : zero_of<T>();
      T nx = zero_of<T>();
#pragma unroll
      for (int c8 = 0; c8 < KB; c8 += 8) {
        if (c8 + 7 < jj) continue;  // uniform: chunk entirely left of the pivot column
#pragma unroll
        for (int q = c8; q < c8 + 8; ++q) {
          if (q > jj) fms_acc(a[j][q], l, prow[q]);
          if (q == jj && el) a[j][q] = l;
          if (q == jj + 1) nx = a[j][q];
        }
      }
      cur[j] = nx;
    }
    PT(4);
  }
#ifdef CPF_PANEL_TIMING
  if (rank == 0 && tid == 0)
    for (int i = 0; i < 6; ++i) atomicAdd((unsigned long long*)&g_panel_cycles[i], (unsigned long long)tacc[i]);
  if (rank == 0 && tid == 0) atomicAdd((unsigned long long*)&g_panel_cycles[7], 1ull);
#endif
#undef PT
  __syncthreads();
  // ---- interchange bookkeeping (same rule as k_panel_lu): D (non-pivot top rows, ascending)
  // -> V (pivot rows from below, pick order)
  if (wid == 0) {
    const bool live = lane < kb;
    const int toprow = k0 + lane;
    bool top_is_piv = false;
    for (int q = 0; q < kb; ++q) top_is_piv |= (pivrows[q] == toprow);
    const unsigned dmask = __ballot_sync(0xffffffffu, live && !top_is_piv);
    const unsigned vmask = __ballot_sync(0xffffffffu, live && pivrows[live ? lane : 0] >= k0 + kb);
    if (live && !top_is_piv) Dl[__popc(dmask & ((1u << lane) - 1u))] = toprow;
    if (live && pivrows[lane] >= k0 + kb) Vl[__popc(vmask & ((1u << lane) - 1u))] = pivrows[lane];
    if (lane == 0) misc[0] = __popc(dmask);
  }
  __syncthreads();
  const int nd = misc[0];
  // non-pivot rows: final position (own row, or V[d] when the row is a displaced top row)
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    if (!alive[j]) continue;
    const int o = k0 + myrow[j];
    int pos = o;
    if (o < k0 + kb)
      for (int d = 0; d < nd; ++d)
        if (Dl[d] == o) pos = Vl[d];
    T* dst = A + (int64_t)pos + (int64_t)lda * k0;
#pragma unroll
    for (int q = 0; q < KB; ++q)
      if (q < kb) dst[(int64_t)lda * q] = a[j][q];
  }
  if (rank == 0) {
    // pivot rows -> top block positions
    for (int e = tid; e < kb * kb; e += NTHR) {
      const int r = e % kb, q = e / kb;
      A[(int64_t)(k0 + r) + (int64_t)lda * (k0 + q)] = top[r * KB + q];
    }
    // inv(L11): lane c solves L x = e_c (unit lower)
    if (wid == 0 && invL) {
      const int c = lane;
      T x[KB];
#pragma unroll
      for (int i = 0; i < KB; ++i) {
        T v = from_real<T>((i == c) ? 1.0 : 0.0);
#pragma unroll
        for (int j = 0; j < i; ++j) fms_acc(v, top[i * KB + j], x[j]);
        x[i] = (i < c) ? zero_of<T>() : v;
      }
      if (c < kb)
#pragma unroll
        for (int i = 0; i < KB; ++i)
          if (i < kb) invL[i + KB * c] = x[i];
    }
    if (wid == 1) {
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
  }
  cluster.sync();
  lu_trace(0, k0 / KB, 1);
  panel_latch_next(st, gate_running, w, k0 / KB);
}

// U12 = inv(L11) A12 in place: CTA per 64-column tile of A12 (rows k0..k0+kb).
template <class T, int KB>
__global__ void __launch_bounds__(256) k_u12(T* __restrict__ A, int cend, int lda, int k0, int kb,
                                             const T* __restrict__ invL, const LmDeviceState* st, int gate_running,
                                             int cbeg) {
  pdl_wait();
  if (lu_gated(st, gate_running)) return;
  lu_trace(1, k0 / KB, 0);
  __shared__ T Li[KB * KB];
  __shared__ T Bt[KB * 64];
  const int c0 = cbeg + blockIdx.x * 64;
  const int ncol = min(64, cend - c0);
  for (int e = threadIdx.x; e < KB * KB; e += 256) Li[e] = invL[e];
  for (int e = threadIdx.x; e < KB * 64; e += 256) {
    const int i = e % KB, c = e / KB;
    Bt[c * KB + i] = (i < kb && c < ncol) ? A[(int64_t)(k0 + i) + (int64_t)lda * (c0 + c)] : zero_of<T>();
  }
  __syncthreads();
  for (int e = threadIdx.x; e < KB * 64; e += 256) {
    const int i = e % KB, c = e / KB;
    if (i >= kb || c >= ncol) continue;
    T acc = zero_of<T>();
    for (int j = 0; j <= i; ++j) fma_acc(acc, Li[i + KB * j], Bt[j + c * KB]);
    A[(int64_t)(k0 + i) + (int64_t)lda * (c0 + c)] = acc;
  }
  lu_trace(1, k0 / KB, 1);
}

// C -= A B on the fp64 tensor cores.  C: m x nn at (r0, c0); A = L21 at (r0, k0); B = U12 at (k0, c0).
// K = k <= 32.  CTA 64x64, 4 warps each 32x32 = 4x4 m8n8 tiles; mma.sync.m8n8k4.row.col.f64.
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128) k_gemm_dmma(double* __restrict__ M, int lda, int r0, int c0, int k0, int m,
                                                   int nn, int k, const LmDeviceState* st, int gate_running) {
  pdl_wait();
  if (lu_gated(st, gate_running)) return;
  lu_trace(2, k0 / 32, 0);
  constexpr int TM = 64, TN = 64, KM = 32, PADA = 68, PADB = 68;
  __shared__ double As[KM * PADA];  // As[q][i] (k-major), stride PADA
  __shared__ double Bs[KM * PADB];  // Bs[q][j]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int bm = blockIdx.x * TM, bn = blockIdx.y * TN;
  // stage A (64 x k) and B (k x 64); zero-fill out of range and K tail to a multiple of 4
  const int wm = (wid & 1) * 32, wn = (wid >> 1) * 32;
  const int g = lane >> 2, t = lane & 3;
  // C[row = g, cols 2t, 2t+1] of each 8x8 tile, fetched first (in flight with the A/B staging) and
  // all before any store (the compiler cannot hoist loads over stores through the same pointer):
  // one memory round trip per CTA instead of 32.  C1's first 4736 x 4704 x 32 update 185 -> 106 us,
  // C1 51 -> 57 it/s.
  double cv[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gi = bm + wm + 8 * i + g, gj = bn + wn + 8 * j + 2 * t + h;
        cv[i][j][h] = (gi < m && gj < nn) ? M[(int64_t)(r0 + gi) + (int64_t)lda * (c0 + gj)] : 0.0;
      }
  const int kp = (k + 3) & ~3;
  // stage A (64 x KM) and B (KM x 64): constant trip counts so all 32 loads per thread are in
  // flight at once (rows/cols beyond the block and K beyond k are zero)
  {
    double va[TM * KM / 128], vb[TN * KM / 128];
#pragma unroll
    for (int t = 0; t < TM * KM / 128; ++t) {
      const int e = tid + 128 * t;
      const int i = e % TM, q = e / TM;
      const int gi = bm + i;
      va[t] = (gi < m && q < k) ? M[(int64_t)(r0 + gi) + (int64_t)lda * (k0 + q)] : 0.0;
    }
#pragma unroll
    for (int t = 0; t < TN * KM / 128; ++t) {
      const int e = tid + 128 * t;
      const int q = e % KM, j = e / KM;
      const int gj = bn + j;
      vb[t] = (gj < nn && q < k) ? M[(int64_t)(k0 + q) + (int64_t)lda * (c0 + gj)] : 0.0;
    }
#pragma unroll
    for (int t = 0; t < TM * KM / 128; ++t) {
      const int e = tid + 128 * t;
      As[(e / TM) * PADA + e % TM] = va[t];
    }
#pragma unroll
    for (int t = 0; t < TN * KM / 128; ++t) {
      const int e = tid + 128 * t;
      Bs[(e % KM) * PADB + e / KM] = vb[t];
    }
  }
  __syncthreads();
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) { acc[i][j][0] = 0.0; acc[i][j][1] = 0.0; }
  for (int q = 0; q < kp; q += 4) {
    double af[4], bf[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) af[i] = As[(q + t) * PADA + wm + 8 * i + g];
#pragma unroll
    for (int j = 0; j < 4; ++j) bf[j] = Bs[(q + t) * PADB + wn + 8 * j + g];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gi = bm + wm + 8 * i + g, gj = bn + wn + 8 * j + 2 * t + h;
        if (gi < m && gj < nn) M[(int64_t)(r0 + gi) + (int64_t)lda * (c0 + gj)] = cv[i][j][h] - acc[i][j][h];
      }
  lu_trace(2, k0 / 32, 1);
}

}  // namespace cpf
