// LU v4 panel: k_panel_lu4 -- register-resident m x 32 panel with a ROTATING register frame.
//
// Round 2: the frame now rotates by ONE column per column (CH = 1).  With 8-column unrolled chunks
// the column loop was ~80 KB of SASS and ncu showed no_instructions as the top stall (29-40 %);
// the 31 register moves of a per-column shift cost less than the instruction-cache misses:
// measured (1 x B200, bench.py, same box) LU phase config 4 2.38-2.43 -> 2.24-2.25 ms, 164-166 ->
// 168-170 it/s; config 1 (n_B = 4800) LU 9.44 -> 8.53 ms, 57.5 -> 62.6 it/s (CH = 2 and 4 in
// between).
//
// Same algorithm and interface as k_panel_lu3 (lu3.cuh): partial pivoting by |a| (|re|+|im| for
// complex, LAPACK's cabs1), ties to the smaller row, pivot rows retired logically and written
// once at the end, interchange emitted as a gather list, inv(L11) for k_u12.  What changes is
// how a thread addresses its row registers.  The 32 columns are processed in 4 chunks of 8; the
// 8 columns of a chunk are unrolled at compile time and the thread's row is kept in a frame
// a[0..31] whose column u is the chunk's u-th column -- so the pivot column, the next column and
// the elimination range are all static register indices (no 32-way predicated selects per
// column).  At the end of a chunk the 8 finished columns are flushed to shared memory and the
// frame shifts left by 8.  Rows per CTA are large (RPT x NTHR = 512 for fp64), so the panel of a
// 1200-row system needs a cluster of 3 CTAs instead of 10 -- small clusters also co-schedule
// next to a running tensor pass.
//
// Load: the previous step's interchange and rank-32 update of this panel's columns are applied
// while loading (panel_load, lu3.cuh: look-ahead without kernels between consecutive panels).
// Per column: warp argmax (computed inside the previous column's elimination, right after the
// column itself is updated) -> the warp's best row is staged -> CTA argmax (one __syncthreads)
// -> the CTA's candidate packet (frame row, {|pivot|, row}, 1/pivot) is pushed into every CTA of
// the cluster with st.async, completing tx-bytes on the receiver's mbarrier -> wait on the local
// mbarrier -> winner -> elimination of the (static) remaining frame columns.  A single-CTA panel
// (m <= 512) takes its winner straight from the staged rows (no packets).  Measured ~2350 cycles
// per column, 66-69 us per 32-column panel of a 1200-row system (tools/panel_phases.py).
#pragma once
#include <cooperative_groups.h>
#include "cpf_common.cuh"
#include "lu.cuh"
#include "lu3.cuh"

namespace cpf {

template <class T>
size_t panel4_smem_bytes(int CL, int nthr, int rpt) {
  constexpr int KB = kLuMaxKB;
  const size_t NW = (size_t)nthr / 32;
  const size_t pkc = (size_t)KB * sizeof(T) / 16 + 2;
  size_t b = 16 + 16 * 2 * (size_t)CL * pkc;                     // mbarriers + packets
  b += sizeof(T) * ((size_t)KB * nthr * rpt + 2 * NW * KB + (size_t)KB * KB);  // fin + wrow_s[2] + top
  b += sizeof(double) * 2 * NW + sizeof(int) * 2 * NW + sizeof(int) * 4 * KB;
  b = (b + 15) & ~(size_t)15;
  b += sizeof(T) * (size_t)KB * KB;  // inv(L11) of the previous step (fused load)
  return (b + 15) & ~(size_t)15;
}

template <class T, int RPT, int NTHR>
__global__ void __launch_bounds__(NTHR, 1) k_panel_lu4(T* __restrict__ A, int n, int lda, int k0, int kb, LuWork w,
                                                       T* __restrict__ invL, const LmDeviceState* st, int gate_running,
                                                       PanelPrev<T> pv) {
  pdl_wait();
  if (panel_gated(st, gate_running, w, k0 / kLuMaxKB)) return;
  lu_trace(0, k0 / kLuMaxKB, 0);
#ifdef CPF_PANEL_TIMING
  const long long seg0 = clock64();
#endif
  constexpr int KB = kLuMaxKB;  // 32
  constexpr int CH = 1;         // columns per static chunk (see the header: 1 is fastest)
  constexpr int NW = NTHR / 32;
  constexpr int ROWS = RPT * NTHR;  // rows per CTA
  using PK = PanelPacket<T, KB>;
  cg::cluster_group cluster = cg::this_cluster();
  const int CL = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* pbar = reinterpret_cast<uint64_t*>(smem_raw);               // [2] packet arrivals (by parity)
  double2* cand_pk = reinterpret_cast<double2*>(smem_raw + 16);         // [2][CL][PKC]
  T* fin = reinterpret_cast<T*>(cand_pk + (size_t)2 * CL * PK::PKC);   // [KB][ROWS] finished columns
  T* wrow_s = fin + (size_t)KB * ROWS;                                  // [2][NW][KB] warp candidates (by parity)
  T* top = wrow_s + (size_t)2 * NW * KB;                                // [KB][KB] (rank 0: L11 for inv)
  double* wkey_v = reinterpret_cast<double*>(top + (size_t)KB * KB);    // [2][NW]
  int* wkey_r = reinterpret_cast<int*>(wkey_v + 2 * NW);                // [2][NW]
  int* pivrows = wkey_r + 2 * NW;                                       // [KB]
  int* Dl = pivrows + KB;                                               // [KB]
  int* Vl = Dl + KB;                                                    // [KB]
  int* misc = Vl + KB;                                                  // [KB]
  T* linv_s = reinterpret_cast<T*>((reinterpret_cast<uintptr_t>(misc + KB) + 15) & ~(uintptr_t)15);  // [KB][KB]

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int m = n - k0;
  T a[RPT][KB];  // frame: a[j][q] = column (c8 + q) of row j
  bool alive[RPT];
  int myrow[RPT];  // panel-relative row index
  int pcol[RPT];   // pivot column of a retired row
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    myrow[j] = rank * ROWS + j * NTHR + tid;
    alive[j] = myrow[j] < m;
    pcol[j] = -1;
  }
  // PanelPrev scratch: gather list in pivrows..misc, U12 in top, rows staged in fin (all used later)
  panel_load<T, RPT, NTHR>(a, A, lda, k0, kb, myrow, alive, pv, pivrows, top, fin, linv_s);
  if (tid == 0) {
    mbar_init(&pbar[0], 1);
    mbar_init(&pbar[1], 1);
    fence_mbar_init();
  }
  cluster.sync();  // remote CTAs may target pbar only once it is initialised
#ifdef CPF_PANEL_TIMING
  const long long seg1 = clock64();
#endif
  if (rank == 0) panel_prev_store<T, NTHR>(A, lda, k0, kb, pv, top);  // every CTA is past its loads
  const uint32_t pk_tx = (uint32_t)(CL * PK::PKC * 16);
  const uint32_t bar0_u32 = smem_u32(&pbar[0]), bar1_u32 = smem_u32(&pbar[1]);

#ifdef CPF_PANEL_TIMING
  long long tacc[6] = {0, 0, 0, 0, 0, 0};
  long long tprev = clock64();
#define PT(i) do { long long tn = clock64(); tacc[i] += tn - tprev; tprev = tn; } while (0)
#else
#define PT(i) do {} while (0)
#endif

  // (a) my best alive row in a frame column, then the warp argmax (ties -> smaller row).  Column
  // u+1's search runs inside column u's elimination, right after column u+1 itself is updated, so
  // its reduction latency overlaps the remaining columns' FMAs.
  auto warp_best = [&](int fc, double& wv, int& wrow, int& wlane, int& bj) {
    double bv = 0.0;
    int brow = 0x7fffffff;
    bj = 0;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      if (!alive[j]) continue;
      const double v = pivmag(a[j][fc]);
      if (brow == 0x7fffffff || v > bv) { bv = v; bj = j; brow = myrow[j]; }
    }
    warp_argmax_redux(bv, brow, wv, wrow, wlane);
  };
  double nwv;
  int nwrow, nwlane, nbj;
  warp_best(0, nwv, nwrow, nwlane, nbj);
#pragma unroll 1
  for (int c8 = 0; c8 < kb; c8 += CH) {
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int jj = c8 + u;
      if (jj >= kb) break;
      const int par = jj & 1;
      const double wv = nwv;
      const int wrow = nwrow, wlane = nwlane, bj = nbj;
      PT(0);
      // ---- (b) the warp's best lane stages its frame row; lane 0 posts the warp key (buffers by
      // column parity: a warp staging column jj+2 has passed column jj+1's barrier, so nobody still
      // reads column jj's buffer)
      T* wrow_p = wrow_s + (size_t)par * NW * KB;
      double* wkv_p = wkey_v + par * NW;
      int* wkr_p = wkey_r + par * NW;
      if (lane == wlane) {
        T* dst = wrow_p + wid * KB;
        if constexpr (sizeof(T) == 8) {  // 16-byte stores
#pragma unroll
          for (int q = 0; q < KB; q += 2) {
            T s0 = a[0][q], s1 = a[0][q + 1];
#pragma unroll
            for (int j = 1; j < RPT; ++j)
              if (bj == j) { s0 = a[j][q]; s1 = a[j][q + 1]; }
            *reinterpret_cast<double2*>(dst + q) = make_double2(as_d2(s0).x, as_d2(s1).x);
          }
        } else {
#pragma unroll
          for (int q = 0; q < KB; ++q) {
            T sel = a[0][q];
#pragma unroll
            for (int j = 1; j < RPT; ++j)
              if (bj == j) sel = a[j][q];
            dst[q] = sel;
          }
        }
        wkv_p[wid] = wv;
        wkr_p[wid] = wrow;
      }
      __syncthreads();
      PT(5);
      // ---- (c) every warp: CTA argmax over the NW warp keys
      double cv;
      int crow, cw;
      {
        const double kv = lane < NW ? wkv_p[lane] : 0.0;
        const int kr = lane < NW ? wkr_p[lane] : 0x7fffffff;
        warp_argmax_redux(kv, kr, cv, crow, cw);
      }
      double gv;
      int cr;
      const double2* wpk;
      T rcp;
      if (CL == 1) {
        // single-CTA panel (m <= RPT*NTHR rows): the CTA's candidate is the pivot; read its staged
        // row directly, no packet exchange
        gv = cv;
        cr = crow;
        wpk = reinterpret_cast<const double2*>(wrow_p + cw * KB);
        rcp = cv != 0.0 ? rcp_of(wrow_p[cw * KB + u]) : zero_of<T>();
        PT(1);
      } else {
        // the CTA's threads push its candidate packet into every CTA of the cluster
        const double2* src = reinterpret_cast<const double2*>(wrow_p + cw * KB);
        const uint32_t slot = smem_u32(cand_pk + (size_t)(par * CL + rank) * PK::PKC);
        for (int si = tid; si < CL * PK::PKC; si += NTHR) {
          const int r = si / PK::PKC, c = si - r * PK::PKC;
          double2 v;
          if (c < PK::DC) v = src[c];
          else if (c == PK::DC) v = make_double2(cv, __longlong_as_double((long long)crow));
          else v = as_d2(cv != 0.0 ? rcp_of(wrow_p[cw * KB + u]) : zero_of<T>());
          uint32_t raddr, rbar;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(slot + 16u * c), "r"(r));
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(par ? bar1_u32 : bar0_u32), "r"(r));
          st_async16(raddr, v.x, v.y, rbar);
        }
        if (tid == 0) mbar_expect_tx(&pbar[par], pk_tx);
        PT(1);
        mbar_wait(&pbar[par], (uint32_t)((jj >> 1) & 1));
        PT(2);
        // ---- (d) winner among the CL CTA candidates (identical everywhere)
        int gl;
        {
          double2 kk = make_double2(0.0, __longlong_as_double(0x7fffffffLL));
          if (lane < CL) kk = cand_pk[(size_t)(par * CL + lane) * PK::PKC + PK::DC];
          warp_argmax_redux(kk.x, (int)__double_as_longlong(kk.y), gv, cr, gl);
        }
        wpk = cand_pk + (size_t)(par * CL + gl) * PK::PKC;
        rcp = from_d2<T>(wpk[PK::DC + 1]);
      }
      const bool zero_piv = (gv == 0.0);
      if (tid == 0) pivrows[jj] = k0 + cr;
      if (zero_piv && rank == 0 && tid == 0 && *w.info == 0) *w.info = k0 + jj + 1;
      PT(3);
      // ---- (e) elimination of the frame columns u+1 .. KB-1 (static range)
      T l[RPT];
      bool el[RPT];
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        if (alive[j] && myrow[j] == cr) { alive[j] = false; pcol[j] = jj; }
        el[j] = alive[j] && !zero_piv;
        l[j] = el[j] ? mul(a[j][u], rcp) : zero_of<T>();
      }
      // column u+1 first, then its pivot search, then the rest
      if (u + 1 < KB) {
        T v1;
        if constexpr (sizeof(T) == 8) {
          const double2 pr = wpk[(u + 1) / 2];
          v1 = from_d2<T>(make_double2(((u + 1) & 1) ? pr.y : pr.x, 0.0));
        } else {
          v1 = from_d2<T>(wpk[u + 1]);
        }
#pragma unroll
        for (int j = 0; j < RPT; ++j) fms_acc(a[j][u + 1], l[j], v1);
      }
      if (jj + 1 < kb) warp_best(u + 1, nwv, nwrow, nwlane, nbj);
      if constexpr (sizeof(T) == 8) {
#pragma unroll
        for (int c = (u + 2) / 2; c < KB / 2; ++c) {
          const double2 v = wpk[c];
#pragma unroll
          for (int j = 0; j < RPT; ++j) {
            if (2 * c > u + 1) fms_acc(a[j][2 * c], l[j], from_d2<T>(make_double2(v.x, 0.0)));
            fms_acc(a[j][2 * c + 1], l[j], from_d2<T>(make_double2(v.y, 0.0)));
          }
        }
      } else {
#pragma unroll
        for (int c = u + 2; c < KB; ++c) {
          const T v = from_d2<T>(wpk[c]);
#pragma unroll
          for (int j = 0; j < RPT; ++j) fms_acc(a[j][c], l[j], v);
        }
      }
#pragma unroll
      for (int j = 0; j < RPT; ++j)
        if (el[j]) a[j][u] = l[j];  // L multiplier; the pivot row keeps its U entry
      PT(4);
    }
    // ---- chunk end: flush the 8 finished frame columns, shift the frame left by 8
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
#pragma unroll
      for (int q = 0; q < CH; ++q) fin[(size_t)(c8 + q) * ROWS + j * NTHR + tid] = a[j][q];
#pragma unroll
      for (int q = 0; q < KB - CH; ++q) a[j][q] = a[j][q + CH];
#pragma unroll
      for (int q = KB - CH; q < KB; ++q) a[j][q] = zero_of<T>();
    }
  }
#ifdef CPF_PANEL_TIMING
  const long long seg2 = clock64();
  if (rank == 0 && tid == 0) {
    atomicAdd((unsigned long long*)&g_panel_seg[0], (unsigned long long)(seg1 - seg0));
    atomicAdd((unsigned long long*)&g_panel_seg[1], (unsigned long long)(seg2 - seg1));
  }
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
  // every row to its final position: pivot rows to k0 + pivot column, displaced top rows to
  // V[d], the rest stay
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    if (myrow[j] >= m) continue;
    const int o = k0 + myrow[j];
    int pos = o;
    if (pcol[j] >= 0) {
      pos = k0 + pcol[j];
    } else if (o < k0 + kb) {
      for (int d = 0; d < nd; ++d)
        if (Dl[d] == o) pos = Vl[d];
    }
    T* dst = A + (int64_t)pos + (int64_t)lda * k0;
    for (int q = 0; q < kb; ++q) dst[(int64_t)lda * q] = fin[(size_t)q * ROWS + j * NTHR + tid];
  }
  cluster.sync();  // every CTA's rows are in place (global writes ordered at cluster scope)
#ifdef CPF_PANEL_TIMING
  if (rank == 0 && tid == 0) atomicAdd((unsigned long long*)&g_panel_seg[2], (unsigned long long)(clock64() - seg2));
#endif
  if (rank == 0) {
    for (int e = tid; e < KB * KB; e += NTHR) {
      const int r = e / KB, q = e % KB;
      top[e] = (r < kb && q < kb) ? A[(int64_t)(k0 + r) + (int64_t)lda * (k0 + q)] : zero_of<T>();
    }
    __syncthreads();
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
#ifdef CPF_PANEL_TIMING
  if (rank == 0 && tid == 0) atomicAdd((unsigned long long*)&g_panel_seg[3], (unsigned long long)(clock64() - seg0));
#endif
  lu_trace(0, k0 / kLuMaxKB, 1);
  panel_latch_next(st, gate_running, w, k0 / kLuMaxKB);
}

}  // namespace cpf
