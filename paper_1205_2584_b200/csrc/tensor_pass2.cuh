// Tensor passes v2: TMA bulk-copy pipelines (cp.async.bulk + mbarrier) feeding register-tiled
// fp64 / complex128 FMA loops.  Same math and outputs as tensor_pass.cuh (see the layout comment
// there); this is the production path whenever the tensor rows are 16-byte aligned (I_1 even for
// float64, always for complex128).
//
// Pass A: CTA = (i1 tile, range of m).  A stage holds Y[rowblock, c0:c0+CKY] (CKY contiguous
// runs, one per c) plus the CKY conj(A_N) rows.  Thread (ti, tm) owns RPT consecutive i1 rows of
// the m = m_first + tm row of the block and accumulates its P rows over all c in registers; at the
// end of each row block it folds P into its M_1 accumulator (registers) and reduces
// P conj(A_1) over i1 for Z (warp-parallel column sums in shared memory).
// Pass B: CTA = (c, i1 tile, m chunk).  A stage holds Y[i1 tile, m0:m0+MS, c] plus MS
// conj(KRmid) rows; thread (ti, tm) owns RPT i1 rows, accumulates over its m's, multiplies by
// conj(A_1) and the CTA reduces to one partial M_N[c, :] per (tile, chunk).
#pragma once
#include "cpf_common.cuh"
#include "small_ops.cuh"

namespace cpf {

template <class T, int RPT>
struct RowVec {
  T v[RPT];
};

template <class T, int RPT>
__device__ __forceinline__ void lds_rows(const T* p, T (&y)[RPT]) {
  if constexpr (RPT == 2 && sizeof(T) == 8) {
    double2 t = *reinterpret_cast<const double2*>(p);
    y[0] = t.x;
    y[1] = t.y;
  } else {
#pragma unroll
    for (int j = 0; j < RPT; ++j) y[j] = p[j];
  }
}

template <class T>
__device__ __forceinline__ void lds_pair(const T* p, T& a, T& b) {
  if constexpr (sizeof(T) == 8) {
    double2 t = *reinterpret_cast<const double2*>(p);
    a = t.x;
    b = t.y;
  } else {
    a = p[0];
    b = p[1];
  }
}

struct PassGeom {
  int64_t I1, Lmid, C;  // C = local slab length of mode N
  int TI, TM, RPT;      // threads along i1 / along m, rows per thread
  int tiles;            // ceil(I1 / (TI*RPT))
  int full;             // 1 if one tile covers I1 (row blocks of TM m's are contiguous)
  int64_t SL;           // elements per c (pass A) / per stage row (pass B) in smem
  int CK;               // pass A: c per stage; pass B: m per stage
  int NST;              // pipeline depth
  int64_t m_per_cta;    // pass A: m range per CTA; pass B: m chunk per CTA
  size_t stage_elems;   // T elements per stage (data + operand rows)
};

// ------------------------------------------------------------------------------------------
constexpr int kConsumers = 256;  // consumer threads; one extra producer warp issues the TMA copies

template <class T, int RP, int RPT>
__global__ void __launch_bounds__(kConsumers + 32, 1) k_pass_a2(const T* __restrict__ Y, PassGeom g, const T* __restrict__ WNc,
                                                    const T* __restrict__ A1c, const T* __restrict__ KMc,
                                                    T* __restrict__ z_part, T* __restrict__ m1_part,
                                                    const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);  // [0,NST) full, [NST,2NST) empty
  T* stages = reinterpret_cast<T*>(smem_raw + 128);
  T* zs = stages + (size_t)g.NST * g.stage_elems;  // RP * nthr
  T* m1s = zs + (size_t)RP * kConsumers;            // RPT * RP * nthr, [j][r][thread]
  const int tid = threadIdx.x, nthr = kConsumers;
  const int lane = tid & 31, wid = tid >> 5, nw = nthr >> 5;
  const int ti = tid % g.TI, tm = tid / g.TI;
  const int64_t TIL = (int64_t)g.TI * RPT;
  const int64_t tile = blockIdx.x;
  const int64_t a0 = tile * TIL;
  const int64_t Lrows = g.I1 * g.Lmid;
  const int64_t i1_0 = a0 + (int64_t)ti * RPT;
  const bool row_ok = (tm < g.TM) && (i1_0 < g.I1);
  const int64_t mbeg = (int64_t)blockIdx.y * g.m_per_cta;
  const int64_t mend = min(g.Lmid, mbeg + g.m_per_cta);
  if (mbeg >= mend) return;
  const int64_t nrb = (mend - mbeg + g.TM - 1) / g.TM;
  const int64_t ncc = (g.C + g.CK - 1) / g.CK;
  const int64_t nq = nrb * ncc;
  const int64_t rowlen = g.full ? g.I1 : min(TIL, g.I1 - a0);  // contiguous elements per (m, c)
  const size_t wofs = (size_t)g.CK * g.SL;                        // W rows after the Y block

  auto issue = [&](int64_t q) {
    const int s = (int)(q % g.NST);
    const int64_t rb = q / ncc, cc = q % ncc;
    const int64_t mf = mbeg + rb * g.TM;
    const int64_t mc = min((int64_t)g.TM, mend - mf);
    const int64_t c0 = cc * g.CK;
    const int ck = (int)min((int64_t)g.CK, g.C - c0);
    T* dst = stages + (size_t)s * g.stage_elems;
    const uint32_t ybytes = (uint32_t)((g.full ? g.I1 * mc : rowlen) * sizeof(T));
    const uint32_t wbytes = (uint32_t)((ck * RP * sizeof(T) + 15) & ~(size_t)15);
    fence_proxy_async();
    mbar_expect_tx(&bars[s], ybytes * ck + wbytes);
    const T* src = Y + a0 + g.I1 * mf + Lrows * c0;
    for (int k = 0; k < ck; ++k) bulk_g2s(dst + (size_t)k * g.SL, src + Lrows * k, ybytes, &bars[s]);
    bulk_g2s(dst + wofs, WNc + c0 * RP, wbytes, &bars[s]);
  };

  if (tid == 0) {
    for (int s = 0; s < g.NST; ++s) {
      mbar_init(&bars[s], 1);
      mbar_init(&bars[g.NST + s], nw);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid >= nthr) {  // ---- producer warp
    if (lane == 0)
      for (int64_t q = 0; q < nq; ++q) {
        const int s = (int)(q % g.NST);
        if (q >= g.NST) mbar_wait(&bars[g.NST + s], (uint32_t)(((q / g.NST) - 1) & 1));
        issue(q);
      }
    return;
  }

  T acc[RPT][RP];
#pragma unroll
  for (int j = 0; j < RPT; ++j)
#pragma unroll
    for (int r = 0; r < RP; ++r) { acc[j][r] = zero_of<T>(); m1s[((size_t)j * RP + r) * nthr + tid] = zero_of<T>(); }

  const int64_t yoff = (int64_t)tm * g.I1 + (int64_t)ti * RPT;  // tm*I1 only matters when full
  for (int64_t q = 0; q < nq; ++q) {
    const int s = (int)(q % g.NST);
    const int64_t rb = q / ncc, cc = q % ncc;
    const int64_t mf = mbeg + rb * g.TM;
    const int64_t c0 = cc * g.CK;
    const int ck = (int)min((int64_t)g.CK, g.C - c0);
    const bool ok = row_ok && (mf + tm < mend);
    mbar_wait(&bars[s], (uint32_t)((q / g.NST) & 1));
    const T* ys = stages + (size_t)s * g.stage_elems;
    const T* ws = ys + wofs;
    if (ok) {
#pragma unroll 2
      for (int k = 0; k < ck; ++k) {
        T y0[RPT], w[RP];
        lds_rows<T, RPT>(ys + (size_t)k * g.SL + yoff, y0);
#pragma unroll
        for (int r = 0; r < RP; r += 2) lds_pair(ws + k * RP + r, w[r], w[r + 1]);
#pragma unroll
        for (int r = 0; r < RP; ++r)
#pragma unroll
          for (int j = 0; j < RPT; ++j) fma_acc(acc[j][r], y0[j], w[r]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars[g.NST + s]);  // stage s consumed by this warp
    if (cc == ncc - 1) {
      // ---- row-block epilogue: M_1 (registers) and Z (column sums over i1)
      const int64_t m = mf + tm;
      if (ok) {
        const T* km = KMc + m * RP;
#pragma unroll
        for (int r = 0; r < RP; ++r) {
          const T kv = ld_ro(km + r);
          T zt = mul(acc[0][r], ld_ro(A1c + i1_0 * RP + r));
#pragma unroll
          for (int j = 0; j < RPT; ++j) {
            T* mp = m1s + ((size_t)j * RP + r) * nthr + tid;
            T t = *mp;
            fma_acc(t, acc[j][r], kv);
            *mp = t;
          }
#pragma unroll
          for (int j = 1; j < RPT; ++j) fma_acc(zt, acc[j][r], ld_ro(A1c + (i1_0 + j) * RP + r));
          zs[r * nthr + tid] = zt;
        }
      } else {
#pragma unroll
        for (int r = 0; r < RP; ++r) zs[r * nthr + tid] = zero_of<T>();
      }
#pragma unroll
      for (int j = 0; j < RPT; ++j)
#pragma unroll
        for (int r = 0; r < RP; ++r) acc[j][r] = zero_of<T>();
      named_sync(1, nthr);
      const int ncol = g.TM * RP;
      for (int col = wid; col < ncol; col += nw) {
        const int tm2 = col / RP, r2 = col % RP;
        const T* zc = zs + r2 * nthr + tm2 * g.TI;
        T sacc = zero_of<T>();
        for (int t = lane; t < g.TI; t += 32) sacc = add(sacc, zc[t]);
        sacc = warp_sum(sacc);
        const int64_t m2 = mf + tm2;
        if (lane == 0 && m2 < mend) z_part[(tile * g.Lmid + m2) * RP + r2] = sacc;
      }
      named_sync(1, nthr);
    }
  }
  // ---- M_1 partial of this CTA: reduce the TM groups (fixed order), one j at a time
  named_sync(1, nthr);
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    if (tm == 0 && row_ok && i1_0 + j < g.I1) {
      for (int r = 0; r < RP; ++r) {
        const T* mp = m1s + ((size_t)j * RP + r) * nthr;
        T sacc = mp[ti];
        for (int q2 = 1; q2 < g.TM; ++q2) sacc = add(sacc, mp[q2 * g.TI + ti]);
        m1_part[((int64_t)blockIdx.y * g.I1 + i1_0 + j) * RP + r] = sacc;
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
template <class T, int RP, int RPT>
__global__ void __launch_bounds__(kConsumers + 32, 1) k_pass_b2(const T* __restrict__ Y, PassGeom g, const T* __restrict__ A1c,
                                                    const T* __restrict__ KMc, T* __restrict__ part,
                                                    const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  T* stages = reinterpret_cast<T*>(smem_raw + 128);
  T* red = stages + (size_t)g.NST * g.stage_elems;  // RP * nwarps
  const int tid = threadIdx.x, nthr = kConsumers;
  const int lane = tid & 31, wid = tid >> 5, nw = nthr >> 5;
  const int ti = tid % g.TI, tm = tid / g.TI;
  const int64_t TIL = (int64_t)g.TI * RPT;
  const int64_t c = blockIdx.x;
  const int64_t tile = blockIdx.z;
  const int64_t a0 = tile * TIL;
  const int64_t Lrows = g.I1 * g.Lmid;
  const int64_t i1_0 = a0 + (int64_t)ti * RPT;
  const bool row_ok = (tm < g.TM) && (i1_0 < g.I1);
  const int64_t mbeg = (int64_t)blockIdx.y * g.m_per_cta;
  const int64_t mend = min(g.Lmid, mbeg + g.m_per_cta);
  const int64_t nq = mend > mbeg ? (mend - mbeg + g.CK - 1) / g.CK : 0;
  const int64_t rowlen = g.full ? g.I1 : min(TIL, g.I1 - a0);
  const size_t kofs = (size_t)g.CK * g.SL;
  const T* ycol = Y + Lrows * c + a0;

  auto issue = [&](int64_t q) {
    const int s = (int)(q % g.NST);
    const int64_t m0 = mbeg + q * g.CK;
    const int mc = (int)min((int64_t)g.CK, mend - m0);
    T* dst = stages + (size_t)s * g.stage_elems;
    const uint32_t kbytes = (uint32_t)((mc * RP * sizeof(T) + 15) & ~(size_t)15);
    fence_proxy_async();
    if (g.full) {
      const uint32_t yb = (uint32_t)(g.I1 * mc * sizeof(T));
      mbar_expect_tx(&bars[s], yb + kbytes);
      bulk_g2s(dst, ycol + g.I1 * m0, yb, &bars[s]);
    } else {
      const uint32_t yb = (uint32_t)(rowlen * sizeof(T));
      mbar_expect_tx(&bars[s], yb * mc + kbytes);
      for (int k = 0; k < mc; ++k) bulk_g2s(dst + (size_t)k * g.SL, ycol + g.I1 * (m0 + k), yb, &bars[s]);
    }
    bulk_g2s(dst + kofs, KMc + m0 * RP, kbytes, &bars[s]);
  };

  if (tid == 0) {
    for (int s = 0; s < g.NST; ++s) {
      mbar_init(&bars[s], 1);
      mbar_init(&bars[g.NST + s], nw);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid >= nthr) {  // ---- producer warp
    if (lane == 0)
      for (int64_t q = 0; q < nq; ++q) {
        const int s = (int)(q % g.NST);
        if (q >= g.NST) mbar_wait(&bars[g.NST + s], (uint32_t)(((q / g.NST) - 1) & 1));
        issue(q);
      }
    return;
  }

  T acc[RPT][RP];
#pragma unroll
  for (int j = 0; j < RPT; ++j)
#pragma unroll
    for (int r = 0; r < RP; ++r) acc[j][r] = zero_of<T>();

  // row of (ti, m-in-stage k): full -> k*I1 + ti*RPT (SL = I1), else k*SL + ti*RPT
  for (int64_t q = 0; q < nq; ++q) {
    const int s = (int)(q % g.NST);
    const int64_t m0 = mbeg + q * g.CK;
    const int mc = (int)min((int64_t)g.CK, mend - m0);
    mbar_wait(&bars[s], (uint32_t)((q / g.NST) & 1));
    const T* ys = stages + (size_t)s * g.stage_elems;
    const T* ks = ys + kofs;
    if (row_ok) {
#pragma unroll 2
      for (int k = tm; k < mc; k += g.TM) {
        T y0[RPT], kv[RP];
        lds_rows<T, RPT>(ys + (size_t)k * g.SL + ti * RPT, y0);
#pragma unroll
        for (int r = 0; r < RP; r += 2) lds_pair(ks + k * RP + r, kv[r], kv[r + 1]);
#pragma unroll
        for (int r = 0; r < RP; ++r)
#pragma unroll
          for (int j = 0; j < RPT; ++j) fma_acc(acc[j][r], y0[j], kv[r]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars[g.NST + s]);
  }
  // multiply by conj(A_1) and reduce over the CTA
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    T v = zero_of<T>();
    if (row_ok) {
      v = mul(acc[0][r], ld_ro(A1c + i1_0 * RP + r));
#pragma unroll
      for (int j = 1; j < RPT; ++j)
        if (i1_0 + j < g.I1) fma_acc(v, acc[j][r], ld_ro(A1c + (i1_0 + j) * RP + r));
    }
    v = warp_sum(v);
    if (lane == 0) red[r * nw + wid] = v;
  }
  named_sync(1, nthr);
  if (tid < RP) {
    T sacc = zero_of<T>();
    for (int w = 0; w < nw; ++w) sacc = add(sacc, red[tid * nw + w]);
    part[((c * gridDim.y + blockIdx.y) * gridDim.z + blockIdx.z) * RP + tid] = sacc;
  }
}

// M_1 reduce over CTA groups (parallel): out[i1 + I1 r] = sum_g m1_part[g][i1][r], block of 8
// lanes per output, fixed order (lane-strided partial sums, then a fixed 8-way tree).
template <class T>
__global__ void k_m1_reduce(const T* __restrict__ m1_part, int ngroups, int64_t I1, int R, int RP, T* __restrict__ M1,
                            const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  const int64_t o = (int64_t)blockIdx.x * 32 + (threadIdx.x & 31);
  const int sub = threadIdx.x >> 5;  // 0..7
  __shared__ T sh[8][32];
  T acc = zero_of<T>();
  if (o < I1 * R) {
    const int64_t i = o % I1;
    const int r = (int)(o / I1);
    for (int g = sub; g < ngroups; g += 8) acc = add(acc, m1_part[((int64_t)g * I1 + i) * RP + r]);
  }
  sh[sub][threadIdx.x & 31] = acc;
  __syncthreads();
  if (sub == 0 && o < I1 * R) {
    T sacc = sh[0][threadIdx.x];
    for (int q = 1; q < 8; ++q) sacc = add(sacc, sh[q][threadIdx.x]);
    M1[o] = sacc;
  }
}

// Z reduce over i1 tiles: Z[m + Lmid r] = sum_t z_part[t][m][r]
template <class T>
__global__ void k_z_reduce(const T* __restrict__ z_part, int ntiles, int64_t Lmid, int R, int RP, T* __restrict__ Z,
                           const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Lmid * R) return;
  const int64_t m = idx % Lmid;
  const int r = (int)(idx / Lmid);
  T sacc = z_part[m * RP + r];
  for (int t = 1; t < ntiles; ++t) sacc = add(sacc, z_part[((int64_t)t * Lmid + m) * RP + r]);
  Z[idx] = sacc;
}

}  // namespace cpf

namespace cpf {

// Unfolding Gram G_n = Y_(n) Y_(n)^H (I_n x I_n) for the SVD initialisation (kruskal.py:227-242:
// the leading left singular vectors of Y_(n) are the leading eigenvectors of G_n).
// Y_(n)[i, k] with k = a + P b  ->  Y[a + P i + P I_n b]  (a over modes < n, b over modes > n).
// grid (tiles_i * tiles_j, ksplit); 32x32 output tile per CTA, 256 threads x (2x2); per-CTA partial
// tiles are summed by k_gram_reduce in fixed order.  Cross form (sharded mode-N Gram): the
// column operand comes from Yb with Inb columns, G = Y_(n) Yb_(n)^H (In x Inb); Yb = Y, Inb = In
// is the plain Gram.
template <class T>
__global__ void __launch_bounds__(256) k_unfold_gram(const T* __restrict__ Y, const T* __restrict__ Yb, int64_t P,
                                                     int64_t In, int64_t Inb, int64_t Q, int64_t kchunk,
                                                     T* __restrict__ part) {
  pdl_wait();
  __shared__ T As[32][33];
  __shared__ T Bs[32][33];
  const int ntile = (int)((In + 31) / 32);
  const int ti = blockIdx.x % ntile, tj = blockIdx.x / ntile;
  const int64_t K = P * Q;
  const int64_t kbeg = (int64_t)blockIdx.y * kchunk, kend = min(K, kbeg + kchunk);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  T acc[2][2];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) acc[u][v] = zero_of<T>();
  for (int64_t k0 = kbeg; k0 < kend; k0 += 32) {
    for (int e = threadIdx.x; e < 32 * 32; e += 256) {
      int kk, ii;
      if (P == 1) { ii = e % 32; kk = e / 32; } else { kk = e % 32; ii = e / 32; }
      const int64_t k = k0 + kk;
      const int64_t gi = (int64_t)ti * 32 + ii, gj = (int64_t)tj * 32 + ii;
      T va = zero_of<T>(), vb = zero_of<T>();
      if (k < kend) {
        const int64_t a = k % P, b = k / P;
        const int64_t base = a + P * In * b;
        if (gi < In) va = Y[base + P * gi];
        if (gj < Inb) vb = Yb[base + P * gj];
      }
      As[kk][ii] = va;
      Bs[kk][ii] = vb;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      const T a0 = As[kk][ty], a1 = As[kk][ty + 16];
      const T b0 = cj(Bs[kk][tx]), b1 = cj(Bs[kk][tx + 16]);
      fma_acc(acc[0][0], a0, b0);
      fma_acc(acc[0][1], a0, b1);
      fma_acc(acc[1][0], a1, b0);
      fma_acc(acc[1][1], a1, b1);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int64_t gi = (int64_t)ti * 32 + ty + 16 * u, gj = (int64_t)tj * 32 + tx + 16 * v;
      if (gi < In && gj < Inb) part[((int64_t)blockIdx.y * Inb + gj) * In + gi] = acc[u][v];  // column-major
    }
}

template <class T>
__global__ void k_gram_reduce(const T* __restrict__ part, int nsplit, int64_t n2, T* __restrict__ G) {
  pdl_wait();
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n2) return;
  T s = part[e];
  for (int q = 1; q < nsplit; ++q) s = add(s, part[(int64_t)q * n2 + e]);
  G[e] = s;
}

}  // namespace cpf
