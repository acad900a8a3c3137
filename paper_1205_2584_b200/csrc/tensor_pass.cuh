// The O(J R) tensor passes: all-mode MTTKRP of a column-major dense tensor.
//
// Reference: cpfast/kruskal.py:126-135 (mttkrp = unfold(Y, n) @ conj(KR_{k!=n})) called N
// times per accepted iteration (solver.py:364-366), plus the full reconstruction inside
// relative_error (kruskal.py:159-167) every iteration.  Here the tensor is never unfolded
// or reconstructed: Y (column-major, mode 1 fastest) is viewed as a 3-level array
//     Y[i1, m, c]   i1 in [0,I1), m in [0,Lmid) (modes 2..N-1, mode 2 fastest), c in the
//                   local slab of mode N
// and two streaming passes produce every MTTKRP:
//   pass A ("contract mode N"):   P[i1,m,r] = sum_c Y[i1,m,c] conj(A_N[c,r])
//        M_1[i1,r] = sum_m P conj(KRmid[m,r])      Z[m,r] = sum_i1 P conj(A_1[i1,r])
//        (M_2..M_{N-1} are small contractions of Z; <Y,X> = sum M_1 conj(A_1))
//   pass B ("contract modes 1..N-1"):
//        M_N[c,r] = sum_i1 conj(A_1[i1,r]) sum_m Y[i1,m,c] conj(KRmid[m,r])
// Both passes read Y exactly once with coalesced loads along i1 and perform R (complex: 4R)
// FMAs per element; the Khatri-Rao rows are never materialised beyond KRmid (Lmid x R).
// All cross-CTA reductions go through fixed-order workspaces (bit-reproducible results).
#pragma once
#include "cpf_common.cuh"
#include "small_ops.cuh"

namespace cpf {

// Row-major conj copies used by the passes: dst[i*RP + r] = conj(src[i + ld*r]) (r<R), 0 pad.
template <class T>
__global__ void k_conj_rowmajor(const T* __restrict__ src, int64_t rows, int64_t row0, int64_t ld, int R, int RP,
                                T* __restrict__ dst, const LmDeviceState* st, const DevFlags* fl, int gate,
                                int do_conj = 1) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * RP) return;
  int64_t i = idx / RP;
  int r = (int)(idx % RP);
  T v = r < R ? src[(row0 + i) + ld * r] : zero_of<T>();
  dst[idx] = do_conj ? cj(v) : v;
}

// KRmid[m, r] = prod_{k=2..N-1} A_k[i_k(m), r]  (conj, row-major, padded).  m: mode 2 fastest.
struct MidGeom {
  int nmid;               // N - 2
  int64_t dims[6];        // dims of modes 2..N-1
  int64_t offs[6];        // offsets of those factors in the stacked factor vector
};

template <class T>
__global__ void k_krmid(const T* __restrict__ A, MidGeom g, int64_t Lmid, int R, int RP, T* __restrict__ dst,
                        const LmDeviceState* st, const DevFlags* fl, int gate, int do_conj = 1) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= Lmid * RP) return;
  int64_t m = idx / RP;
  int r = (int)(idx % RP);
  if (r >= R) { dst[idx] = zero_of<T>(); return; }
  T v = from_real<T>(1.0);
  int64_t rem = m;
  for (int k = 0; k < g.nmid; ++k) {
    int64_t ik = rem % g.dims[k];
    rem /= g.dims[k];
    v = k == 0 ? A[g.offs[k] + ik + g.dims[k] * r] : mul(v, A[g.offs[k] + ik + g.dims[k] * r]);
  }
  dst[idx] = do_conj ? cj(v) : v;
}

constexpr int kPassCK = 32;  // W rows staged in shared memory per step

// Fused pass A.  CTA = (i1 tile, m group).  Thread (ti, tm): i1 = tile*TI + ti, handles
// m = m0 + tm, m0 + tm + TM, ... inside the CTA's m range.  For each (i1, m) it accumulates the
// P row over all c in registers, then
//   * adds P*conj(KRmid[m]) into its private M_1 accumulator (shared memory, per thread),
//   * writes P*conj(A_1[i1]) for the Z reduction into shared memory, reduced over ti by the
//     threads of the same tm group after a barrier.
// Outputs (fixed-order partials):
//   z_part[(tile) * Lmid*RP + m*RP + r]      (reduced over the CTA's i1 tile)
//   m1_part[(mgrp) * I1*RP + i1*RP + r]      (reduced over the CTA's m range)
template <class T, int RP>
__global__ void __launch_bounds__(256) k_pass_a(const T* __restrict__ Y, int64_t I1, int64_t Lmid, int64_t C,
                                                const T* __restrict__ WNc,  // C x RP (conj A_N slab)
                                                const T* __restrict__ A1c,  // I1 x RP
                                                const T* __restrict__ KMc,  // Lmid x RP
                                                int TI, int TM, int64_t m_per_cta,
                                                T* __restrict__ z_part, T* __restrict__ m1_part,
                                                const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* w_s = reinterpret_cast<T*>(smem_raw);                 // kPassCK * RP
  T* m1_s = w_s + kPassCK * RP;                            // blockDim * RP   ([r][thread])
  T* z_s = m1_s + (size_t)blockDim.x * RP;                 // blockDim * RP   ([r][thread])
  const int tid = threadIdx.x;
  const int nthr = blockDim.x;
  const int ti = tid % TI, tm = tid / TI;
  const int64_t tile = blockIdx.x;
  const int64_t i1 = tile * TI + ti;
  const bool row_ok = (tm < TM) && (i1 < I1);
  const int64_t Lrows = I1 * Lmid;
  const int64_t mbeg = (int64_t)blockIdx.y * m_per_cta;
  const int64_t mend = min(Lmid, mbeg + m_per_cta);

#pragma unroll
  for (int r = 0; r < RP; ++r) m1_s[r * nthr + tid] = zero_of<T>();

  // all threads iterate the same number of m-rounds so barriers stay uniform
  const int64_t span = mend - mbeg;
  const int64_t rounds = (span + TM - 1) / TM;
  for (int64_t rd = 0; rd < rounds; ++rd) {
    const int64_t m = mbeg + rd * TM + tm;
    const bool ok = row_ok && (m < mend);
    T acc[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) acc[r] = zero_of<T>();
    const T* yrow = Y + (ok ? (i1 + I1 * m) : 0);
    for (int64_t c0 = 0; c0 < C; c0 += kPassCK) {
      const int ck = (int)(C - c0 < (int64_t)kPassCK ? C - c0 : (int64_t)kPassCK);
      __syncthreads();
      for (int e = tid; e < ck * RP; e += nthr) w_s[e] = WNc[c0 * RP + e];
      __syncthreads();
      if (ok) {
        int k = 0;
        for (; k + 4 <= ck; k += 4) {
          T y0 = ld_stream(yrow + Lrows * (c0 + k));
          T y1 = ld_stream(yrow + Lrows * (c0 + k + 1));
          T y2 = ld_stream(yrow + Lrows * (c0 + k + 2));
          T y3 = ld_stream(yrow + Lrows * (c0 + k + 3));
#pragma unroll
          for (int r = 0; r < RP; ++r) {
            fma_acc(acc[r], y0, w_s[(k + 0) * RP + r]);
            fma_acc(acc[r], y1, w_s[(k + 1) * RP + r]);
            fma_acc(acc[r], y2, w_s[(k + 2) * RP + r]);
            fma_acc(acc[r], y3, w_s[(k + 3) * RP + r]);
          }
        }
        for (; k < ck; ++k) {
          T y0 = ld_stream(yrow + Lrows * (c0 + k));
#pragma unroll
          for (int r = 0; r < RP; ++r) fma_acc(acc[r], y0, w_s[k * RP + r]);
        }
      }
    }
    // epilogue for this (i1, m)
    if (ok) {
      const T* km = KMc + m * RP;
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        T t = m1_s[r * nthr + tid];
        fma_acc(t, acc[r], km[r]);
        m1_s[r * nthr + tid] = t;
        z_s[r * nthr + tid] = mul(acc[r], ld_ro(A1c + i1 * RP + r));
      }
    } else {
#pragma unroll
      for (int r = 0; r < RP; ++r) z_s[r * nthr + tid] = zero_of<T>();
    }
    __syncthreads();
    // reduce z over ti for each tm group: thread (ti, tm) with ti < RP handles r = ti
    if (tm < TM) {
      for (int r = ti; r < RP; r += TI) {
        const int64_t mm = mbeg + rd * TM + tm;
        if (mm < mend) {
          T s = zero_of<T>();
          const T* zz = z_s + r * nthr + tm * TI;
          for (int q = 0; q < TI; ++q) s = add(s, zz[q]);
          z_part[tile * Lmid * RP + mm * RP + r] = s;
        }
      }
    }
  }
  __syncthreads();
  if (row_ok) {
    // reduce m1 over the TM groups sharing this i1: group tm==0 sums in fixed order
    if (tm == 0) {
      for (int r = 0; r < RP; ++r) {
        T s = zero_of<T>();
        for (int q = 0; q < TM; ++q) s = add(s, m1_s[r * nthr + q * TI + ti]);
        m1_part[(int64_t)blockIdx.y * I1 * RP + i1 * RP + r] = s;
      }
    }
  }
}

// Reduce pass-A partials: M1[i1 + I1*r] = sum_g m1_part[g][i1][r];  Z[m + Lmid*r] = sum_t z_part[t][m][r]
template <class T>
__global__ void k_pass_a_reduce(const T* __restrict__ m1_part, int ngroups, const T* __restrict__ z_part, int ntiles,
                                int64_t I1, int64_t Lmid, int R, int RP, T* __restrict__ M1, T* __restrict__ Z,
                                const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n1 = I1 * R, n2 = Lmid * R;
  if (idx < n1) {
    int64_t i = idx % I1;
    int r = (int)(idx / I1);
    T s = zero_of<T>();
    for (int g = 0; g < ngroups; ++g) s = add(s, m1_part[(int64_t)g * I1 * RP + i * RP + r]);
    M1[idx] = s;
  } else if (idx < n1 + n2) {
    int64_t j = idx - n1;
    int64_t m = j % Lmid;
    int r = (int)(j / Lmid);
    T s = zero_of<T>();
    for (int t = 0; t < ntiles; ++t) s = add(s, z_part[(int64_t)t * Lmid * RP + m * RP + r]);
    Z[j] = s;
  }
}

// ------------------------------------------------------------------------------------------
// Pass B: CTA = (c, m chunk, i1 tile).  Thread (ti, tm) accumulates
//   U[r] = sum_{m in chunk, m = m0+tm (mod TM)} Y[i1, m, c] conj(KRmid[m, r])
// then multiplies by conj(A_1[i1, r]) and the CTA reduces over all its threads.
// ------------------------------------------------------------------------------------------
template <class T, int RP>
__global__ void __launch_bounds__(256) k_pass_b(const T* __restrict__ Y, int64_t I1, int64_t Lmid, int64_t C,
                                                const T* __restrict__ A1c, const T* __restrict__ KMc,
                                                int TI, int TM, int64_t m_per_cta, T* __restrict__ part,
                                                const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* red = reinterpret_cast<T*>(smem_raw);  // RP * (blockDim/32)
  const int tid = threadIdx.x;
  const int ti = tid % TI, tm = tid / TI;
  const int64_t c = blockIdx.x;
  const int64_t i1 = (int64_t)blockIdx.z * TI + ti;
  const bool row_ok = (tm < TM) && (i1 < I1);
  const int64_t Lrows = I1 * Lmid;
  const int64_t mbeg = (int64_t)blockIdx.y * m_per_cta;
  const int64_t mend = min(Lmid, mbeg + m_per_cta);
  T acc[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) acc[r] = zero_of<T>();
  if (row_ok) {
    const T* ycol = Y + Lrows * c + i1;
    int64_t m = mbeg + tm;
    for (; m + 3 * TM < mend; m += 4 * TM) {
      T y0 = ld_stream(ycol + I1 * m);
      T y1 = ld_stream(ycol + I1 * (m + TM));
      T y2 = ld_stream(ycol + I1 * (m + 2 * TM));
      T y3 = ld_stream(ycol + I1 * (m + 3 * TM));
      const T* k0 = KMc + m * RP;
      const T* k1 = KMc + (m + TM) * RP;
      const T* k2 = KMc + (m + 2 * TM) * RP;
      const T* k3 = KMc + (m + 3 * TM) * RP;
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        fma_acc(acc[r], y0, ld_ro(k0 + r));
        fma_acc(acc[r], y1, ld_ro(k1 + r));
        fma_acc(acc[r], y2, ld_ro(k2 + r));
        fma_acc(acc[r], y3, ld_ro(k3 + r));
      }
    }
    for (; m < mend; m += TM) {
      T y0 = ld_stream(ycol + I1 * m);
      const T* k0 = KMc + m * RP;
#pragma unroll
      for (int r = 0; r < RP; ++r) fma_acc(acc[r], y0, ld_ro(k0 + r));
    }
#pragma unroll
    for (int r = 0; r < RP; ++r) acc[r] = mul(acc[r], A1c[i1 * RP + r]);
  }
  // block reduction of RP values
  const int lane = tid & 31, wid = tid >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    T v = warp_sum(acc[r]);
    if (lane == 0) red[r * nw + wid] = v;
  }
  __syncthreads();
  if (tid < RP) {
    T s = zero_of<T>();
    for (int w = 0; w < nw; ++w) s = add(s, red[tid * nw + w]);
    part[((c * gridDim.y + blockIdx.y) * gridDim.z + blockIdx.z) * RP + tid] = s;
  }
}

// MN[c + ldm*r] = sum_{g} part[c][g][r]   (g over m-chunks x i1-tiles)
template <class T>
__global__ void k_pass_b_reduce(const T* __restrict__ part, int64_t C, int ng, int R, int RP, int64_t ldm,
                                T* __restrict__ MN, const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= C * R) return;
  int64_t c = idx % C;
  int r = (int)(idx / C);
  T s = zero_of<T>();
  for (int g = 0; g < ng; ++g) s = add(s, part[(c * ng + g) * RP + r]);
  MN[c + ldm * r] = s;
}

// Mid-mode MTTKRPs from Z (N >= 4): M_n[i_n, r] = sum_{m: i_n(m)=i_n} Z[m,r] conj(prod_{k!=n} A_k[i_k(m), r])
template <class T>
__global__ void k_mid_mttkrp(const T* __restrict__ Z, int64_t Lmid, const T* __restrict__ A, MidGeom g, int which,
                             int R, T* __restrict__ Mn, const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  const int64_t In = g.dims[which];
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= In * R) return;
  const int64_t in = idx % In;
  const int r = (int)(idx / In);
  // strides of the mid modes in m
  int64_t stride[6];
  int64_t s = 1;
  for (int k = 0; k < g.nmid; ++k) { stride[k] = s; s *= g.dims[k]; }
  const int64_t others = Lmid / In;
  T acc = zero_of<T>();
  for (int64_t q = 0; q < others; ++q) {
    // decode q over the other mid modes (ascending), build m and the KR product
    int64_t rem = q, m = in * stride[which];
    T kr = from_real<T>(1.0);
    bool first = true;
    for (int k = 0; k < g.nmid; ++k) {
      if (k == which) continue;
      int64_t ik = rem % g.dims[k];
      rem /= g.dims[k];
      m += ik * stride[k];
      T a = A[g.offs[k] + ik + g.dims[k] * r];
      kr = first ? a : mul(kr, a);
      first = false;
    }
    fma_cacc(acc, kr, Z[m + Lmid * r]);
  }
  Mn[idx] = acc;
}

// Direct residual ||Y - X||^2 (guard band and relative_error API; kruskal.py:159-167).
// Thread per row l = i1 + I1*m: p[r] = A_1[i1,r] KRmid[m,r] (non-conj), then for every local c
// x = sum_r p[r] A_N[c,r] and acc += |y - x|^2.  Per-block partials, fixed order.
template <class T, int RP>
__global__ void __launch_bounds__(256) k_direct_resid(const T* __restrict__ Y, int64_t I1, int64_t Lmid, int64_t C,
                                                      const T* __restrict__ WN, const T* __restrict__ A1r,
                                                      const T* __restrict__ KM, double* __restrict__ part,
                                                      const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* w_s = reinterpret_cast<T*>(smem_raw);
  __shared__ double scratch[32];
  const int64_t Lrows = I1 * Lmid;
  double acc = 0.0;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < Lrows; base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = base + threadIdx.x;
    const bool ok = l < Lrows;
    T p[RP];
    if (ok) {
      const int64_t i1 = l % I1, m = l / I1;
#pragma unroll
      for (int r = 0; r < RP; ++r) p[r] = mul(A1r[i1 * RP + r], KM[m * RP + r]);
    }
    for (int64_t c0 = 0; c0 < C; c0 += kPassCK) {
      const int ck = (int)(C - c0 < (int64_t)kPassCK ? C - c0 : (int64_t)kPassCK);
      __syncthreads();
      for (int e = threadIdx.x; e < ck * RP; e += blockDim.x) w_s[e] = WN[c0 * RP + e];
      __syncthreads();
      if (ok)
        for (int k = 0; k < ck; ++k) {
          T x = zero_of<T>();
#pragma unroll
          for (int r = 0; r < RP; ++r) fma_acc(x, p[r], w_s[k * RP + r]);
          acc += abs2(sub(Y[l + Lrows * (c0 + k)], x));
        }
    }
  }
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

}  // namespace cpf
