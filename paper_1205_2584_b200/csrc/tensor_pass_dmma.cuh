// Tensor passes on the fp64 tensor cores (mma.sync.aligned.m8n8k4.row.col.f64 -> SASS DMMA.8x8x4).
//
// Used for float64 tensors whose mode-1 extent is large (I1 >= 256, e.g. BASELINE config 4), where a
// CTA tile of 512 consecutive i1 rows shares one m.  Both passes are GEMMs with a tall-skinny
// output (rows = i1, cols = R padded to 8*NT):
//   MODE 0 (pass A): per m:  P_m[i1, :] = sum_c Y[i1, m, c] conj(A_N[c, :])      K = local c
//                    M1[i1, :] += P_m[i1, :] o conj(KRmid[m, :])   (shared-memory accumulator)
//                    Z[m, :]    = sum_i1 P_m[i1, :] o conj(A_1[i1, :])
//   MODE 1 (pass B): per c:  U_c[i1, :] = sum_m Y[i1, m, c] conj(KRmid[m, :])   K = m chunk
//                    M_N[c, :] (partial) = sum_i1 U_c[i1, :] o conj(A_1[i1, :])
// Data movement is the same warp-specialised TMA bulk-copy ring as tensor_pass2.cuh (one producer
// warp, full/empty mbarriers); each stage holds CK K-rows of 512 Y values (padded stride 516 so the
// A-fragment loads are bank-conflict free) and CK operand rows (stride WS = 8*NT + 4).
// Warp w owns rows [64 w, 64 w + 64): 8 m8-tiles x NT n8-tiles of accumulators (2 doubles each).
#pragma once
#include "cpf_common.cuh"
#include "small_ops.cuh"
#include "tensor_pass2.cuh"

namespace cpf {

constexpr int kDmmaRows = 512;   // rows (i1) per CTA tile
constexpr int kDmmaSLp = 516;    // padded smem row stride (== 4 mod 16 doubles)
constexpr int kDmmaCK = 16;      // K rows per pipeline stage

struct DmmaGeom {
  int64_t I1, Lmid, C;
  int tiles;           // ceil(I1 / 512)
  int CK;              // K rows per stage (multiple of 4)
  int NST;             // stages
  int WS;              // operand row stride in global and smem (8*NT + 4)
  int64_t m_per_cta;   // MODE 0: m range per CTA; MODE 1: m chunk per CTA
  size_t stage_elems;  // doubles per stage
};

__device__ __forceinline__ void dmma8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int NT, int MODE, int CKT>
__global__ void __launch_bounds__(kConsumers + 32, 1) k_pass_dmma(const double* __restrict__ Y, DmmaGeom g,
                                                                  const double* __restrict__ Op,   // K rows x WS
                                                                  const double* __restrict__ A1c,  // I1 x RPg
                                                                  const double* __restrict__ KMc,  // Lmid x RPg
                                                                  int RPg, int R, double* __restrict__ z_part,
                                                                  double* __restrict__ m1_part, const LmDeviceState* st,
                                                                  const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  constexpr int NCOL = 8 * NT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  double* stages = reinterpret_cast<double*>(smem_raw + 128);
  double* red = stages + (size_t)g.NST * g.stage_elems;  // [8 warps][NCOL]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int64_t tile = blockIdx.x;
  const int64_t a0 = tile * kDmmaRows;
  const int64_t rows_valid = min((int64_t)kDmmaRows, g.I1 - a0);
  const int64_t Lrows = g.I1 * g.Lmid;
  int64_t kbeg, kend, nrb;  // K range and number of row blocks
  int64_t mbeg = 0, mend = 0, cfix = 0;
  if (MODE == 0) {
    mbeg = (int64_t)blockIdx.y * g.m_per_cta;
    mend = min(g.Lmid, mbeg + g.m_per_cta);
    if (mbeg >= mend) return;
    kbeg = 0;
    kend = g.C;
    nrb = mend - mbeg;
  } else {
    cfix = blockIdx.y;
    mbeg = (int64_t)blockIdx.z * g.m_per_cta;
    mend = min(g.Lmid, mbeg + g.m_per_cta);
    if (mbeg >= mend) return;
    kbeg = mbeg;
    kend = mend;
    nrb = 1;
  }
  const int64_t nkc = (kend - kbeg + CKT - 1) / CKT;  // chunks per row block
  const int64_t nq = nrb * nkc;
  const size_t oofs = (size_t)CKT * kDmmaSLp;
  const uint32_t ybytes = (uint32_t)(rows_valid * sizeof(double));

  auto issue = [&](int64_t q) {
    const int s = (int)(q % g.NST);
    const int64_t rb = q / nkc, kc = q % nkc;
    const int64_t k0 = kbeg + kc * CKT;
    const int ck = (int)min((int64_t)CKT, kend - k0);
    double* dst = stages + (size_t)s * g.stage_elems;
    const uint32_t obytes = (uint32_t)(ck * g.WS * sizeof(double));
    fence_proxy_async();
    mbar_expect_tx(&bars[s], ybytes * ck + obytes);
    if (MODE == 0) {
      const double* src = Y + a0 + g.I1 * (mbeg + rb) + Lrows * k0;
      for (int k = 0; k < ck; ++k) bulk_g2s(dst + (size_t)k * kDmmaSLp, src + Lrows * k, ybytes, &bars[s]);
    } else {
      const double* src = Y + Lrows * cfix + a0 + g.I1 * k0;
      for (int k = 0; k < ck; ++k) bulk_g2s(dst + (size_t)k * kDmmaSLp, src + g.I1 * k, ybytes, &bars[s]);
    }
    bulk_g2s(dst + oofs, Op + k0 * g.WS, obytes, &bars[s]);
  };

  if (tid == 0) {
    for (int s = 0; s < g.NST; ++s) {
      mbar_init(&bars[s], 1);
      mbar_init(&bars[g.NST + s], kConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid >= kConsumers) {  // ---- producer warp
    if (lane == 0)
      for (int64_t q = 0; q < nq; ++q) {
        const int s = (int)(q % g.NST);
        if (q >= g.NST) mbar_wait(&bars[g.NST + s], (uint32_t)(((q / g.NST) - 1) & 1));
        issue(q);
      }
    return;
  }

  double acc[8][NT][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int rbase = wid * 64;
  // MODE 0: the CTA's M_1 partial accumulates in place in m1_part (global, L2-resident: 96 KB per
  // CTA, read-modify-written once per row block = once per C/4 k-steps)
  double* m1g = m1_part + (int64_t)blockIdx.y * g.I1 * RPg;
  if (MODE == 0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t row = rbase + 8 * i + gq;
      if (row >= rows_valid) continue;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 8 * j + 2 * tq + h;
          if (col < R) m1g[(a0 + row) * RPg + col] = 0.0;
        }
    }
  }

  int64_t rb = 0, kc = 0;
  int s = 0;
  uint32_t ph = 0;
  for (int64_t q = 0; q < nq; ++q) {
    const int64_t k0 = kbeg + kc * CKT;
    const int ck = (int)min((int64_t)CKT, kend - k0);
    mbar_wait(&bars[s], ph);
    const double* ys = stages + (size_t)s * g.stage_elems;
    const double* os = ys + oofs;
    double af[2][8], bf[2][NT];
    auto load_frag = [&](int step, int b) {
      const int kk = 4 * step + tq;
      const bool kv = kk < ck;
#pragma unroll
      for (int i = 0; i < 8; ++i) af[b][i] = kv ? ys[(size_t)kk * kDmmaSLp + rbase + 8 * i + gq] : 0.0;
#pragma unroll
      for (int j = 0; j < NT; ++j) bf[b][j] = kv ? os[(size_t)kk * g.WS + 8 * j + gq] : 0.0;
    };
    load_frag(0, 0);
#pragma unroll
    for (int step = 0; step < CKT / 4; ++step) {
      if (step + 1 < CKT / 4) load_frag(step + 1, (step + 1) & 1);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma8x8x4(acc[i][j][0], acc[i][j][1], af[step & 1][i], bf[step & 1][j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars[g.NST + s]);
    if (++s == g.NST) { s = 0; ph ^= 1u; }

    if (MODE == 0 && kc == nkc - 1) {
      // ---- row-block epilogue for m = mbeg + rb
      const int64_t m = mbeg + rb;
      double zt[NT][2];
#pragma unroll
      for (int j = 0; j < NT; ++j) zt[j][0] = zt[j][1] = 0.0;
      double km[NT][2];
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 8 * j + 2 * tq + h;
          km[j][h] = col < R ? __ldg(KMc + m * RPg + col) : 0.0;
        }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t row = rbase + 8 * i + gq;
        const bool rv = row < rows_valid;
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int col = 8 * j + 2 * tq + h;
            const double p = acc[i][j][h];
            if (rv && col < R) {
              double* mp = m1g + (a0 + row) * RPg + col;
              *mp = fma(p, km[j][h], *mp);
              zt[j][h] = fma(p, __ldg(A1c + (a0 + row) * RPg + col), zt[j][h]);
            }
            acc[i][j][h] = 0.0;
          }
      }
      // reduce zt over the 8 row-groups (gq) of the warp, then over warps
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double v = zt[j][h];
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 8);
          v += __shfl_xor_sync(0xffffffffu, v, 16);
          if (gq == 0) red[wid * NCOL + 8 * j + 2 * tq + h] = v;
        }
      named_sync(1, kConsumers);
      if (tid < R) {
        double sacc = red[tid];
        for (int w = 1; w < 8; ++w) sacc += red[w * NCOL + tid];
        z_part[(tile * g.Lmid + m) * RPg + tid] = sacc;
      }
      named_sync(1, kConsumers);
    }
    if (++kc == nkc) { kc = 0; ++rb; }
  }

  if (MODE == 1) {
    // M_N partial: sum_i1 U[i1, col] conj(A_1[i1, col]) over the CTA's rows
    double zt[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) zt[j][0] = zt[j][1] = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t row = rbase + 8 * i + gq;
      const bool rv = row < rows_valid;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 8 * j + 2 * tq + h;
          if (rv && col < R) zt[j][h] = fma(acc[i][j][h], __ldg(A1c + (a0 + row) * RPg + col), zt[j][h]);
        }
    }
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double v = zt[j][h];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if (gq == 0) red[wid * NCOL + 8 * j + 2 * tq + h] = v;
      }
    named_sync(1, kConsumers);
    if (tid < R) {
      double sacc = red[tid];
      for (int w = 1; w < 8; ++w) sacc += red[w * NCOL + tid];
      // same layout as k_pass_b2: part[((c * chunks + chunk) * tiles + tile) * RPg + r]
      m1_part[((cfix * gridDim.z + blockIdx.z) * gridDim.x + tile) * RPg + tid] = sacc;
    }
  }
}

}  // namespace cpf

namespace cpf {

// Persistent pass B (MODE 1 of k_pass_dmma) over a bounded number of CTAs: every CTA loops over
// work items (tile, c, m-chunk), the TMA ring and its mbarrier phases continue across items.
// Launched with fewer CTAs than SMs when it runs concurrently with the LU of the next step, so
// the LU's panel cluster always finds free SMs.
template <int NT, int CKT>
__global__ void __launch_bounds__(kConsumers + 32, 1) k_pass_b_dmma_pers(const double* __restrict__ Y, DmmaGeom g,
                                                                         const double* __restrict__ Op,
                                                                         const double* __restrict__ A1c, int RPg, int R,
                                                                         int ncloc, int nchunks,
                                                                         double* __restrict__ part,
                                                                         const LmDeviceState* st, const DevFlags* fl,
                                                                         int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  constexpr int NCOL = 8 * NT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  double* stages = reinterpret_cast<double*>(smem_raw + 128);
  double* red = stages + (size_t)g.NST * g.stage_elems;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int64_t Lrows = g.I1 * g.Lmid;
  const int64_t nitems = (int64_t)g.tiles * ncloc * nchunks;
  const size_t oofs = (size_t)CKT * kDmmaSLp;
  // item -> (tile, c, chunk) with the tile fastest so concurrent CTAs share the same c (L2 locality)
  auto decode = [&](int64_t it, int64_t& tile, int64_t& c, int64_t& mb, int64_t& me) {
    tile = it % g.tiles;
    const int64_t rest = it / g.tiles;
    c = rest % ncloc;
    const int64_t ch = rest / ncloc;
    mb = ch * g.m_per_cta;
    me = min(g.Lmid, mb + g.m_per_cta);
  };
  if (tid == 0) {
    for (int s = 0; s < g.NST; ++s) {
      mbar_init(&bars[s], 1);
      mbar_init(&bars[g.NST + s], kConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid >= kConsumers) {  // ---- producer warp: all chunks of all my items
    if (lane == 0) {
      int64_t q = 0;
      for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        int64_t tile, c, mb, me;
        decode(it, tile, c, mb, me);
        const int64_t a0 = tile * kDmmaRows;
        const int64_t rows_valid = min((int64_t)kDmmaRows, g.I1 - a0);
        const uint32_t ybytes = (uint32_t)(rows_valid * sizeof(double));
        for (int64_t k0 = mb; k0 < me; k0 += CKT, ++q) {
          const int s = (int)(q % g.NST);
          if (q >= g.NST) mbar_wait(&bars[g.NST + s], (uint32_t)(((q / g.NST) - 1) & 1));
          const int ck = (int)min((int64_t)CKT, me - k0);
          double* dst = stages + (size_t)s * g.stage_elems;
          const uint32_t obytes = (uint32_t)(ck * g.WS * sizeof(double));
          fence_proxy_async();
          mbar_expect_tx(&bars[s], ybytes * ck + obytes);
          const double* src = Y + Lrows * c + a0 + g.I1 * k0;
          for (int k = 0; k < ck; ++k) bulk_g2s(dst + (size_t)k * kDmmaSLp, src + g.I1 * k, ybytes, &bars[s]);
          bulk_g2s(dst + oofs, Op + k0 * g.WS, obytes, &bars[s]);
        }
      }
    }
    return;
  }
  const int rbase = wid * 64;
  int s = 0;
  uint32_t ph = 0;
  for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    int64_t tile, c, mb, me;
    decode(it, tile, c, mb, me);
    const int64_t a0 = tile * kDmmaRows;
    const int64_t rows_valid = min((int64_t)kDmmaRows, g.I1 - a0);
    double acc[8][NT][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int64_t k0 = mb; k0 < me; k0 += CKT) {
      const int ck = (int)min((int64_t)CKT, me - k0);
      mbar_wait(&bars[s], ph);
      const double* ys = stages + (size_t)s * g.stage_elems;
      const double* os = ys + oofs;
      double af[2][8], bf[2][NT];
      auto load_frag = [&](int step, int b) {
        const int kk = 4 * step + tq;
        const bool kv = kk < ck;
#pragma unroll
        for (int i = 0; i < 8; ++i) af[b][i] = kv ? ys[(size_t)kk * kDmmaSLp + rbase + 8 * i + gq] : 0.0;
#pragma unroll
        for (int j = 0; j < NT; ++j) bf[b][j] = kv ? os[(size_t)kk * g.WS + 8 * j + gq] : 0.0;
      };
      load_frag(0, 0);
#pragma unroll
      for (int step = 0; step < CKT / 4; ++step) {
        if (step + 1 < CKT / 4) load_frag(step + 1, (step + 1) & 1);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma8x8x4(acc[i][j][0], acc[i][j][1], af[step & 1][i], bf[step & 1][j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[g.NST + s]);
      if (++s == g.NST) { s = 0; ph ^= 1u; }
    }
    // item epilogue: sum_i1 U[i1, col] conj(A_1[i1, col])
    double zt[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) zt[j][0] = zt[j][1] = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t row = rbase + 8 * i + gq;
      const bool rv = row < rows_valid;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 8 * j + 2 * tq + h;
          if (rv && col < R) zt[j][h] = fma(acc[i][j][h], __ldg(A1c + (a0 + row) * RPg + col), zt[j][h]);
        }
    }
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double v = zt[j][h];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if (gq == 0) red[wid * NCOL + 8 * j + 2 * tq + h] = v;
      }
    named_sync(1, kConsumers);
    if (tid < R) {
      double sacc = red[tid];
      for (int w = 1; w < 8; ++w) sacc += red[w * NCOL + tid];
      const int64_t ch = (it / g.tiles) / ncloc;
      part[((c * nchunks + ch) * g.tiles + tile) * RPg + tid] = sacc;
    }
    named_sync(1, kConsumers);
  }
}

}  // namespace cpf
