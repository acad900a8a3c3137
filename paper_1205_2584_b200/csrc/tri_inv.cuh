// Explicit inverse of the core system's LU factors, so that the three B-applications of a step
// (candidate + two refinement rounds) are triangular matrix-VECTOR products instead of
// latency-bound substitutions.  The reference itself applies an explicit inverse:
// B = np.linalg.inv(K^-1 + Psi) (hessian.py:196-211, LAPACK getri); here the inverse is kept
// factored, B w = inv(U) inv(L) P w.
//
// Storage: Inv (n x n, column-major) holds inv(L) strictly below the diagonal (unit diagonal
// implicit) and inv(U) on and above it -- the same packing as the LU factors.
// Algorithm (by block rows of inv(L) / block columns of inv(U), k_tri_row): block k needs the
// inverse of the leading blocks and block k of the factors, so the engine runs it on a side stream
// right behind the LU's step k (engine.cu tri_progress) and only the last block's step is left
// when the factorisation ends.  Used for n_B <= 1024 (config 2: 457 -> 473, config 3: 842 -> 875
// it/s over the pair form).  For larger systems the chain of per-block long products does not
// keep up with the panels beside config 4's pass B (measured 180-182 vs 188 it/s), so they use
// recursive doubling over block pairs (k_tri_level): fewer, larger products, each launched as soon
// as the LU has finalised the pair; the pairs that end at the last block stay behind the LU.
#pragma once
#include "cpf_common.cuh"

namespace cpf {

template <class T>
__global__ void __launch_bounds__(64) k_tri_inv_diag(const T* __restrict__ LU, int n, T* __restrict__ Inv,
                                                     const LmDeviceState* st, int gate_running, int blk0, int tstep) {
  pdl_wait();
  if (lu_gated(st, gate_running)) return;
  lu_trace(1, 256 + tstep, 0);
  __shared__ T blk[32][33];
  const int b0 = (blk0 + blockIdx.x) * 32;
  const int bs = min(32, n - b0);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int e = tid; e < 32 * 32; e += 64) {
    const int i = e % 32, j = e / 32;
    blk[i][j] = (i < bs && j < bs) ? LU[(int64_t)(b0 + i) + (int64_t)n * (b0 + j)] : zero_of<T>();
  }
  __syncthreads();
  const int c = lane;
  if (c >= bs) { lu_trace(1, 256 + tstep, 1); return; }
  T x[32];
  if (wid == 0) {
    // unit lower: x = inv(L) e_c, rows i > c
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      T v = from_real<T>(i == c ? 1.0 : 0.0);
#pragma unroll
      for (int j = 0; j < i; ++j) fms_acc(v, blk[i][j], x[j]);
      x[i] = i < c ? zero_of<T>() : v;
    }
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i > c && i < bs) Inv[(int64_t)(b0 + i) + (int64_t)n * (b0 + c)] = x[i];
  } else {
    // upper: x = inv(U) e_c, rows i <= c
#pragma unroll
    for (int i = 31; i >= 0; --i) {
      T v = from_real<T>(i == c ? 1.0 : 0.0);
#pragma unroll
      for (int j = i + 1; j < 32; ++j) fms_acc(v, blk[i][j], x[j]);
      x[i] = (i > c || i >= bs) ? zero_of<T>() : mul(v, rcp_of(blk[i][i]));
    }
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i <= c) Inv[(int64_t)(b0 + i) + (int64_t)n * (b0 + c)] = x[i];
  }
  lu_trace(1, 256 + tstep, 1);
}

// Operand kinds of the level products
enum TriOp { kOpFull = 0, kOpInvL = 1, kOpInvU = 2 };

template <class T>
__device__ __forceinline__ T tri_elem(const T* M, int n, int r, int c, int kind) {
  if (kind == kOpInvL) {
    if (r == c) return from_real<T>(1.0);
    if (r < c) return zero_of<T>();
  } else if (kind == kOpInvU) {
    if (r > c) return zero_of<T>();
  }
  return M[(int64_t)r + (int64_t)n * c];
}

// One product C = alpha * opA(A) * opB(B) of the block inverse, all blocks inside n x n column-major
// matrices; a CTA computes one 64x64 tile (fp64 on the DMMA tensor pipe, complex128 as DFMA; 16
// K-rows per smem stage).  Triangular operands skip the K range that only multiplies zeros.
// Split-K (ksplit > 1): split ks covers its share of the K range and writes alpha * partial into
// part[ks] (n x n layout); the reduce kernel adds the partials in fixed order -- deterministic.
template <class T>
struct TriProd {
  int m, nn, kk;            // C is m x nn, inner dimension kk
  const T* Am; int ra, ca, kindA;
  const T* Bm; int rb, cb, kindB;
  T* Cm; int rc, cc;
  double alpha;
};

template <class T>
__device__ __forceinline__ void tri_tile_product(const TriProd<T>& q, int n, int tm, int tn, int ks, int ksplit,
                                                 T* __restrict__ part, int tstep) {
  const int m = q.m, nn = q.nn, kk = q.kk, ra = q.ra, ca = q.ca, rb = q.rb, cb = q.cb, rc = q.rc, cc = q.cc;
  const int kindA = q.kindA, kindB = q.kindB;
  const T *Am = q.Am, *Bm = q.Bm;
  T* Cm = q.Cm;
  const double alpha = q.alpha;
  if (tm >= m || tn >= nn) return;
  lu_trace(1, 256 + tstep, 0);
  constexpr int KS = 16 * 8 / (int)sizeof(T);  // K rows per stage (8 for complex: 48 KB static smem)
  // triangular operands: skip the K range that only multiplies zeros
  int kbeg = 0, kend = kk;
  if (kindA == kOpInvL) kend = min(kend, tm + 64);  // row i needs k <= i
  if (kindA == kOpInvU) kbeg = tm;                   // row i needs k >= i
  if (kindB == kOpInvL) kbeg = max(kbeg, tn);        // col j needs k >= j
  if (kindB == kOpInvU) kend = min(kend, tn + 64);   // col j needs k <= j
  kbeg &= ~(KS - 1);
  if (ksplit > 1) {  // this split's share of [kbeg, kend), in whole K slabs
    const int per = ((max(kend - kbeg, 0) + ksplit - 1) / ksplit + KS - 1) / KS * KS;
    const int lo = kbeg + ks * per;
    kend = min(kend, lo + per);
    kbeg = lo;
  }
  if (ksplit > 1) Cm = part + (size_t)ks * n * n;
  __shared__ T As[2][KS][64 + 1];
  __shared__ T Bs[2][KS][64 + 1];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;  // 16 x 16 threads, 4 x 4 outputs each
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = zero_of<T>();
  // register-staged prefetch of the next K slab (KS x 64 of A and B: 4 + 4 elements per thread)
  constexpr int PER = 64 * KS / 256;
  T pa[PER], pb[PER];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const int e = tid + 256 * t;
      const int i = e % 64, q = e / 64;
      pa[t] = (tm + i < m && k0 + q < kend) ? tri_elem(Am, n, ra + tm + i, ca + k0 + q, kindA) : zero_of<T>();
      const int q2 = e % KS, j = e / KS;
      pb[t] = (k0 + q2 < kend && tn + j < nn) ? tri_elem(Bm, n, rb + k0 + q2, cb + tn + j, kindB) : zero_of<T>();
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const int e = tid + 256 * t;
      As[buf][e / 64][e % 64] = pa[t];
      Bs[buf][e % KS][e / KS] = pb[t];
    }
  };
  int buf = 0;
  if (kbeg < kend) {
    fetch(kbeg);
    stash(0);
  }
  __syncthreads();
  if constexpr (sizeof(T) == 8) {
    // fp64: the 64x64 tile on the tensor cores (mma.sync m8n8k4.f64 -> DMMA), 8 warps of 32x16:
    // per 4-deep K step 4 A and 2 B fragments feed 8 DMMAs (the SIMT loop needs 8 LDS per 16 FMA)
    const int lane = tid & 31, wid = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int wm = (wid & 1) * 32, wn = (wid >> 1) * 16;
    double dacc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) dacc[i][j][0] = dacc[i][j][1] = 0.0;
    for (int k0 = kbeg; k0 < kend; k0 += KS) {
      const bool more = k0 + KS < kend;
      if (more) fetch(k0 + KS);
#pragma unroll
      for (int q = 0; q < KS; q += 4) {
        double af[4], bf[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = As[buf][q + t4][wm + 8 * i + g];
#pragma unroll
        for (int j = 0; j < 2; ++j) bf[j] = Bs[buf][q + t4][wn + 8 * j + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(dacc[i][j][0]), "+d"(dacc[i][j][1])
                         : "d"(af[i]), "d"(bf[j]));
      }
      if (more) stash(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = tm + wm + 8 * i + g, c = tn + wn + 8 * j + 2 * t4 + h;
          if (r < m && c < nn) Cm[(int64_t)(rc + r) + (int64_t)n * (cc + c)] = alpha * dacc[i][j][h];
        }
    lu_trace(1, 256 + tstep, 1);
    return;
  } else {
    for (int k0 = kbeg; k0 < kend; k0 += KS) {
      const bool more = k0 + KS < kend;
      if (more) fetch(k0 + KS);
#pragma unroll
      for (int q = 0; q < KS; ++q) {
        T av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = As[buf][q][tx + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = Bs[buf][q][ty + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) fma_acc(acc[i][j], av[i], bv[j]);
      }
      if (more) stash(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = tm + tx + 16 * i, c = tn + ty + 16 * j;
        if (r < m && c < nn) Cm[(int64_t)(rc + r) + (int64_t)n * (cc + c)] = scale(acc[i][j], alpha);
      }
    lu_trace(1, 256 + tstep, 1);
  }
}

// Row-by-row form of the inverse (the order LAPACK's trtri uses, by block rows / columns): once the
// LU has finalised block k (rows/columns [r0, r0 + bs)), with the inverse of the leading part
// [base, r0) of its diagonal block already in Inv,
//   L:  Inv[k, base:r0] = -inv(L_kk) (L[k, base:r0] inv(L)[base:r0, base:r0])
//   U:  Inv[base:r0, k] = -(inv(U)[base:r0, base:r0] U[base:r0, k]) inv(U_kk)
// STEP 0 is the long product (K = r0 - base, needs only the leading inverse: it can run while the
// diagonal block is still being inverted), STEP 1 the bs-deep one.  blockIdx.x: 64-wide tile along
// the leading part, blockIdx.y: 64-wide tile along the block, blockIdx.z = tri * ksplit + ks (tri 0:
// L, 1: U).  The engine applies it at two granularities (tri_row_step): every 32-row LU block
// against the start of its group of G rows, and every completed group (bs = G) against the start of
// the inverse (base = 0: full inverse; the DB x DB diagonal block: block-inverse substitution).
template <class T, int STEP>
__global__ void __launch_bounds__(256) k_tri_row(const T* __restrict__ LU, T* __restrict__ Inv, T* __restrict__ Tmp,
                                                 int n, int r0, int bs, int base, const LmDeviceState* st,
                                                 int gate_running, int ksplit, T* __restrict__ part, int tstep) {
  pdl_wait();
  if (lu_gated(st, gate_running)) return;
  const int ks = blockIdx.z % ksplit, tri = blockIdx.z / ksplit;
  const int lead = r0 - base;
  TriProd<T> q;
  int tm, tn;
  if (tri == 0) {
    q.m = bs; q.nn = lead; tm = blockIdx.y * 64; tn = blockIdx.x * 64;
    if (STEP == 0) { q.kk = lead; q.Am = LU; q.ra = r0; q.ca = base; q.kindA = kOpFull; q.Bm = Inv; q.rb = base; q.cb = base; q.kindB = kOpInvL; q.Cm = Tmp; q.alpha = 1.0; }
    else { q.kk = bs; q.Am = Inv; q.ra = r0; q.ca = r0; q.kindA = kOpInvL; q.Bm = Tmp; q.rb = r0; q.cb = base; q.kindB = kOpFull; q.Cm = Inv; q.alpha = -1.0; }
    q.rc = r0; q.cc = base;
  } else {
    q.m = lead; q.nn = bs; tm = blockIdx.x * 64; tn = blockIdx.y * 64;
    if (STEP == 0) { q.kk = lead; q.Am = Inv; q.ra = base; q.ca = base; q.kindA = kOpInvU; q.Bm = LU; q.rb = base; q.cb = r0; q.kindB = kOpFull; q.Cm = Tmp; q.alpha = 1.0; }
    else { q.kk = bs; q.Am = Tmp; q.ra = base; q.ca = r0; q.kindA = kOpFull; q.Bm = Inv; q.rb = r0; q.cb = r0; q.kindB = kOpInvU; q.Cm = Inv; q.alpha = -1.0; }
    q.rc = base; q.cc = r0;
  }
  tri_tile_product(q, n, tm, tn, ks, ksplit, part, tstep);
}

// Sum of the split-K partials of a row step's long product (fixed order) into Tmp.  grid.y = 2.
template <class T>
__global__ void k_tri_row_reduce(T* __restrict__ Tmp, const T* __restrict__ part, int ksplit, int n, int r0, int bs,
                                 int base, const LmDeviceState* st, int gate_running, int tstep) {
  pdl_wait();
  if (lu_gated(st, gate_running)) return;
  const int tri = blockIdx.y, lead = r0 - base;
  const int rc = tri == 0 ? r0 : base, cc = tri == 0 ? base : r0;
  const int m = tri == 0 ? bs : lead, nn = tri == 0 ? lead : bs;
  const size_t nn2 = (size_t)n * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)m * nn; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % m), c = (int)(e / m);
    const size_t off = (size_t)(rc + r) + (size_t)n * (cc + c);
    T v = part[off];
    for (int k = 1; k < ksplit; ++k) v = add(v, part[(size_t)k * nn2 + off]);
    Tmp[off] = v;
  }
  lu_trace(1, 256 + tstep, 1);
}

// Recursive doubling over adjacent block pairs (the form used for n_B > 1024, where a chain of
// per-block products does not keep up with the panels beside config 4's pass B): level s merges
// blocks (b1, b2) of size s
//     L: inv([L11 0; L21 L22])  -> X21 = -inv(L22) (L21 inv(L11))
//     U: inv([U11 U12; 0 U22])  -> X12 = -inv(U11) (U12 inv(U22))
// blockIdx.z = (2 * (pair - pair0) + tri) * ksplit + ks (tri 0: L, 1: U).
//   step 0 (T):  L: T[b2,b1] = L21 * inv(L11)      U: T[b1,b2] = U12 * inv(U22)
//   step 1 (X):  L: X[b2,b1] = -inv(L22) * T        U: X[b1,b2] = -inv(U11) * T
template <class T, int STEP>
__global__ void __launch_bounds__(256) k_tri_level(const T* __restrict__ LU, T* __restrict__ Inv, T* __restrict__ Tmp,
                                                   int n, int s, const LmDeviceState* st, int gate_running,
                                                   int ksplit, T* __restrict__ part, int pair0, int tstep) {
  pdl_wait();
  if (lu_gated(st, gate_running)) return;
  const int ks = blockIdx.z % ksplit, pt = blockIdx.z / ksplit;
  const int pair = pair0 + (pt >> 1), tri = pt & 1;
  const int b1 = 2 * pair * s, b2 = b1 + s;
  if (b2 >= n) return;
  const int s1 = s, s2 = min(s, n - b2);
  TriProd<T> q;
  if (tri == 0) {  // L
    q.m = s2; q.nn = s1;
    if (STEP == 0) { q.kk = s1; q.Am = LU; q.ra = b2; q.ca = b1; q.kindA = kOpFull; q.Bm = Inv; q.rb = b1; q.cb = b1; q.kindB = kOpInvL; q.alpha = 1.0; q.Cm = Tmp; }
    else { q.kk = s2; q.Am = Inv; q.ra = b2; q.ca = b2; q.kindA = kOpInvL; q.Bm = Tmp; q.rb = b2; q.cb = b1; q.kindB = kOpFull; q.alpha = -1.0; q.Cm = Inv; }
    q.rc = b2; q.cc = b1;
  } else {  // U
    q.m = s1; q.nn = s2;
    if (STEP == 0) { q.kk = s2; q.Am = LU; q.ra = b1; q.ca = b2; q.kindA = kOpFull; q.Bm = Inv; q.rb = b2; q.cb = b2; q.kindB = kOpInvU; q.alpha = 1.0; q.Cm = Tmp; }
    else { q.kk = s1; q.Am = Inv; q.ra = b1; q.ca = b1; q.kindA = kOpInvU; q.Bm = Tmp; q.rb = b1; q.cb = b2; q.kindB = kOpFull; q.alpha = -1.0; q.Cm = Inv; }
    q.rc = b1; q.cc = b2;
  }
  tri_tile_product(q, n, (int)blockIdx.x * 64, (int)blockIdx.y * 64, ks, ksplit, part, tstep);
}

// Sum of the split-K partials of one level (fixed order) into its output blocks: STEP 0 -> Tmp,
// STEP 1 -> Inv.  grid.y = 2 * npairs (pair, triangle).
template <class T, int STEP>
__global__ void k_tri_reduce(T* __restrict__ Inv, T* __restrict__ Tmp, const T* __restrict__ part, int ksplit, int n,
                             int s, const LmDeviceState* st, int gate_running, int pair0, int tstep) {
  pdl_wait();
  if (lu_gated(st, gate_running)) return;
  const int pair = pair0 + (blockIdx.y >> 1), tri = blockIdx.y & 1;
  const int b1 = 2 * pair * s, b2 = b1 + s;
  if (b2 >= n) return;
  const int s1 = s, s2 = min(s, n - b2);
  const int rc = tri == 0 ? b2 : b1, cc = tri == 0 ? b1 : b2;
  const int m = tri == 0 ? s2 : s1, nn = tri == 0 ? s1 : s2;
  T* dst = STEP == 0 ? Tmp : Inv;
  const size_t nn2 = (size_t)n * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)m * nn; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % m), c = (int)(e / m);
    const size_t off = (size_t)(rc + r) + (size_t)n * (cc + c);
    T v = part[off];
    for (int k = 1; k < ksplit; ++k) v = add(v, part[(size_t)k * nn2 + off]);
    dst[off] = v;
  }
  lu_trace(1, 256 + tstep, 1);
}

// y = op(Inv) x for the packed triangular inverse: LOWER -> unit-lower inv(L), else inv(U).
// Two launches: k_tri_mv partial products over (64-row tile) x (128-column slice) CTAs, then
// k_tri_mv_sum adds the slices (fixed order: deterministic).  Part: [nslices][n].
constexpr int kTmvRows = 64, kTmvCols = 128;
template <class T, bool LOWER>
__global__ void __launch_bounds__(256) k_tri_mv(const T* __restrict__ Inv, int n, const T* __restrict__ x,
                                                T* __restrict__ part, const LmDeviceState* st, int gate_running) {
  pdl_wait();
  if (lu_gated(st, gate_running)) return;
  __shared__ T red[4][kTmvRows];
  const int r0 = blockIdx.x * kTmvRows, c0 = blockIdx.y * kTmvCols;
  const int tid = threadIdx.x, rl = tid % kTmvRows, g = tid / kTmvRows;
  const int row = r0 + rl;
  T acc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u] = zero_of<T>();
  const bool tile_live = LOWER ? (c0 < r0 + kTmvRows) : (c0 + kTmvCols > r0);
  if (tile_live && row < n) {
    const int cb = c0 + g * (kTmvCols / 4);
#pragma unroll
    for (int c4 = 0; c4 < kTmvCols / 4; c4 += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = cb + c4 + u;
        const bool in = c < n && (LOWER ? c < row : c >= row);
        if (in) fma_acc(acc[u], Inv[(int64_t)row + (int64_t)n * c], x[c]);
      }
    }
  }
  T v = acc[0];
#pragma unroll
  for (int u = 1; u < 8; ++u) v = add(v, acc[u]);
  red[g][rl] = v;
  __syncthreads();
  if (g == 0 && row < n) part[(int64_t)blockIdx.y * n + row] = add(add(red[0][rl], red[1][rl]), add(red[2][rl], red[3][rl]));
}

template <class T, bool LOWER>
__global__ void k_tri_mv_sum(const T* __restrict__ part, int nslices, int n, const T* __restrict__ x, T* __restrict__ y,
                             const LmDeviceState* st, int gate_running) {
  pdl_wait();
  if (lu_gated(st, gate_running)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  T v = LOWER ? x[i] : zero_of<T>();
  for (int q = 0; q < nslices; ++q) v = add(v, part[(int64_t)q * n + i]);
  y[i] = v;
}

// ---- Block-inverse substitution (n_B too large for the full explicit inverse, config 1's 4800)
// Only the DB x DB diagonal blocks of L and U are inverted (recursive doubling capped at DB / 2), so
// a triangular solve is ceil(n / DB) block steps of chip-wide mat-vecs instead of a chain of n / 32
// flag hand-offs between 32-row substitution blocks:
//   L:  x_b = inv(L_bb) (x_b - L[b, 0:b) x[0:b))        b ascending
//   U:  x_b = inv(U_bb) (x_b - U[b, b+1:) x[b+1:))      b descending
// k_blk_mv writes per-(64-row tile, 128-column slice) partial products, k_blk_sum adds the slices
// in fixed order (deterministic).  MODE 0: full block of the LU factors; 1: unit-lower inverse
// diagonal block (columns < row); 2: upper inverse diagonal block (columns >= row).
template <class T, int MODE>
__global__ void __launch_bounds__(256) k_blk_mv(const T* __restrict__ Mx, int n, int r0, int r1, int c0, int c1,
                                                const T* __restrict__ x, T* __restrict__ part,
                                                const LmDeviceState* st, int gate_running) {
  pdl_wait();
  if (lu_gated(st, gate_running)) return;
  __shared__ T red[4][kTmvRows];
  const int rt = r0 + blockIdx.x * kTmvRows, cs = c0 + blockIdx.y * kTmvCols;
  const int tid = threadIdx.x, rl = tid % kTmvRows, g = tid / kTmvRows;
  const int row = rt + rl;
  T acc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u] = zero_of<T>();
  const bool tile_live = MODE == 0 ? true : MODE == 1 ? (cs < rt + kTmvRows) : (cs + kTmvCols > rt);
  if (tile_live && row < r1) {
    const int cb = cs + g * (kTmvCols / 4);
#pragma unroll
    for (int c4 = 0; c4 < kTmvCols / 4; c4 += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = cb + c4 + u;
        const bool in = c < c1 && (MODE == 0 ? true : MODE == 1 ? c < row : c >= row);
        if (in) fma_acc(acc[u], Mx[(int64_t)row + (int64_t)n * c], x[c]);
      }
    }
  }
  T v = acc[0];
#pragma unroll
  for (int u = 1; u < 8; ++u) v = add(v, acc[u]);
  red[g][rl] = v;
  __syncthreads();
  if (g == 0 && row < r1) part[(int64_t)blockIdx.y * n + row] = add(add(red[0][rl], red[1][rl]), add(red[2][rl], red[3][rl]));
}

// MODE 0: x[row] -= sum of slices (right-hand side minus the off-diagonal product); 1: x[row] +=
// sum (unit-lower inverse block: the implicit diagonal); 2: x[row] = sum (upper inverse block)
template <class T, int MODE>
__global__ void k_blk_sum(const T* __restrict__ part, int nslices, int n, int r0, int r1, T* __restrict__ x,
                          const LmDeviceState* st, int gate_running) {
  pdl_wait();
  if (lu_gated(st, gate_running)) return;
  const int i = r0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r1) return;
  T v = zero_of<T>();
  for (int q = 0; q < nslices; ++q) v = add(v, part[(int64_t)q * n + i]);
  x[i] = MODE == 0 ? sub(x[i], v) : MODE == 1 ? add(x[i], v) : v;
}

}  // namespace cpf
