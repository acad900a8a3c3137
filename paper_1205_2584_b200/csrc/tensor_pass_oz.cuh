// Tensor passes on the int8 tensor cores: fp64 contractions by exact digit splitting (Ozaki
// scheme) with tcgen05.mma kind::i8, TMEM accumulators and TMA.
//
// Why: the fp64 passes (tensor_pass_dmma.cuh) are bound by the DMMA pipe (83-85 % issue, ~3.3 ms
// per 16 GB pass at config 4), while HBM would allow ~2.45 ms.  sm_100a has no fp64 tcgen05 kind,
// but its int8 tensor cores run at ~4.5 POPS: splitting both operands into 7-bit digit planes turns
// one fp64 GEMM into 36 exact int8 GEMMs, which together use ~40 % of the int8 pipe -- the pass
// becomes HBM-bound.
//
// Representation.  Y (fixed for the whole fit) is split ONCE per pass into a tile-image copy: per
// output row (pass A: row (i1, m), contracted c; pass B: row (i1, c), contracted m) with e the
// binary exponent of the row's max |y| and F = 56 - e, X = trunc(|y| 2^F) < 2^56 is written as 8
// base-128 digits d_1..d_8 (most significant first), stored as signed int8 planes sign(y) d_i
// (X = rint(|y| 2^F): round to nearest, so the representation error is unbiased).
// The per-iteration operand B (A_N slab for pass A, the Khatri-Rao rows for pass B; K x R) is split
// the same way per column r (F_r).  Then
//     sum_k y_k b_kr = 2^-(F_row+F_r) sum_{i,j} 128^(16-i-j) S_ij,   S_ij = sum_k yd_i(k) bd_j(k)
// and every S_ij is an exact int32 (|S_ij| <= 8 K 127^2 per accumulator).  Pairs with i + j >= 11
// contribute below ~2^-58 of a product of row/column maxima and are dropped (43 of 64 pairs kept);
// pairs with equal d = i + j share an accumulator.  What remains is rounding each operand at 2^-57
// of its row's (column's) max: per product, below fp64's own rounding unless the element is far
// below its row max (measured: tools/microbench/oz_pass_test; profiles/r01_oz_pass.txt).
//
// Layout.  Each copy is stored as the exact shared-memory images the MMAs read: per (tile, K block)
// 8 planes x 32 K-rows x 128 i1-bytes, 128B-swizzled (16-byte chunk j of K-row k at chunk j ^ (k%8)),
// tiles' K blocks consecutive -- one 32 KB contiguous bulk copy per pipeline stage and a 2 MB
// contiguous stream per tile, so HBM sees long sequential reads in both passes.  The two copies
// (2 x 16.5 GB at config 4) are the price of that; HBM has room for them.
//
// The 43 products per K step are 8 MMAs: Y plane i (M = 128 rows x K = 32, MN-major, 128B swizzle)
// times B planes 1..min(8, 10-i) stacked along N (N = 32 min(8, 10-i), K-major, no swizzle),
// accumulating from TMEM column 32 (i - 1) -- so pair (i, j) lands in column block d - 2 = i + j - 2
// of one 9 x 32-column accumulator.  One accumulator: the epilogue copies it to registers
// (~1 us) and releases it; the 5-stage copy ring keeps HBM busy meanwhile.
//
// Passes (rows of the output tile are i1; the K dimension is the contracted mode):
//   MODE 0 (pass A): tile (i1 block, m), K = c:  P[r][m][i1] = sum_c Y[i1, m, c] B[c, r]
//   MODE 1 (pass B): tile (i1 block, c), K = m:  U[r][c][i1] = sum_m Y[i1, m, c] B[m, r]
// The epilogue reduces each tile straight into the partial sums the fp64 passes produce (M_1 rows,
// Z, M_N rows); nothing tensor-sized is written.
// Warp roles: warp 0 lane 0 = bulk-copy producer, warp 1 = TMEM allocator + MMA issuer (lane 0),
// warps 2-5 = epilogue (TMEM lane quarter = warp % 4).  Persistent grid, static tile schedule.
#pragma once
#include "cpf_common.cuh"
#include "small_ops.cuh"

namespace cpf {

constexpr int kOzPlanes = 8;
constexpr int kOzDmax = 10;                            // pairs (i, j) with i + j <= 10 are kept (43)
constexpr int kOzBlocks = kOzDmax - 1;                 // accumulator blocks d = 2..10
constexpr int kOzM = 128;                              // tile rows (i1)
constexpr int kOzK = 32;                               // K per stage (one MMA K step)
constexpr int kOzN = 32;                               // R padded
constexpr int kOzStages = 5;
constexpr int kOzAPlane = kOzM * kOzK;                 // 4 KB
constexpr int kOzABytes = kOzPlanes * kOzAPlane;       // 32 KB
constexpr int kOzBPlane = kOzN * kOzK;                 // 1 KB
constexpr int kOzBBytes = kOzPlanes * kOzBPlane;       // 8 KB
constexpr int kOzStageBytes = kOzABytes + kOzBBytes;   // 40 KB (multiple of 1024)
constexpr int kOzThreads = 192;
constexpr size_t kOzSmem = 1024 + (size_t)kOzStages * kOzStageBytes + 128 + 2 * 128 * sizeof(double);

struct OzGeom {
  int64_t I1, Lmid, C;  // tensor view (C = local slab extent)
  int nb;               // i1 tiles of 128 rows
  int nkb;              // K blocks of 32 (MODE 0: over c, MODE 1: over m)
  int64_t nouter;       // MODE 0: Lmid, MODE 1: C
  int64_t ntiles;       // nb * nouter; tile t = outer * nb + i1 block
  int R;
  int dbg;              // experiments: bit 0 = no output stores, bit 1 = no MMAs, bit 2 = no L2 hint
};

__device__ __forceinline__ int oz_scale_exp(double amax) {
  if (!(amax > 0.0)) return 0;
  int e;
  frexp(amax, &e);  // amax = f 2^e, f in [0.5, 1): amax < 2^e
  return 56 - e;
}

// digits of X = rint(|v| 2^F), most significant first, signed like v.  X < 2^56 always: an element
// within 8x of its row max has |v| 2^F an exact integer (< 2^56), smaller ones stay < 2^55.
__device__ __forceinline__ void oz_digits(double v, int F, int8_t (&d)[kOzPlanes]) {
  const unsigned long long X = __double2ull_rn(ldexp(fabs(v), F));
  const bool neg = v < 0.0;
#pragma unroll
  for (int i = 0; i < kOzPlanes; ++i) {
    const int dd = (int)((X >> (7 * (kOzPlanes - 1 - i))) & 127ull);
    d[i] = (int8_t)(neg ? -dd : dd);
  }
}

template <int MODE>
__device__ __forceinline__ int64_t oz_yidx(const OzGeom& g, int64_t i1, int64_t o, int64_t k) {
  return MODE == 0 ? i1 + g.I1 * (o + g.Lmid * k) : i1 + g.I1 * (k + g.Lmid * o);
}

// ---- accuracy envelope ------------------------------------------------------------------------
// The split represents every element of a row (column) in fixed point against the row's max: an
// element within 16x of the max is exact, a smaller one carries an absolute error <= 2^-57 * 2^e
// (2^(e-1) <= max < 2^e).  The rigorous error of one K-term contraction is therefore
//     E_oz <= 2^-56 (ymax ||b||_1 + bmax ||y||_1) + (dropped digit pairs, ~2^-58 K ymax bmax).
// The guard keeps the int8 path only while every row of Y and every column of the operand has a
// peak-to-rms ratio <= 16 (max^2 K <= 256 sum x^2): then E_oz <= 2^-51 K rms_y rms_b, i.e. a few
// units of fp64 rounding on the K-term dot product's natural scale -- the scale of fp64's own
// accumulation error for such data.  Spikier data (a few entries carrying the row) is outside that
// envelope and the pass runs in fp64 (DMMA): Y is checked once when the tensor is bound (the plan
// drops the int8 images), the operand on every launch (k_oz_split_b sets DevFlags::oz_bad, which
// gates the int8 kernels off and the fp64 fallback on for that launch).
constexpr double kOzPeakRms2 = 256.0;

__device__ __forceinline__ bool oz_outside(double amax, double sumsq, int64_t K) {
  return amax * amax * (double)K > kOzPeakRms2 * sumsq;
}

// ---- one-time split of Y into a pass's tile images ------------------------------------------
// row exponents: thread per tile row (t, row); F = 0 for padding rows.  *ybad counts the rows
// outside the accuracy envelope (cleared by the host before the launch).
template <int MODE>
__global__ void k_oz_rowexp(const double* __restrict__ Y, OzGeom g, int* __restrict__ Frow, int* __restrict__ ybad,
                            int64_t t0 = 0, int64_t t1 = -1) {
  pdl_wait();
  const int64_t K = MODE == 0 ? g.C : g.Lmid;
  if (t1 < 0) t1 = g.ntiles;  // tiles [t0, t1): the whole image, or the part of it already uploaded
  for (int64_t idx = t0 * kOzM + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < t1 * kOzM;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = idx / kOzM;
    const int row = (int)(idx - t * kOzM);
    const int64_t o = t / g.nb;
    const int64_t i1 = (int64_t)kOzM * (t - o * g.nb) + row;
    double m = 0.0, ss = 0.0;
    if (i1 < g.I1)
      for (int64_t k = 0; k < K; ++k) {
        const double v = Y[oz_yidx<MODE>(g, i1, o, k)];
        m = fmax(m, fabs(v));
        ss = fma(v, v, ss);
      }
    Frow[idx] = oz_scale_exp(m);
    if (oz_outside(m, ss, K)) atomicAdd(ybad, 1);
  }
}

// digit planes: work item = (tile, K block, K row k, quad of 4 i1) -> 8 x 4 bytes of the image
template <int MODE>
__global__ void k_oz_split_y(const double* __restrict__ Y, OzGeom g, const int* __restrict__ Frow,
                             uint8_t* __restrict__ Yimg, int64_t t0 = 0, int64_t t1 = -1) {
  pdl_wait();
  const int64_t K = MODE == 0 ? g.C : g.Lmid;
  if (t1 < 0) t1 = g.ntiles;
  const int64_t per = g.nkb * (kOzK * kOzM / 4);  // work items per tile
  const int64_t total = t1 * per;
  for (int64_t idx = t0 * per + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int quad = (int)(idx & 31);
    const int k = (int)((idx >> 5) & 31);
    const int64_t tk = idx >> 10;  // t * nkb + kb
    const int64_t t = tk / g.nkb;
    const int64_t kb = tk - t * g.nkb;
    const int64_t o = t / g.nb;
    const int64_t b = t - o * g.nb;
    const int64_t kk = kb * kOzK + k;
    uint32_t w[kOzPlanes];
#pragma unroll
    for (int p = 0; p < kOzPlanes; ++p) w[p] = 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int row = 4 * quad + u;
      const int64_t i1 = (int64_t)kOzM * b + row;
      if (i1 >= g.I1 || kk >= K) continue;
      int8_t d[kOzPlanes];
      oz_digits(Y[oz_yidx<MODE>(g, i1, o, kk)], Frow[t * kOzM + row], d);
#pragma unroll
      for (int p = 0; p < kOzPlanes; ++p) w[p] |= (uint32_t)(uint8_t)d[p] << (8 * u);
    }
    const int byte = 4 * quad;
    uint8_t* dst = Yimg + tk * (int64_t)kOzABytes + k * 128 + (((byte >> 4) ^ (k & 7)) << 4) + (byte & 15);
#pragma unroll
    for (int p = 0; p < kOzPlanes; ++p) *reinterpret_cast<uint32_t*>(dst + p * kOzAPlane) = w[p];
  }
}

// ---- per-iteration split of the K x R operand (row-major, stride ld) -----------------------
// Bq layout per K block kb (8 KB, one bulk copy per stage): plane j (1 KB) = 4 groups of 8 rows
// (r) x 2 K chunks of 16 bytes: byte (r, k) at kb*8192 + j*1024 + (r/8)*256 + (k%32/16)*128 + (r%8)*16 + k%16
// (the canonical K-major no-swizzle UMMA layout: LBO = 128 B between K chunks, SBO = 256 B between
// 8-row groups).  Columns r >= R and rows k >= K stay zero (buffer cleared at allocation).
// The block of column r also writes bad[r] (the accuracy guard: 1 = outside the envelope).
__global__ void k_oz_split_b(const double* __restrict__ src, int64_t K, int R, int ld, uint8_t* __restrict__ Bq,
                             int* __restrict__ Fr, int* __restrict__ bad, const LmDeviceState* st, const DevFlags* fl,
                             int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  const int r = blockIdx.x;
  __shared__ double red[32], red2[32];
  double m = 0.0, ss = 0.0;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    const double v = src[k * ld + r];
    m = fmax(m, fabs(v));
    ss = fma(v, v, ss);
  }
  for (int o = 16; o > 0; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = m;
    red2[threadIdx.x >> 5] = ss;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    double w = threadIdx.x < (blockDim.x >> 5) ? red2[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
      w += __shfl_xor_sync(0xffffffffu, w, o);
    }
    if (threadIdx.x == 0) {
      red[0] = v;
      red2[0] = w;
    }
  }
  __syncthreads();
  const int F = oz_scale_exp(red[0]);
  if (threadIdx.x == 0) {
    Fr[r] = F;
    if (bad && r < kOzGuardCols) bad[r] = oz_outside(red[0], red2[0], K) ? 1 : 0;
  }
  const int64_t rofs = (int64_t)(r >> 3) * 256 + (r & 7) * 16;
  for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
    int8_t d[kOzPlanes];
    oz_digits(src[k * ld + r], F, d);
    const int64_t kb = k >> 5, kk = k & 31;
    uint8_t* dst = Bq + kb * kOzBBytes + rofs + (kk >> 4) * 128 + (kk & 15);
#pragma unroll
    for (int p = 0; p < kOzPlanes; ++p) dst[p * kOzBPlane] = (uint8_t)d[p];
  }
}

// counts the launches whose operand fell outside the envelope (gated kGateIfOzBad)
__global__ void k_oz_note_fallback(DevFlags* fl, const LmDeviceState* st, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  atomicAdd(&fl->oz_fallbacks, 1);
}

// ---- tcgen05 / TMA primitives ---------------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// MN-major, 128B-swizzled operand (K-rows of 128 bytes along M, 8-row / 1024 B atoms along K)
__device__ __forceinline__ uint64_t oz_desc_a(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(kOzAPlane >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
// K-major, no swizzle: 8 x 16 B core matrices, LBO (K) = 128 B, SBO (N) = 256 B
__device__ __forceinline__ uint64_t oz_desc_b(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}
// kind::i8: D s32, A s8 MN-major, B s8 K-major, M = 128
__host__ __device__ constexpr uint32_t oz_idesc(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kOzM >> 4) << 24);
}
__device__ __forceinline__ void oz_mma(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, int accum) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void oz_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// streaming bulk copy with an L2 evict-first policy: the 16 GB image stream should not push the
// concurrently running LU's matrix (11.5 MB) and the B operands out of L2
__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void oz_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- the pass ------------------------------------------------------------------------------
// Schedule: CTA = (i1 block b, chunk of outer indices); grid = nb * nchunks.  A fixed b per CTA
// lets pass A keep its rows' M_1 partials in registers across all of its tiles.
// Epilogue per tile (thread = tile row i1, value p[r] = (Y x_K B)[i1, o, r]):
//   MODE 0: m1[r] += p[r] KM[o, r] (registers; written once: m1part[chunk][i1][r])
//           zpart[b][o][r] = sum over the tile's rows of p[r] A1[i1, r]
//   MODE 1: bpart[o][b][r] = sum over the tile's rows of p[r] A1[i1, r]
// (the formats of k_m1_reduce / k_z_reduce / k_pass_b_reduce; all sums in fixed order).
struct OzOut {
  const double* A1c;  // I1 x RP row-major
  const double* KMc;  // Lmid x RP row-major (MODE 0)
  int RP;
  int nchunks;
  int64_t ochunk;     // outer indices per chunk
  double* m1part;     // MODE 0: [nchunks][I1][RP]
  double* red;        // MODE 0: zpart [nb][Lmid][RP]; MODE 1: bpart [C][nb][RP]
};

// lane l ends with the warp sum of v[l] (31 shuffles: recursive halving with exchange)
__device__ __forceinline__ double oz_warp_transpose_sum(double (&v)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const double send = up ? v[i] : v[i + s];
      const double keep = up ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

template <int MODE>
__global__ void __launch_bounds__(kOzThreads, 1)
    k_oz_pass(const uint8_t* __restrict__ Yimg, const int* __restrict__ Frow, const uint8_t* __restrict__ Bq,
              const int* __restrict__ Fr, OzGeom g, OzOut out, const LmDeviceState* st, const DevFlags* fl, int gate) {
  pdl_wait();
  if (!gate_open(st, fl, gate)) return;
  extern __shared__ unsigned char oz_smem_raw[];
  unsigned char* base =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(oz_smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + (size_t)kOzStages * kOzStageBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kOzStages;
  uint64_t* tfull = bars + 2 * kOzStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  double* red = reinterpret_cast<double*>(base + (size_t)kOzStages * kOzStageBytes + 128);  // [2][4][32]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = (int)(blockIdx.x % g.nb);
  const int chunk = (int)(blockIdx.x / g.nb);
  const int64_t obeg = (int64_t)chunk * out.ochunk;
  const int64_t oend = min(g.nouter, obeg + out.ochunk);

  if (tid == 0) {
    for (int s = 0; s < kOzStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tempty[0], 128);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {  // ---- bulk-copy producer
      int s = 0;
      uint32_t ph = 0;
      const uint64_t pol = policy_evict_first();
      for (int64_t o = obeg; o < oend; ++o) {
        const int64_t t = o * g.nb + b;
        for (int kb = 0; kb < g.nkb; ++kb) {
          mbar_wait(&empty[s], ph ^ 1u);
          unsigned char* sa = base + (size_t)s * kOzStageBytes;
          mbar_expect_tx(&full[s], kOzStageBytes);
          if (g.dbg & 4) bulk_g2s(sa, Yimg + (size_t)(t * g.nkb + kb) * kOzABytes, kOzABytes, &full[s]);
          else bulk_g2s_stream(sa, Yimg + (size_t)(t * g.nkb + kb) * kOzABytes, kOzABytes, &full[s], pol);
          bulk_g2s(sa + kOzABytes, Bq + (size_t)kb * kOzBBytes, kOzBBytes, &full[s]);
          if (++s == kOzStages) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int64_t o = obeg; o < oend; ++o, ++it) {
        mbar_wait(&tempty[0], (uint32_t)((it & 1) ^ 1));
        tc_fence_after();
        const uint32_t dcol = tmem;
        for (int kb = 0; kb < g.nkb; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(base + (size_t)s * kOzStageBytes);
          const uint64_t bdesc = oz_desc_b(sa + kOzABytes);
          // Plane i accumulates into columns 32 i .. 32 (i + nb_i) - 1.  Plane 0 (accumulate off at
          // kb = 0) initialises columns 0..255; the d = 10 block (columns 256..287) is first
          // written by plane 1, so at kb = 0 plane 1's last 32 columns are a separate MMA with
          // accumulate off (else it would add stale TMEM contents of the previous tile).
          if (!(g.dbg & 2))
#pragma unroll
            for (int i = 0; i < kOzPlanes; ++i) {
              const int nbp = kOzDmax - 1 - i < kOzPlanes ? kOzDmax - 1 - i : kOzPlanes;  // B planes used
              if (i == 1 && kb == 0 && 32 * (i + nbp) > 256) {
                oz_mma(dcol + 32u, oz_desc_a(sa + kOzAPlane), bdesc, oz_idesc(kOzN * (nbp - 1)), 1);
                oz_mma(dcol + 256u, oz_desc_a(sa + kOzAPlane), oz_desc_b(sa + kOzABytes + (nbp - 1) * kOzBPlane),
                       oz_idesc(kOzN), 0);
              } else {
                oz_mma(dcol + 32u * i, oz_desc_a(sa + i * kOzAPlane), bdesc, oz_idesc(kOzN * nbp),
                       (kb > 0 || i > 0) ? 1 : 0);
              }
            }
          oz_commit(&empty[s]);
          if (++s == kOzStages) { s = 0; ph ^= 1u; }
        }
        oz_commit(&tfull[0]);
      }
    }
  } else {  // ---- epilogue: warps 2..5, TMEM lane quarter warp % 4
    const int q = warp & 3;
    const int row = 32 * q + lane;
    const int64_t i1 = (int64_t)kOzM * b + row;
    const bool rv = i1 < g.I1;
    const double* a1row = out.A1c + (rv ? i1 : 0) * out.RP;
    double m1[kOzN];
#pragma unroll
    for (int r = 0; r < kOzN; ++r) m1[r] = 0.0;
    int it = 0;
    for (int64_t o = obeg; o < oend; ++o, ++it) {
      const int64_t t = o * g.nb + b;
      mbar_wait(&tfull[0], (uint32_t)(it & 1));
      tc_fence_after();
      double p[kOzN];
#pragma unroll
      for (int r = 0; r < kOzN; ++r) p[r] = 0.0;
#pragma unroll 1
      for (int d = kOzDmax; d >= 2; --d) {  // smallest weight first
        uint32_t v[32];
        oz_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(32 * (d - 2)), v);
        const double sc = ldexp(1.0, 7 * (2 * kOzPlanes - d));
#pragma unroll
        for (int r = 0; r < kOzN; ++r) p[r] = fma((double)(int)v[r], sc, p[r]);
      }
      tc_fence_before();
      mbar_arrive(&tempty[0]);  // accumulator free: the next tile's MMAs start
      const int fy = __ldg(Frow + t * kOzM + row);
#pragma unroll
      for (int r = 0; r < kOzN; ++r) {
        const bool cv = r < g.R;
        const double pr = cv ? ldexp(p[r], -(fy + __ldg(Fr + r))) : 0.0;  // exact power-of-two scaling
        if (MODE == 0 && cv) m1[r] = fma(pr, __ldg(out.KMc + o * out.RP + r), m1[r]);
        p[r] = (cv && rv) ? pr * __ldg(a1row + r) : 0.0;
      }
      // tile sum over the 128 rows: warp transpose-sum, then the 4 warps in fixed order
      const double ws = oz_warp_transpose_sum(p, lane);
      double* rb = red + (it & 1) * 128;
      rb[q * 32 + lane] = ws;
      named_sync(1, 128);
      if (q == 0 && lane < g.R) {
        const double tot = ((rb[lane] + rb[32 + lane]) + rb[64 + lane]) + rb[96 + lane];
        if (MODE == 0) out.red[((int64_t)b * g.Lmid + o) * out.RP + lane] = tot;
        else out.red[(o * g.nb + b) * out.RP + lane] = tot;
      }
    }
    if (MODE == 0 && rv) {
      double* mp = out.m1part + ((int64_t)chunk * g.I1 + i1) * out.RP;
#pragma unroll
      for (int r = 0; r < kOzN; ++r)
        if (r < g.R) mp[r] = m1[r];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

}  // namespace cpf
