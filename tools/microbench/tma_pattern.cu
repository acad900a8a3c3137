// Achievable HBM read bandwidth of the two DMMA-pass access patterns, with the same warp-specialised
// bulk-copy ring (one producer lane, NST stages, consumers only wait + release):
//   pattern 0 (pass A): CTA = (i1 tile, m group); per m, K = c: CK rows of 512 doubles, stride I1*Lmid
//   pattern 1 (pass B): CTA = (i1 tile, c);       K = m: CK rows of 512 doubles, stride I1 (contiguous)
//   pattern 2 (pass A, c-split): CTA = (i1 tile, c group); per c: K = m rows (contiguous)... same as 1
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1205_2584_b200/csrc tma_pattern.cu -o tma_pattern
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "cpf_common.cuh"


struct Geo {
  int64_t I1, L, C;
  int CK, NST, mode;
  int64_t per;  // m per CTA (mode 0) / m chunk (mode 1)
};

__global__ void __launch_bounds__(288, 1) k_pat(const double* Y, Geo g) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  double* stages = reinterpret_cast<double*>(smem_raw + 128);
  const size_t se = (size_t)g.CK * 516;
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t a0 = (int64_t)blockIdx.x * 512;
  const int64_t rows = min((int64_t)512, g.I1 - a0);
  const uint32_t yb = (uint32_t)(rows * 8);
  const int64_t Lrows = g.I1 * g.L;
  int64_t nq, nkc;
  int64_t mbeg = 0, mend = 0, cfix = 0;
  if (g.mode == 0) {
    mbeg = blockIdx.y * g.per; mend = min(g.L, mbeg + g.per);
    if (mbeg >= mend) return;
    nkc = (g.C + g.CK - 1) / g.CK;
    nq = (mend - mbeg) * nkc;
  } else {
    cfix = blockIdx.y;
    mbeg = blockIdx.z * g.per; mend = min(g.L, mbeg + g.per);
    if (mbeg >= mend) return;
    nkc = (mend - mbeg + g.CK - 1) / g.CK;
    nq = nkc;
  }
  if (tid == 0) {
    for (int s = 0; s < g.NST; ++s) { mbar_init(&bars[s], 1); mbar_init(&bars[g.NST + s], 8); }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid >= 256) {
    if (lane == 0)
      for (int64_t q = 0; q < nq; ++q) {
        const int s = (int)(q % g.NST);
        if (q >= g.NST) mbar_wait(&bars[g.NST + s], (uint32_t)(((q / g.NST) - 1) & 1));
        double* dst = stages + s * se;
        const int64_t rb = q / nkc, kc = q % nkc;
        if (g.mode == 0) {
          const int64_t k0 = kc * g.CK;
          const int ck = (int)min((int64_t)g.CK, g.C - k0);
          fence_proxy_async();
          mbar_expect_tx(&bars[s], yb * ck);
          const double* src = Y + a0 + g.I1 * (mbeg + rb) + Lrows * k0;
          for (int k = 0; k < ck; ++k) bulk_g2s(dst + k * 516, src + Lrows * k, yb, &bars[s]);
        } else {
          const int64_t k0 = mbeg + kc * g.CK;
          const int ck = (int)min((int64_t)g.CK, mend - k0);
          fence_proxy_async();
          mbar_expect_tx(&bars[s], yb * ck);
          const double* src = Y + Lrows * cfix + a0 + g.I1 * k0;
          for (int k = 0; k < ck; ++k) bulk_g2s(dst + k * 516, src + g.I1 * k, yb, &bars[s]);
        }
      }
    return;
  }
  int s = 0;
  uint32_t ph = 0;
  for (int64_t q = 0; q < nq; ++q) {
    mbar_wait(&bars[s], ph);
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars[g.NST + s]);
    if (++s == g.NST) { s = 0; ph ^= 1u; }
  }
}

int main(int argc, char** argv) {
  const int64_t I1 = 1000, L = 1000, C = 2000;
  double* Y;
  const size_t n = (size_t)I1 * L * C;
  if (cudaMalloc(&Y, n * 8) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(Y, 0, n * 8);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(k_pat, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  struct Case { int mode, CK, NST; int64_t groups; };
  Case cases[] = {{0, 16, 3, 72}, {0, 8, 6, 72}, {0, 4, 12, 72}, {0, 16, 3, 74}, {0, 8, 6, 148}, {1, 16, 3, 1}, {1, 8, 6, 1}, {1, 16, 3, 2}};
  for (auto cs : cases) {
    Geo g{I1, L, C, cs.CK, cs.NST, cs.mode, 0};
    dim3 grid;
    if (cs.mode == 0) {
      g.per = (L + cs.groups - 1) / cs.groups;
      grid = dim3(2, (unsigned)((L + g.per - 1) / g.per));
    } else {
      g.per = (L + cs.groups - 1) / cs.groups;
      grid = dim3(2, (unsigned)C, (unsigned)cs.groups);
    }
    const size_t smem = 128 + (size_t)cs.NST * cs.CK * 516 * 8;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      k_pat<<<grid, 288, smem>>>(Y, g);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 3)
        printf("mode %d CK %2d NST %2d grid (%u,%u,%u) smem %zu: %.3f ms  %.0f GB/s  err=%s\n", cs.mode, cs.CK, cs.NST,
               grid.x, grid.y, grid.z, smem, ms, n * 8 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
