// Are the fp64 DFMA pipe and the DMMA (fp64 tensor) pipe independent on B200?
// mode 0: DMMA only; mode 1: DFMA only; mode 2: both interleaved in the same warps.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
  double x[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    if (MODE != 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int iters = 20000, blocks = sms * 8, thr = 256;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, thr>>>(d, iters);
      if (mode == 1) k<1><<<blocks, thr>>>(d, iters);
      if (mode == 2) k<2><<<blocks, thr>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double warps = (double)blocks * thr / 32;
      double fl_mma = (mode != 1) ? 8.0 * 512 * iters * warps : 0;        // 8 DMMA x 8x8x4x2 flops
      double fl_fma = (mode != 0) ? 16.0 * 2 * 32 * iters * warps : 0;     // 16 DFMA per thread
      if (rep) printf("mode %d: %.2f TF/s total (dmma %.2f, dfma %.2f)\n", mode, (fl_mma + fl_fma) / ms / 1e9,
                      fl_mma / ms / 1e9, fl_fma / ms / 1e9);
    }
  }
  return 0;
}
