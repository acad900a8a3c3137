// Micro-benchmarks that pin the fp64 roofline denominators on B200
// (MEASURED_PEAKS.json only carries HBM copy and bf16 GEMM numbers):
//   * DFMA throughput (CUDA-core fp64)
//   * DMMA m8n8k4 throughput (legacy fp64 tensor-core path; tcgen05 has no f64 kind)
//   * streaming HBM read bandwidth with 128-bit loads (read-only, like the MTTKRP pass)
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void read_kernel(const double2* __restrict__ p, size_t n2, double* out) {
  double s = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 v0 = __ldcs(p + i), v1 = __ldcs(p + i + stride), v2 = __ldcs(p + i + 2 * stride), v3 = __ldcs(p + i + 3 * stride);
    s += v0.x + v0.y + v1.x + v1.y + v2.x + v2.y + v3.x + v3.y;
  }
  for (; i < n2; i += stride) { double2 v = p[i]; s += v.x + v.y; }
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d", prop.name, sms);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // DFMA: blocks=sms*8, 256 threads, 16 chains per thread
  {
    int iters = 20000, blocks = sms * 8, threads = 256;
    dfma_kernel<<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * (double)iters * blocks * threads;
    printf(", \"dfma_tflops\": %.2f", flops / (ms * 1e-3) / 1e12);
  }
  {
    int iters = 20000, blocks = sms * 8, threads = 256;
    dmma_kernel<<<blocks, threads>>>(out, 100);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
    printf(", \"dmma_tflops\": %.2f", flops / (ms * 1e-3) / 1e12);
  }
  {
    size_t bytes = (size_t)8 << 30;  // 8 GiB
    double2* p; CK(cudaMalloc(&p, bytes));
    CK(cudaMemset(p, 0, bytes));
    size_t n2 = bytes / 16;
    float best = 1e9;
    for (int blocksPerSm = 2; blocksPerSm <= 8; blocksPerSm *= 2) {
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        read_kernel<<<sms * blocksPerSm, 512>>>(p, n2, out);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
      }
    }
    printf(", \"hbm_read_gbs\": %.1f", bytes / (best * 1e-3) / 1e9);
    cudaFree(p);
  }
  printf("}\n");
  return 0;
}
