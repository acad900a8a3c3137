// Latency probe (B200): dependent chains of DFMA, REDUX (__reduce_max_sync), SHFL, LDS, and an
// L2 pointer chase, one warp, clock64 around each chain.  nvcc -arch=sm_100a lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(double* out, long long* cyc, const int* chase, int nchase) {
  __shared__ int sm[1024];
  const int lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) sm[i] = (i * 7 + 1) & 1023;
  __syncwarp();
  double x = 1.0 + lane * 1e-9, y = 0.999999;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = fma(x, y, 1e-12);
  long long t1 = clock64();
  unsigned v = lane;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) v = __reduce_max_sync(0xffffffffu, v + (unsigned)lane) & 0xffff;
  long long t2 = clock64();
  double s = x;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) s = __shfl_sync(0xffffffffu, s, (lane + 1) & 31) + 1e-30;
  long long t3 = clock64();
  int idx = lane;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) idx = sm[idx];
  long long t4 = clock64();
  int p = lane;
#pragma unroll 1
  for (int i = 0; i < nchase; ++i) p = __ldcg(chase + p);
  long long t5 = clock64();
  double z = x;
  long long t6a = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { __syncthreads(); z += 1e-30; }
  long long t6 = clock64();
  if (lane == 0) {
    cyc[0] = (t1 - t0) / 1024; cyc[1] = (t2 - t1) / 1024; cyc[2] = (t3 - t2) / 1024; cyc[3] = (t4 - t3) / 1024;
    cyc[4] = (t5 - t4) / nchase; cyc[5] = (t6 - t6a) / 256;
  }
  out[lane] = x + s + v + idx + p + z;
}

int main() {
  const int n = 1 << 24;
  int* h = new int[n];
  for (int i = 0; i < n; ++i) h[i] = (int)(((long long)i * 2654435761LL + 12345) % n);
  int* d; double* o; long long* c;
  cudaMalloc(&d, n * sizeof(int)); cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 8 * 8);
  cudaMemcpy(d, h, n * sizeof(int), cudaMemcpyHostToDevice);
  probe<<<1, 32>>>(o, c, d, 4096);  // warm (L2 fill)
  probe<<<1, 32>>>(o, c, d, 4096);
  long long hc[8];
  cudaMemcpy(hc, c, 8 * 8, cudaMemcpyDeviceToHost);
  printf("latency cycles: DFMA %lld | REDUX.MAX %lld | SHFL(f64) %lld | LDS %lld | LDG.cg chase (64 MB, mostly DRAM/L2) %lld | BAR(1 warp) %lld\n",
         hc[0], hc[1], hc[2], hc[3], hc[4], hc[5]);
  return 0;
}
