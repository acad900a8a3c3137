// Throughput of the fp64 mma.sync shapes on B200 (sm_100a): m8n8k4 (the only shape before
// sm_90) vs m16n8k4 / m16n8k8 / m16n8k16 (sm_90+).  Each warp issues 8 independent
// accumulator chains; the numeric check at the end compares one m16n8k16 product against
// DFMA on known fragments (fragment layout probe).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_shapes.cu -o dmma_shapes
#include <cstdio>
#include <cuda_runtime.h>

template <int SHAPE>
__global__ void k_mma(double* out, int iters) {
  const double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (SHAPE == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
      } else if (SHAPE == 1) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a), "d"(b), "d"(b));
      } else if (SHAPE == 2) {
        asm volatile(
            "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
            : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
            : "d"(a), "d"(b), "d"(a), "d"(b), "d"(b), "d"(a));
      } else {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
            "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
            : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
            : "d"(a), "d"(b), "d"(a), "d"(b), "d"(a), "d"(b), "d"(a), "d"(b), "d"(b), "d"(a), "d"(b), "d"(a));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

// layout probe: A 16x16 (row-major A[r][k] = r*16 + k + 1), B 16x8 (B[k][n] = (k+1)*(n+2) / 7)
// fragments per the PTX ISA m16n8k16 f64 layout: a_i = A[g + 8*(i%2)][t + 4*(i/2)],
// b_i = B[t + 4*i][g], c: c0,c1 = D[g][2t + {0,1}], c2,c3 = D[g+8][2t + {0,1}]
__global__ void k_probe(double* err) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[8], b[4], c[4] = {0, 0, 0, 0};
  for (int i = 0; i < 8; ++i) a[i] = (g + 8 * (i % 2)) * 16 + (t + 4 * (i / 2)) + 1;
  for (int i = 0; i < 4; ++i) b[i] = (t + 4 * i + 1) * (g + 2) / 7.0;
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]),
        "d"(b[2]), "d"(b[3]));
  double e = 0;
  for (int q = 0; q < 4; ++q) {
    const int r = g + 8 * (q / 2), n = 2 * t + (q % 2);
    double ref = 0;
    for (int k = 0; k < 16; ++k) ref += (r * 16 + k + 1) * ((k + 1) * (n + 2) / 7.0);
    e = fmax(e, fabs(ref - c[q]));
  }
  atomicMax((unsigned long long*)err, __double_as_longlong(e));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaMemset(out, 0, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  const char* names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  const double fma_per[4] = {256, 512, 1024, 2048};
  for (int shape = 0; shape < 4; ++shape)
    for (int wpb : {4, 8, 16}) {
      auto run = [&](int it) {
        switch (shape) {
          case 0: k_mma<0><<<sms, 32 * wpb>>>(out, it); break;
          case 1: k_mma<1><<<sms, 32 * wpb>>>(out, it); break;
          case 2: k_mma<2><<<sms, 32 * wpb>>>(out, it); break;
          default: k_mma<3><<<sms, 32 * wpb>>>(out, it); break;
        }
      };
      run(10);
      cudaEventRecord(e0);
      run(iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 2.0 * fma_per[shape] * 8 * iters * (double)sms * wpb;
      printf("%-9s warps/SM %2d: %.2f TFLOP/s\n", names[shape], wpb, flops / (ms * 1e-3) / 1e12);
    }
  cudaMemset(out, 0, 8);
  k_probe<<<1, 32>>>(out);
  double err;
  cudaMemcpy(&err, out, 8, cudaMemcpyDeviceToHost);
  printf("m16n8k16 layout probe max abs err: %g (%s)\n", err, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
