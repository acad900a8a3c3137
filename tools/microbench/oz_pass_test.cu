// Standalone check + timing of the Ozaki int8 tcgen05 tensor passes (tensor_pass_oz.cuh).
//  1. small tensor: pass A / pass B outputs vs a long-double CPU contraction (error relative to
//     sum |y||b|, which bounds fp64 GEMM error by gamma_K);
//  2. config-4 size (1000 x 1000 x 2000): split once, then time both passes (CUDA events).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1205_2584_b200/csrc oz_pass_test.cu -o oz_pass_test
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "tensor_pass_oz.cuh"
using namespace cpf;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1); } } while (0)

static uint64_t rs = 88172645463325252ull;
static double urand() { rs ^= rs << 13; rs ^= rs >> 7; rs ^= rs << 17; return (rs >> 11) * (1.0 / 9007199254740992.0); }
static double nrand() { double u = urand() + 1e-300, v = urand(); return sqrt(-2 * log(u)) * cos(6.283185307179586 * v); }

__global__ void k_fill(double* Y, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = (uint64_t)i * 0x9E3779B97F4A7C15ull; h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
    Y[i] = ((double)(h >> 11) * (1.0 / 9007199254740992.0) - 0.5) * 3.0;
  }
}

struct Setup {
  int64_t I1, Lmid, C; int R, RP, nsm;
  double *Y, *BA, *BB, *A1, *KM, *m1p, *zp, *bp; uint8_t *YA, *YB, *BqA, *BqB; int *FrA, *FrB, *FrowA, *FrowB;
  OzGeom gA, gB;
};

static void setup(Setup& s, int64_t I1, int64_t Lmid, int64_t C, int R, const double* hY, int nsm) {
  s.I1 = I1; s.Lmid = Lmid; s.C = C; s.R = R; s.RP = 24; s.nsm = nsm;
  const int64_t J = I1 * Lmid * C;
  CK(cudaMalloc(&s.Y, J * 8));
  if (hY) CK(cudaMemcpy(s.Y, hY, J * 8, cudaMemcpyHostToDevice));
  else { k_fill<<<4096, 256>>>(s.Y, J); CK(cudaGetLastError()); }
  const int nb = (int)((I1 + kOzM - 1) / kOzM);
  const int nkA = (int)((C + 31) / 32), nkB = (int)((Lmid + 31) / 32);
  s.gA = OzGeom{I1, Lmid, C, nb, nkA, Lmid, (int64_t)nb * Lmid, R, 0};
  s.gB = OzGeom{I1, Lmid, C, nb, nkB, C, (int64_t)nb * C, R, 0};
  CK(cudaMalloc(&s.YA, (size_t)s.gA.ntiles * nkA * kOzABytes));
  CK(cudaMalloc(&s.YB, (size_t)s.gB.ntiles * nkB * kOzABytes));
  CK(cudaMalloc(&s.FrowA, (size_t)s.gA.ntiles * kOzM * 4));
  CK(cudaMalloc(&s.FrowB, (size_t)s.gB.ntiles * kOzM * 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_oz_rowexp<0><<<2048, 256>>>(s.Y, s.gA, s.FrowA);
  k_oz_split_y<0><<<8192, 256>>>(s.Y, s.gA, s.FrowA, s.YA);
  k_oz_rowexp<1><<<2048, 256>>>(s.Y, s.gB, s.FrowB);
  k_oz_split_y<1><<<8192, 256>>>(s.Y, s.gB, s.FrowB, s.YB);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("split (both copies): %.2f ms\n", ms);
  CK(cudaGetLastError());
  CK(cudaMalloc(&s.BqA, (size_t)nkA * kOzBBytes)); CK(cudaMemset(s.BqA, 0, (size_t)nkA * kOzBBytes));
  CK(cudaMalloc(&s.BqB, (size_t)nkB * kOzBBytes)); CK(cudaMemset(s.BqB, 0, (size_t)nkB * kOzBBytes));
  CK(cudaMalloc(&s.FrA, 128)); CK(cudaMalloc(&s.FrB, 128));
  CK(cudaMalloc(&s.BA, C * s.RP * 8)); CK(cudaMalloc(&s.BB, Lmid * s.RP * 8));
  CK(cudaMalloc(&s.A1, I1 * s.RP * 8)); CK(cudaMalloc(&s.KM, Lmid * s.RP * 8));
  CK(cudaMalloc(&s.m1p, (size_t)nsm * I1 * s.RP * 8)); CK(cudaMalloc(&s.zp, (size_t)nb * Lmid * s.RP * 8));
  CK(cudaMalloc(&s.bp, (size_t)C * nb * s.RP * 8));
  CK(cudaFuncSetAttribute(k_oz_pass<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOzSmem));
  CK(cudaFuncSetAttribute(k_oz_pass<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOzSmem));
}

static int run(Setup& s, int mode, int grid) {
  if (mode == 0) {
    const int nch = grid / s.gA.nb;
    OzOut oo{s.A1, s.KM, s.RP, nch, (s.Lmid + nch - 1) / nch, s.m1p, s.zp};
    k_oz_split_b<<<s.R, 256>>>(s.BA, s.C, s.R, s.RP, s.BqA, s.FrA, nullptr, nullptr, kAlways);
    k_oz_pass<0><<<s.gA.nb * nch, kOzThreads, kOzSmem>>>(s.YA, s.FrowA, s.BqA, s.FrA, s.gA, oo, nullptr, nullptr, kAlways);
    CK(cudaGetLastError());
    return nch;
  }
  const int nch = grid / s.gB.nb;
  OzOut oo{s.A1, nullptr, s.RP, nch, (s.C + nch - 1) / nch, nullptr, s.bp};
  k_oz_split_b<<<s.R, 256>>>(s.BB, s.Lmid, s.R, s.RP, s.BqB, s.FrB, nullptr, nullptr, kAlways);
  k_oz_pass<1><<<s.gB.nb * nch, kOzThreads, kOzSmem>>>(s.YB, s.FrowB, s.BqB, s.FrB, s.gB, oo, nullptr, nullptr, kAlways);
  CK(cudaGetLastError());
  return nch;
}

int main(int argc, char** argv) {
  int nsm = 148; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  // ---- 1. correctness: M1, Z (pass A) and M_N (pass B) vs long double, and plain fp64 for scale
  {
    const int64_t I1 = 300, Lmid = 40, C = 70; const int R = 20, RP = 24;
    const int64_t J = I1 * Lmid * C;
    std::vector<double> Y(J), BA(C * RP, 0.0), BB(Lmid * RP, 0.0), A1(I1 * RP, 0.0), KM(Lmid * RP, 0.0);
    const bool outl = argc > 2;
    for (auto& v : Y) v = nrand() * (outl && urand() < 0.01 ? 1e3 : 1.0);
    for (int64_t c = 0; c < C; ++c) for (int r = 0; r < R; ++r) BA[c * RP + r] = nrand() * pow(10.0, r % 4);
    for (int64_t m = 0; m < Lmid; ++m) for (int r = 0; r < R; ++r) BB[m * RP + r] = nrand() * pow(10.0, -(r % 3));
    for (int64_t i = 0; i < I1; ++i) for (int r = 0; r < R; ++r) A1[i * RP + r] = nrand();
    for (int64_t m = 0; m < Lmid; ++m) for (int r = 0; r < R; ++r) KM[m * RP + r] = nrand();
    Setup s; setup(s, I1, Lmid, C, R, Y.data(), nsm);
    CK(cudaMemcpy(s.BA, BA.data(), BA.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(s.BB, BB.data(), BB.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(s.A1, A1.data(), A1.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(s.KM, KM.data(), KM.size() * 8, cudaMemcpyHostToDevice));
    const int nchA = run(s, 0, nsm), nchB = run(s, 1, nsm);
    CK(cudaDeviceSynchronize());
    const int nb = s.gA.nb;
    std::vector<double> m1p((size_t)nchA * I1 * RP), zp((size_t)nb * Lmid * RP), bp((size_t)C * nb * RP);
    CK(cudaMemcpy(m1p.data(), s.m1p, m1p.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(zp.data(), s.zp, zp.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(bp.data(), s.bp, bp.size() * 8, cudaMemcpyDeviceToHost));
    // exact (long double) P and U, then the three outputs
    std::vector<long double> P((size_t)I1 * Lmid * R), Pa((size_t)I1 * Lmid * R), U((size_t)I1 * C * R), Ua((size_t)I1 * C * R);
    for (int r = 0; r < R; ++r)
      for (int64_t m = 0; m < Lmid; ++m)
        for (int64_t i = 0; i < I1; ++i) {
          long double acc = 0, ab = 0;
          for (int64_t c = 0; c < C; ++c) { long double t = (long double)Y[i + I1 * (m + Lmid * c)] * BA[c * RP + r]; acc += t; ab += fabsl(t); }
          P[(r * Lmid + m) * I1 + i] = acc; Pa[(r * Lmid + m) * I1 + i] = ab;
        }
    for (int r = 0; r < R; ++r)
      for (int64_t c = 0; c < C; ++c)
        for (int64_t i = 0; i < I1; ++i) {
          long double acc = 0, ab = 0;
          for (int64_t m = 0; m < Lmid; ++m) { long double t = (long double)Y[i + I1 * (m + Lmid * c)] * BB[m * RP + r]; acc += t; ab += fabsl(t); }
          U[(r * C + c) * I1 + i] = acc; Ua[(r * C + c) * I1 + i] = ab;
        }
    double eM1 = 0, eZ = 0, eMN = 0;
    for (int r = 0; r < R; ++r) {
      for (int64_t i = 0; i < I1; ++i) {
        long double ex = 0, ab = 0; double got = 0;
        for (int64_t m = 0; m < Lmid; ++m) { ex += P[(r * Lmid + m) * I1 + i] * KM[m * RP + r]; ab += Pa[(r * Lmid + m) * I1 + i] * fabs(KM[m * RP + r]); }
        for (int k = 0; k < nchA; ++k) got += m1p[((size_t)k * I1 + i) * RP + r];
        eM1 = fmax(eM1, (double)(fabsl(got - ex) / ab));
      }
      for (int64_t m = 0; m < Lmid; ++m) {
        long double ex = 0, ab = 0; double got = 0;
        for (int64_t i = 0; i < I1; ++i) { ex += P[(r * Lmid + m) * I1 + i] * A1[i * RP + r]; ab += Pa[(r * Lmid + m) * I1 + i] * fabs(A1[i * RP + r]); }
        for (int b = 0; b < nb; ++b) got += zp[((size_t)b * Lmid + m) * RP + r];
        eZ = fmax(eZ, (double)(fabsl(got - ex) / ab));
      }
      for (int64_t c = 0; c < C; ++c) {
        long double ex = 0, ab = 0; double got = 0;
        for (int64_t i = 0; i < I1; ++i) { ex += U[(r * C + c) * I1 + i] * A1[i * RP + r]; ab += Ua[(r * C + c) * I1 + i] * fabs(A1[i * RP + r]); }
        for (int b = 0; b < nb; ++b) got += bp[((size_t)c * nb + b) * RP + r];
        eMN = fmax(eMN, (double)(fabsl(got - ex) / ab));
      }
    }
    printf("correctness (max |err| / sum|terms|): M1 %.3e  Z %.3e  M_N %.3e\n", eM1, eZ, eMN);
    printf("CHECK %s\n", (eM1 < 3e-15 && eZ < 3e-15 && eMN < 3e-15) ? "PASS" : "FAIL");
  }
  // ---- 2. timing at config-4 size
  if (argc > 1 && atoi(argv[1]) > 0) {
    const int64_t I1 = 1000, Lmid = 1000, C = atoi(argv[1]); const int R = 20;
    Setup s; setup(s, I1, Lmid, C, R, nullptr, nsm);
    std::vector<double> BA(C * 24), BB(Lmid * 24), A1(I1 * 24), KM(Lmid * 24);
    for (auto& v : BA) v = nrand();
    for (auto& v : BB) v = nrand();
    for (auto& v : A1) v = nrand();
    for (auto& v : KM) v = nrand();
    CK(cudaMemcpy(s.BA, BA.data(), BA.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(s.BB, BB.data(), BB.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(s.A1, A1.data(), A1.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(s.KM, KM.data(), KM.size() * 8, cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const double bytesA = (double)s.gA.ntiles * s.gA.nkb * kOzABytes, bytesB = (double)s.gB.ntiles * s.gB.nkb * kOzABytes;
    if (argc > 2) {  // per-launch trace of one pass (clock/power behaviour)
      const int mode = atoi(argv[2]);
      for (int k = 0; k < 60; ++k) {
        cudaEventRecord(e0);
        run(s, mode, nsm);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%d:%.2f ", k, ms);
      }
      printf("\n");
      return 0;
    }
    for (int rep = 0; rep < 2; ++rep)
    for (int dbg = 0; dbg < 4; dbg += (rep ? 4 : 1))
    for (int mode = 0; mode < 2; ++mode)
      for (int grid : {nsm, nsm - 24}) {
        s.gA.dbg = s.gB.dbg = dbg;
        run(s, mode, grid); run(s, mode, grid);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        const int K = 10;
        for (int k = 0; k < K; ++k) run(s, mode, grid);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= K;
        const double bytes = mode ? bytesB : bytesA;
        printf("dbg %d pass %c grid %d: %.3f ms  %.1f GB/s of images (%.2f GB); %.1f GB/s of fp64-equivalent 16 GB\n", dbg, mode ? 'B' : 'A', grid, ms, bytes / ms / 1e6, bytes / 1e9, 8.0 * I1 * Lmid * C / ms / 1e6);
      }
  }
  return 0;
}
