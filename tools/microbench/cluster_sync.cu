// Cost of one cluster-wide rendezvous on B200 (per-column step of the LU panel kernel):
//   mode 0: cooperative_groups cluster.sync()
//   mode 1: barrier.cluster.arrive.relaxed + barrier.cluster.wait
//   mode 2: DSMEM mbarriers: each warp arrives (release.cluster) on every CTA's barrier, waits locally
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void k(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ __align__(8) unsigned long long bar[2];
  __shared__ double slot[64];
  const int CL = cl.num_blocks(), rank = cl.block_rank();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    for (int p = 0; p < 2; ++p)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[p])), "r"(nw * CL));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cl.sync();
  long long t0 = clock64();
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    const int par = it & 1;
    // each warp publishes one value into every CTA
    for (int r = 0; r < CL; ++r)
      if (lane == 0) cl.map_shared_rank(slot, r)[(rank * nw + wid) & 63] = it + wid;
    if (MODE == 0) {
      cl.sync();
    } else if (MODE == 1) {
      asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    } else {
      __syncwarp();
      if (lane < CL) {
        unsigned remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(&bar[par])), "r"(lane));
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
      }
      const unsigned phase = (it >> 1) & 1;
      asm volatile(
          "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
              smem_u32(&bar[par])),
          "r"(phase)
          : "memory");
    }
    acc += slot[(wid + 1) & 63];
  }
  long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0 && rank == 0) { out[0] = (t1 - t0) / iters; out[1] = (long long)acc; }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  for (int mode = 0; mode < 3; ++mode)
    for (int CL = 1; CL <= 8; CL *= 2) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(CL);
      cfg.blockDim = dim3(256);
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = CL; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
      cfg.attrs = a; cfg.numAttrs = 1;
      cudaError_t e;
      if (mode == 0) e = cudaLaunchKernelEx(&cfg, k<0>, 2000, d);
      else if (mode == 1) e = cudaLaunchKernelEx(&cfg, k<1>, 2000, d);
      else e = cudaLaunchKernelEx(&cfg, k<2>, 2000, d);
      cudaDeviceSynchronize();
      long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("mode %d CL %d: %lld cycles/iter (%s)\n", mode, CL, h[0], cudaGetErrorString(e));
    }
  return 0;
}
