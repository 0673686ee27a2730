// Cluster barrier latency vs cluster size, with and without a DSMEM store per round.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(long long* cyc, int n, int store) {
  __shared__ double buf[64];
  unsigned rank, ns;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ns));
  unsigned a = (unsigned)__cvta_generic_to_shared(&buf[threadIdx.x & 63]), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"((rank + 1) % ns));
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (store) asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"((double)i) : "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) cyc[blockIdx.x / ns] = t1 - t0;
}
int main() {
  long long* cyc; long long h;
  cudaMalloc(&cyc, 4096);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {2, 4, 8, 16}) for (int threads : {128, 640}) for (int st : {0, 1}) {
    cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(cs); cfg.blockDim = dim3(threads);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = 2000;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, cyc, n, st);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    int ncl = 0; cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
    printf("cluster %2d threads %4d store %d: %7.1f cycles/barrier  (%s) max active clusters %d\n", cs, threads, st, h / (double)n, cudaGetErrorString(e), ncl);
  }
  return 0;
}
