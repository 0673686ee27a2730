// Co-resident cluster count per cluster size (1 CTA per SM: 200 KB dynamic smem).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k() { extern __shared__ char s[]; if (threadIdx.x == 9999) s[0] = 0; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs = 1; cs <= 16; ++cs) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = 0; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: %3d active clusters (%3d SMs) %s\n", cs, n, n * cs, e ? cudaGetErrorString(e) : "");
  }
}
