// Max co-resident clusters per cluster size with one CTA per SM (228 KB dynamic smem):
// reveals how the 148 SMs group into GPCs for cluster scheduling.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_probe() { extern __shared__ char s[]; if (threadIdx.x == 9999) s[0] = 0; }
int main() {
  const int smem = 227 * 1024;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs = 1; cs <= 16; ++cs) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_probe, &cfg);
    printf("cluster %2d: max active %3d (%3d SMs) %s\n", cs, n, n * cs, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
