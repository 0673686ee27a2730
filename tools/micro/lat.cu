// Microbenchmarks: FP64 DFMA dependent latency, LDS latency, named-barrier round trip (2 warps),
// mbarrier handoff between two warps.  Prints cycles per operation.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double* out, long long* cyc, double a, double b, int n) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}
__global__ void k_dfma_tp(double* out, long long* cyc, double a, double b, int n) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0);
}
__global__ void k_lds(int* out, long long* cyc, int n) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = s[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_bar(long long* cyc, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("bar.sync 1, 64;" ::: "memory");
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_syncthreads(long long* cyc, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; int* iout;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 4096); cudaMalloc(&iout, 1 << 20);
  long long h[148];
  const int n = 4096;
  k_dfma<<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", h[0] / (4.0 * n));
  for (int w : {1, 2, 4, 8, 16, 32}) {
    k_dfma_tp<<<1, 32 * w>>>(out, cyc, 1.0000001, 1e-9, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA throughput, %2d warps/SM: %.3f warp-instr/cycle/SM (%.1f lanes/clk)\n", w, (8.0 * n * w) / h[0], 32.0 * (8.0 * n * w) / h[0]);
  }
  k_lds<<<1, 32>>>(iout, cyc, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("LDS dependent latency: %.2f cycles\n", h[0] / (double)n);
  k_bar<<<1, 64>>>(cyc, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("bar.sync 1,64 (2 warps): %.2f cycles\n", h[0] / (double)n);
  for (int t : {64, 128, 256, 512, 1024}) {
    k_syncthreads<<<1, t>>>(cyc, n); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("__syncthreads %4d threads: %.2f cycles\n", t, h[0] / (double)n);
  }
  return 0;
}
