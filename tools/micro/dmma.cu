// Micro-benchmark: FP64 tensor (DMMA.8x8x4) issue rate on B200 with the c5 kernel's instruction mix.
//   mode 0: 24 independent DMMAs per k-step (the 16 x 32 warp tile's 3M products), operands in registers
//   mode 1: + the 6 DADDs forming the 3M operand sums
//   mode 2: + 6 LDS.128 fragment loads from shared memory (the full inner loop without cp.async)
//   mode 3: mode 2 with the next k-step's fragments loaded before this k-step's DMMAs (explicit prefetch)
// Prints TFLOP/s (8x8x4x2 flops per DMMA) for CTAs of 128 threads at 1..4 CTAs per SM.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE>
__global__ void __launch_bounds__(128) k(double* out, int iters, double seed) {
  __shared__ double2 s[2048];
  for (int i = threadIdx.x; i < 2048; i += 128) s[i] = make_double2(seed * i, seed - i);
  __syncthreads();
  double t[3][2][4][2];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) t[a][b][c][0] = t[a][b][c][1] = 0.0;
  double ar[2] = {seed, seed + 1}, ai[2] = {seed + 2, seed + 3};
  double xr[4] = {seed, seed * 2, seed * 3, seed * 4}, xi[4] = {seed, seed * 5, seed * 6, seed * 7};
  const int lane = threadIdx.x & 31;
  int off = lane;  // 16-byte lane stride: conflict-free LDS.128, like the kernel's tile strides
  double2 na[2], nx[4];
  if (MODE == 3) {
#pragma unroll
    for (int m = 0; m < 2; ++m) na[m] = s[(off + m * 8) & 2047];
#pragma unroll
    for (int n = 0; n < 4; ++n) nx[n] = s[(off + 512 + n * 80) & 2047];
    off += 66;
  }
  for (int it = 0; it < iters; ++it) {
    double sa[2], sx[4];
    if (MODE == 3) {  // consume the prefetched fragments, then issue the next iteration's loads
#pragma unroll
      for (int m = 0; m < 2; ++m) { ar[m] = na[m].x; ai[m] = na[m].y; }
#pragma unroll
      for (int n = 0; n < 4; ++n) { xr[n] = nx[n].x; xi[n] = nx[n].y; }
#pragma unroll
      for (int m = 0; m < 2; ++m) na[m] = s[(off + m * 8) & 2047];
#pragma unroll
      for (int n = 0; n < 4; ++n) nx[n] = s[(off + 512 + n * 80) & 2047];
      off += 66;
    } else if (MODE >= 2) {
#pragma unroll
      for (int m = 0; m < 2; ++m) { const double2 v = s[(off + m * 8) & 2047]; ar[m] = v.x; ai[m] = v.y; }
#pragma unroll
      for (int n = 0; n < 4; ++n) { const double2 v = s[(off + 512 + n * 80) & 2047]; xr[n] = v.x; xi[n] = v.y; }
      off += 66;
    }
    if (MODE >= 1) {
#pragma unroll
      for (int m = 0; m < 2; ++m) sa[m] = ar[m] + ai[m];
#pragma unroll
      for (int n = 0; n < 4; ++n) sx[n] = xr[n] + xi[n];
    } else {
#pragma unroll
      for (int m = 0; m < 2; ++m) sa[m] = ar[m];
#pragma unroll
      for (int n = 0; n < 4; ++n) sx[n] = xr[n];
    }
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < 4; ++n) dmma(t[0][m][n][0], t[0][m][n][1], ar[m], xr[n]);
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < 4; ++n) dmma(t[1][m][n][0], t[1][m][n][1], ai[m], xi[n]);
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < 4; ++n) dmma(t[2][m][n][0], t[2][m][n][1], sa[m], sx[n]);
  }
  double acc = 0.0;
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc += t[a][b][c][0] + t[a][b][c][1];
  out[blockIdx.x * 128 + threadIdx.x] = acc;
}

template <int MODE>
void run(double* out, int sms) {
  const int iters = 20000;
  for (int per = 1; per <= 4; ++per) {
    const int grid = sms * per;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<MODE><<<grid, 128>>>(out, 100, 1e-3);
    cudaEventRecord(e0);
    k<MODE><<<grid, 128>>>(out, iters, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = (double)grid * 4 /*warps*/ * iters * 24 * 512;
    printf("mode %d  CTAs/SM %d  %.2f TFLOP/s\n", MODE, per, flops / (ms * 1e-3) / 1e12);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 4 * 128);
  run<0>(out, sms);
  run<1>(out, sms);
  run<2>(out, sms);
  run<3>(out, sms);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
