// Micro-benchmark: DMMA.8x8x4 issue rate for a REAL FP64 GEMM inner loop (the three real products of a
// matrix-level 3M complex GEMM), operands from shared memory as LDS.128 pairs of consecutive k:
//   warp tile (8 MT) x (8 NT); per iteration = two k4-steps: MT + NT LDS.128, 2 MT NT DMMAs.
// Prints TFLOP/s for CTAs of 128 threads at 1..4 CTAs per SM.  Compare tools/micro/dmma.cu (the
// fragment-level 3M mix of lg_k_zgemm_taylor_n32: 6 LDS.128 + 6 DADD per 24 DMMAs).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MT, int NT>
__global__ void __launch_bounds__(128) k(double* out, int iters, double seed) {
  __shared__ double2 s[2048];
  for (int i = threadIdx.x; i < 2048; i += 128) s[i] = make_double2(seed * i, seed - i);
  __syncthreads();
  double t[MT][NT][2];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b) t[a][b][0] = t[a][b][1] = 0.0;
  const int lane = threadIdx.x & 31;
  int off = lane;
  for (int it = 0; it < iters; ++it) {
    double2 a[MT], b[NT];
#pragma unroll
    for (int m = 0; m < MT; ++m) a[m] = s[(off + m * 40) & 2047];
#pragma unroll
    for (int n = 0; n < NT; ++n) b[n] = s[(off + 1024 + n * 40) & 2047];
    off += 33;
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int n = 0; n < NT; ++n) dmma(t[m][n][0], t[m][n][1], a[m].x, b[n].x);
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int n = 0; n < NT; ++n) dmma(t[m][n][0], t[m][n][1], a[m].y, b[n].y);
  }
  double acc = 0.0;
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b) acc += t[a][b][0] + t[a][b][1];
  out[blockIdx.x * 128 + threadIdx.x] = acc;
}

template <int MT, int NT>
void run(double* out, int sms) {
  const int iters = 20000;
  for (int per = 1; per <= 4; ++per) {
    const int grid = sms * per;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k<MT, NT>, 128, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<MT, NT><<<grid, 128>>>(out, 100, 1e-3);
    cudaEventRecord(e0);
    k<MT, NT><<<grid, 128>>>(out, iters, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = (double)grid * 4 /*warps*/ * iters * 2 * MT * NT * 512;
    printf("tile %dx%d  CTAs/SM %d (fit %d)  %.2f TFLOP/s\n", 8 * MT, 8 * NT, per, occ, flops / (ms * 1e-3) / 1e12);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 4 * 128);
  run<4, 4>(out, sms);
  run<8, 4>(out, sms);
  run<4, 8>(out, sms);
  run<6, 4>(out, sms);
  run<8, 2>(out, sms);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
