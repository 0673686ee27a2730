// Single-warp Taylor term for d <= 64 (2 rows per lane, rows r = 32k + lane) with the
// term vector in registers and every gather a pair of warp shuffles (both register
// slots of the source lane, then a select): no shared memory, no named barrier.
// Compare with tools/micro/term1.cu (2 warps, shared-memory gathers, bar.sync).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void cmac(double2& p, double2& q, double2 a, double2 x) {
  p.x = fma(a.x, x.x, p.x); p.y = fma(a.x, x.y, p.y); q.x = fma(-a.y, x.y, q.x); q.y = fma(a.y, x.x, q.y);
}
__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
template <int NDIAG, int NACC>
__global__ void k(double* out, long long* cyc, int terms) {
  const int lane = threadIdx.x, d = 60;
  double2 a[2][5]; int src[2][5]; bool hi[2][5];
  const int o[5] = {0, -19, 19, -20, 20};
  double2 x[2], cur[2];
  for (int kk = 0; kk < 2; ++kk) {
    const int r = kk * 32 + lane;
    for (int w = 0; w < 5; ++w) {
      a[kk][w] = make_double2(0.01 * (w + 1), 0.02);
      int c = r + o[w]; c = c < 0 ? 0 : (c >= d ? d - 1 : c);
      src[kk][w] = c & 31; hi[kk][w] = c >= 32;
    }
    x[kk] = make_double2(1.0, 0.5); cur[kk] = make_double2(0, 0);
  }
  long long t0 = clock64();
  for (int t = 0; t < terms; ++t) {
    const double r = 0.5 + 1e-3 * (t & 7);
    double2 nx[2];
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      double2 p[NACC], q[NACC];
#pragma unroll
      for (int u = 0; u < NACC; ++u) p[u] = q[u] = make_double2(0, 0);
#pragma unroll
      for (int w = 0; w < 5; ++w) {
        double2 xv;
        if (w < NDIAG) xv = x[kk];
        else { const double2 v0 = shfl2(x[0], src[kk][w]), v1 = shfl2(x[1], src[kk][w]); xv = hi[kk][w] ? v1 : v0; }
        cmac(p[w % NACC], q[w % NACC], a[kk][w], xv);
      }
#pragma unroll
      for (int u = 1; u < NACC; ++u) { p[0].x += p[u].x; p[0].y += p[u].y; q[0].x += q[u].x; q[0].y += q[u].y; }
      nx[kk] = make_double2((p[0].x + q[0].x) * r, (p[0].y + q[0].y) * r);
    }
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) { cur[kk].x += nx[kk].x; cur[kk].y += nx[kk].y; x[kk] = nx[kk]; }
  }
  long long t1 = clock64();
  out[lane] = cur[0].x + cur[1].y;
  if (lane == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; long long h;
  cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64);
  const int T = 20000;
#define RUN(ND, NA) k<ND, NA><<<1, 32>>>(out, cyc, T); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("1 warp, shuffles, diag-in-reg %d, acc pairs %d: %.1f cycles/term\n", ND, NA, h / (double)T);
  RUN(0, 1) RUN(0, 2) RUN(1, 2) RUN(1, 3)
  return 0;
}
