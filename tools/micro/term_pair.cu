// Two Taylor terms per barrier for the c2 chain (d = 60, 2 warps, one row per lane):
//   T_{j+1} = A T_j r1,  T_{j+2} = A^2 T_j r1 r2  (A^2 precomputed per step, 13-point stencil),
// both from the same input; only T_{j+2} is stored.  Compare with tools/micro/term1.cu
// (one term per barrier: 228-265 cycles per term).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void cmac(double2& p, double2& q, double2 a, double2 x) {
  p.x = fma(a.x, x.x, p.x); p.y = fma(a.x, x.y, p.y); q.x = fma(-a.y, x.y, q.x); q.y = fma(a.y, x.x, q.y);
}
template <int W2>
__global__ void k(double* out, long long* cyc, int pairs) {
  __shared__ double2 sm[2 * 64 + 64];
  const int i = threadIdx.x, d = 60;
  double2 a[5], a2[W2]; int col[5], col2[W2];
  const int o[5] = {-19, 19, -20, 20, 0};
  const int o2[13] = {0, -1, 1, -19, 19, -20, 20, -38, 38, -39, 39, -40, 40};
  for (int w = 0; w < 5; ++w) { a[w] = make_double2(0.01 * (w + 1), 0.02); int c = i + o[w]; col[w] = c < 0 ? 0 : (c >= d ? d - 1 : c); }
  for (int w = 0; w < W2; ++w) { a2[w] = make_double2(0.001 * (w + 1), 0.002); int c = i + o2[w % 13]; col2[w] = c < 0 ? 0 : (c >= d ? d - 1 : c); }
  for (int q = i; q < 192; q += blockDim.x) sm[q] = make_double2(1.0, 0.5);
  __syncthreads();
  double2 cur = make_double2(0, 0);
  int X = 0, Y = 64;
  long long t0 = clock64();
  for (int t = 0; t < pairs; ++t) {
    const double r1 = sm[128 + (t & 7)].x, r2 = sm[136 + (t & 7)].x;
    if (i < d) {
      double2 p0 = make_double2(0, 0), q0 = p0, p1 = p0, q1 = p0, u0 = p0, v0 = p0, u1 = p0, v1 = p0;
#pragma unroll
      for (int w = 0; w < 5; ++w) { if (w & 1) cmac(p1, q1, a[w], sm[X + col[w]]); else cmac(p0, q0, a[w], sm[X + col[w]]); }
#pragma unroll
      for (int w = 0; w < W2; ++w) { if (w & 1) cmac(u1, v1, a2[w], sm[X + col2[w]]); else cmac(u0, v0, a2[w], sm[X + col2[w]]); }
      const double2 t1 = make_double2(((p0.x + q0.x) + (p1.x + q1.x)) * r1, ((p0.y + q0.y) + (p1.y + q1.y)) * r1);
      const double rr = r1 * r2;
      const double2 t2 = make_double2(((u0.x + v0.x) + (u1.x + v1.x)) * rr, ((u0.y + v0.y) + (u1.y + v1.y)) * rr);
      cur.x += t1.x + t2.x; cur.y += t1.y + t2.y;
      sm[Y + i] = t2;
    }
    asm volatile("bar.sync 1, 64;\n" ::: "memory");
    int tmp = X; X = Y; Y = tmp;
  }
  long long t1 = clock64();
  out[i] = cur.x + cur.y;
  if (i == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; long long h;
  cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64);
  const int T = 10000;
#define RUN(W2) k<W2><<<1, 64>>>(out, cyc, T); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("pair step, A^2 width %d: %.1f cycles per pair = %.1f per term\n", W2, h / (double)T, h / (2.0 * T));
  RUN(13) RUN(16) RUN(9)
  return 0;
}
