// Standalone replica of one Taylor-term loop (d=60, W=5 banded, 4 warps: 2 per column)
// to find where the per-term latency goes.  Variants toggle parts of the body.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void cmac(double2& p, double2& q, double2 a, double2 x) {
  p.x = fma(a.x, x.x, p.x); p.y = fma(a.x, x.y, p.y); q.x = fma(-a.y, x.y, q.x); q.y = fma(a.y, x.x, q.y);
}
template <int VAR>
__global__ void k(double* out, long long* cyc, int terms) {
  __shared__ double2 sm[4 * 64 + 64];
  const int tl = threadIdx.x, i = tl & 63, d = 60;
  const bool top = tl < 64;
  const int c = top ? 0 : d;
  double2 a[5]; int col[5];
  for (int w = 0; w < 5; ++w) { a[w] = make_double2(0.01 * (w + 1), 0.02); int o[5] = {0, -19, 19, -20, 20}; int cc = i + o[w]; col[w] = cc < 0 ? 0 : (cc >= d ? d - 1 : cc); }
  for (int q = tl; q < 4 * 64 + 64; q += blockDim.x) sm[q] = make_double2(1.0, 0.5);
  __syncthreads();
  double2 cur = make_double2(0, 0);
  int X = 0, Y = 128;
  long long t0 = clock64();
  for (int t = 0; t < terms; ++t) {
    const double r = (VAR & 4) ? 0.5 : sm[256 + (t & 15)].x;
    if (i < d) {
      double2 x[5];
      for (int w = 0; w < 5; ++w) x[w] = (VAR & 1) ? a[w] : sm[X + c + col[w]];
      double2 p0 = make_double2(0, 0), q0 = p0, p1 = p0, q1 = p0;
      for (int w = 0; w < 5; ++w) { if (w & 1) cmac(p1, q1, a[w], x[w]); else cmac(p0, q0, a[w], x[w]); }
      const double2 tt = make_double2(((p0.x + q0.x) + (p1.x + q1.x)) * r, ((p0.y + q0.y) + (p1.y + q1.y)) * r);
      cur.x += tt.x; cur.y += tt.y;
      if (!(VAR & 8)) sm[Y + c + i] = tt;
    }
    if (!(VAR & 2)) asm volatile("bar.sync 1, 128;\n" ::: "memory");
    int tmp = X; X = Y; Y = tmp;
  }
  long long t1 = clock64();
  out[tl] = cur.x + cur.y;
  if (tl == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; long long h;
  cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64);
  const int T = 20000;
#define RUN(V, name) k<V><<<1, 128>>>(out, cyc, T); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%-40s %.1f cycles/term\n", name, h / (double)T);
  RUN(0, "full term");
  RUN(1, "no LDS of x");
  RUN(2, "no bar.sync");
  RUN(4, "r from register");
  RUN(8, "no STS");
  RUN(2 | 8, "no bar, no STS");
  RUN(1 | 2 | 8, "compute only");
  RUN(4 | 2 | 8, "no bar/STS, r reg");
  return 0;
}
