// One-column Taylor term of the c2 forward team (d=60, 2 warps, one row per lane,
// named barrier per term): cycles per term with NG of the W=5 operands gathered
// from shared memory and the rest taken from the lane's own register (diagonal).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void cmac(double2& p, double2& q, double2 a, double2 x) {
  p.x = fma(a.x, x.x, p.x); p.y = fma(a.x, x.y, p.y); q.x = fma(-a.y, x.y, q.x); q.y = fma(a.y, x.x, q.y);
}
template <int NG, int NACC>
__global__ void k(double* out, long long* cyc, int terms) {
  __shared__ double2 sm[2 * 64 + 64];
  const int tl = threadIdx.x, i = tl, d = 60;
  double2 a[5]; int col[5];
  const int o[5] = {-19, 19, -20, 20, 0};
  for (int w = 0; w < 5; ++w) { a[w] = make_double2(0.01 * (w + 1), 0.02); int cc = i + o[w]; col[w] = cc < 0 ? 0 : (cc >= d ? d - 1 : cc); }
  for (int q = tl; q < 192; q += blockDim.x) sm[q] = make_double2(1.0, 0.5);
  __syncthreads();
  double2 cur = make_double2(0, 0), own = make_double2(1.0, 0.5);
  int X = 0, Y = 64;
  long long t0 = clock64();
  for (int t = 0; t < terms; ++t) {
    const double r = sm[128 + (t & 15)].x;
    if (i < d) {
      double2 x[5];
#pragma unroll
      for (int w = 0; w < 5; ++w) x[w] = w < NG ? sm[X + col[w]] : own;
      double2 p[NACC], q[NACC];
#pragma unroll
      for (int u = 0; u < NACC; ++u) p[u] = q[u] = make_double2(0, 0);
#pragma unroll
      for (int w = 0; w < 5; ++w) cmac(p[w % NACC], q[w % NACC], a[w], x[w]);
#pragma unroll
      for (int u = 1; u < NACC; ++u) { p[0].x += p[u].x; p[0].y += p[u].y; q[0].x += q[u].x; q[0].y += q[u].y; }
      const double2 tt = make_double2((p[0].x + q[0].x) * r, (p[0].y + q[0].y) * r);
      cur.x += tt.x; cur.y += tt.y;
      own = tt;
      sm[Y + i] = tt;
    }
    asm volatile("bar.sync 1, 64;\n" ::: "memory");
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
#define RUN(NG, NA) k<NG, NA><<<1, 64>>>(out, cyc, T); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("gathers %d accumulators %d: %.1f cycles/term\n", NG, NA, h / (double)T);
  RUN(5, 1) RUN(5, 2) RUN(4, 1) RUN(4, 2) RUN(3, 2) RUN(0, 2)
  return 0;
}
