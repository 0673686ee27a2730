// Does a warp spinning on mbarrier.try_wait slow a neighbouring team's Taylor term?
// 2-warp team (c2 term: 5 shared-memory gathers, named barrier) + 2 warps that either idle
// (exit), spin on try_wait of a phase that completes only at the end, or spin with nanosleep.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void cmac(double2& p, double2& q, double2 a, double2 x) {
  p.x = fma(a.x, x.x, p.x); p.y = fma(a.x, x.y, p.y); q.x = fma(-a.y, x.y, q.x); q.y = fma(a.y, x.x, q.y);
}
template <int SPIN>
__global__ void k(double* out, long long* cyc, int terms) {
  __shared__ double2 sm[2 * 64 + 64];
  __shared__ __align__(8) unsigned long long mb;
  const int t = threadIdx.x;
  if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&mb)));
  for (int q = t; q < 192; q += blockDim.x) sm[q] = make_double2(1.0, 0.5);
  __syncthreads();
  if (t >= 64) {
    if (SPIN == 0) return;
    const unsigned a = (unsigned)__cvta_generic_to_shared(&mb);
    unsigned done = 0;
    while (!done) {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(a) : "memory");
      if (SPIN == 2 && !done) __nanosleep(200);
    }
    return;
  }
  const int i = t, d = 60;
  double2 a[5]; int col[5];
  const int o[5] = {-19, 19, -20, 20, 0};
  for (int w = 0; w < 5; ++w) { a[w] = make_double2(0.01 * (w + 1), 0.02); int c = i + o[w]; col[w] = c < 0 ? 0 : (c >= d ? d - 1 : c); }
  double2 cur = make_double2(0, 0);
  int X = 0, Y = 64;
  long long t0 = clock64();
  for (int s = 0; s < terms; ++s) {
    const double r = sm[128 + (s & 15)].x;
    if (i < d) {
      double2 p = make_double2(0, 0), q = p;
#pragma unroll
      for (int w = 0; w < 5; ++w) cmac(p, q, a[w], sm[X + col[w]]);
      const double2 tt = make_double2((p.x + q.x) * r, (p.y + q.y) * r);
      cur.x += tt.x; cur.y += tt.y;
      sm[Y + i] = tt;
    }
    asm volatile("bar.sync 1, 64;\n" ::: "memory");
    int tmp = X; X = Y; Y = tmp;
  }
  long long t1 = clock64();
  out[i] = cur.x + cur.y;
  if (i == 0) {
    cyc[0] = t1 - t0;
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"((unsigned)__cvta_generic_to_shared(&mb)) : "memory");
  }
}
int main() {
  double* out; long long* cyc; long long h;
  cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64);
  const int T = 20000;
  const char* nm[3] = {"no spinning warps", "2 warps spinning on try_wait", "2 warps try_wait + nanosleep(200)"};
#define RUN(S) k<S><<<1, 128>>>(out, cyc, T); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%-40s %.1f cycles/term\n", nm[S], h / (double)T);
  RUN(0) RUN(1) RUN(2)
  return 0;
}
