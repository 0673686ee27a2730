// Per-round synchronisation cost inside a cluster (one CTA per SM, 128 threads):
//   0: st.shared::cluster halo push + barrier.cluster arrive.release / wait.acquire (MEMBAR.ALL.GPU)
//   1: same push + relaxed arrive (no ordering guarantee; lower bound only)
//   2: st.async halo push with mbarrier complete_tx into the neighbours' alternating buffers,
//      wait on the own buffer's mbarrier + bar.sync (neighbour-only, no cluster barrier)
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned r) {
  unsigned o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o;
}
template <int V>
__global__ void k(long long* cyc, int n, int halo) {
  __shared__ __align__(16) double2 buf[2][256];
  __shared__ __align__(8) unsigned long long mb[2];
  unsigned rank, ns;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ns));
  const int t = threadIdx.x;
  const bool hasL = rank > 0, hasR = rank + 1 < ns;
  const unsigned nbytes = 16u * halo * ((hasL ? 1 : 0) + (hasR ? 1 : 0));
  if (t == 0) {
    for (int b = 0; b < 2; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mb[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (V == 2 && t == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&mb[1])), "r"(nbytes) : "memory");
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const int ob = (i + 1) & 1;  // output buffer of round i
    double2 v = make_double2((double)i, (double)t);
    buf[ob][64 + t] = v;
    if (V == 2) {
      if (t < halo && hasL)
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(mapa(sa(&buf[ob][192 + t]), rank - 1)), "d"(v.x), "d"(v.y), "r"(mapa(sa(&mb[ob]), rank - 1)) : "memory");
      if (t >= 128 - halo && hasR)
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(mapa(sa(&buf[ob][t - 128 + halo]), rank + 1)), "d"(v.x), "d"(v.y), "r"(mapa(sa(&mb[ob]), rank + 1)) : "memory");
      __syncthreads();
      // wait for the neighbours' pushes into buffer ob (phase (i+1)/2... parity of use count)
      const unsigned par = (unsigned)(i >> 1) & 1u;
      asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(sa(&mb[ob])), "r"(par) : "memory");
      // arm the other buffer for round i + 1 (its previous phase completed at round i - 1)
      if (t == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&mb[ob ^ 1])), "r"(nbytes) : "memory");
    } else {
      if (t < halo && hasL) asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(mapa(sa(&buf[ob][192 + t]), rank - 1)), "d"(v.x), "d"(v.y) : "memory");
      if (t >= 128 - halo && hasR) asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(mapa(sa(&buf[ob][t - 128 + halo]), rank + 1)), "d"(v.x), "d"(v.y) : "memory");
      if (V == 0) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
      else asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
    }
  }
  long long t1 = clock64();
  if (t == 0 && rank == 0) cyc[0] = t1 - t0;
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
int main() {
  long long* cyc; long long h;
  cudaMalloc(&cyc, 64);
  void* fs[3] = {(void*)k<0>, (void*)k<1>, (void*)k<2>};
  const char* nm[3] = {"cluster barrier (release)", "cluster barrier (relaxed)", "st.async + mbarrier"};
  for (int v = 0; v < 3; ++v) cudaFuncSetAttribute(fs[v], cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {4, 8, 16}) for (int halo : {4, 32}) for (int v = 0; v < 3; ++v) {
    cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(cs); cfg.blockDim = dim3(128);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = 4000;
    void* args[3] = {&cyc, &n, &halo};
    cudaError_t e = cudaLaunchKernelExC(&cfg, fs[v], args);
    cudaError_t e2 = cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("cluster %2d halo %2d %-28s %7.1f cycles/round (%s %s)\n", cs, halo, nm[v], h / (double)n, cudaGetErrorString(e), cudaGetErrorString(e2));
  }
  return 0;
}
