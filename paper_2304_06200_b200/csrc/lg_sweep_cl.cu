// Cluster sweep engine (lg_sweep_cl.cuh): shared-memory sizing and kernel lookup
// over the per-ELL-width instantiation units lg_sweep_cl_w3.cu .. lg_sweep_cl_w9.cu.
#include "lg_types.h"

extern "C" void* lg_cl_kernel_w3(int backward, int maxc, int small);
extern "C" void* lg_cl_kernel_w4(int backward, int maxc, int small);
extern "C" void* lg_cl_kernel_w5(int backward, int maxc, int small);
extern "C" void* lg_cl_kernel_w6(int backward, int maxc, int small);
extern "C" void* lg_cl_kernel_w7(int backward, int maxc, int small);
extern "C" void* lg_cl_kernel_w8(int backward, int maxc, int small);
extern "C" void* lg_cl_kernel_w9(int backward, int maxc, int small);

// acw = Kc * Wc when the backward kernel stages the control-generator rows, else 0.
extern "C" int lg_cl_smem_words(int R, int H, int Q, int E, int cmax, int W, int acw) {
  return lg_cl_mb_word(R, H, Q, E, cmax, W, acw) + 1;  // + the two exchange mbarriers
}

// small != 0: the <= 256-thread variant (see ClRegs).
extern "C" void* lg_cl_kernel(int backward, int W, int maxc, int small) {
  switch (W) {
    case 3: return lg_cl_kernel_w3(backward, maxc, small);
    case 4: return lg_cl_kernel_w4(backward, maxc, small);
    case 5: return lg_cl_kernel_w5(backward, maxc, small);
    case 6: return lg_cl_kernel_w6(backward, maxc, small);
    case 7: return lg_cl_kernel_w7(backward, maxc, small);
    case 8: return lg_cl_kernel_w8(backward, maxc, small);
    case 9: return lg_cl_kernel_w9(backward, maxc, small);
  }
  return nullptr;
}
