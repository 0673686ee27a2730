// Cluster sweep engine instantiations for ELL width 9 (see lg_sweep_cl.cuh).
#include "lg_sweep_cl.cuh"

LG_CL_KERNELS(9)
