// Cluster sweep engine instantiations for ELL width 7 (see lg_sweep_cl.cuh).
#include "lg_sweep_cl.cuh"

LG_CL_KERNELS(7)
