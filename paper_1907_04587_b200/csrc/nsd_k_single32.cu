// The single-scene kernels of the fp32 mode: nsd_k_single.cu compiled with the
// operator's J/C coefficients stored as float (NSD_OP32, nsd_engine.cuh opg/ops).
#define NSD_OP32 1
#include "nsd_k_single.cu"
