// Single translation unit of libbimine_b200.so: the device tables
// (exp table, quotient table) and every kernel live in one module, so one
// cudaMemcpyToSymbol initialises what every kernel reads.
#include "bm_kernels.cu"
#include "bm_seq.cu"
#include "bm_ring.cu"
#include "bm_band.cu"
#include "bm_merge.cu"
#include "bm_api.cu"
