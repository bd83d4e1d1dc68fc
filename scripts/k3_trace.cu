// Standalone trace build of libmlsort with MLSORT_K3_TRACE: exposes a setter for the trace buffer.
#define MLSORT_K3_TRACE 1
#include "../paper_1805_04272_b200/csrc/mlsort.cu"
extern "C" int mlsort_debug_set_k3_trace(void* dptr) {
    return cudaMemcpyToSymbol(mlsort::g_k3_trace, &dptr, sizeof(void*)) == cudaSuccess ? 0 : 6;
}
