// harris_shfl_nw2.cu -- instantiation of the warp-shuffle Harris kernel for
// NW=2 warps per CTA (separate TU for a parallel build).
#include "harris_shfl.cuh"

namespace icl {
template cudaError_t dispatch_hshfl<2>(const HarrisParams& p, int batch, int S, cudaStream_t s);
template cudaError_t dispatch_hshfl_tma<2>(const HarrisParams& p, int batch, int S, cudaStream_t s);
}  // namespace icl
