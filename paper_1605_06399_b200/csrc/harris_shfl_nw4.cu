// harris_shfl_nw4.cu -- instantiation of the warp-shuffle Harris kernel for
// NW=4 warps per CTA (separate TU for a parallel build).
#include "harris_shfl.cuh"

namespace icl {
template cudaError_t dispatch_hshfl<4>(const HarrisParams& p, int batch, int S, cudaStream_t s);
}  // namespace icl
