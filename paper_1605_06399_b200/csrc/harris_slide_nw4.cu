// harris_slide_nw4.cu -- instantiation of the separable-window Harris kernel for
// NW=4 warps per CTA (separate TU for a parallel build).
#include "harris_slide.cuh"

namespace icl {
template cudaError_t dispatch_hslide<4, 1>(const HarrisParams& p, int batch, int S, cudaStream_t s);
template cudaError_t dispatch_hslide<4, 2>(const HarrisParams& p, int batch, int S, cudaStream_t s);
template cudaError_t dispatch_hslide<4, 1, true>(const HarrisParams& p, int batch, int S, cudaStream_t s);
}  // namespace icl
