// harris_slide_nw2.cu -- instantiation of the separable-window Harris kernel for
// NW=2 warps per CTA (separate TU for a parallel build).
#include "harris_slide.cuh"

namespace icl {
template cudaError_t dispatch_hslide<2, 1>(const HarrisParams& p, int batch, int S, cudaStream_t s);
template cudaError_t dispatch_hslide<2, 2>(const HarrisParams& p, int batch, int S, cudaStream_t s);
template cudaError_t dispatch_hslide<2, 1, true>(const HarrisParams& p, int batch, int S, cudaStream_t s);
}  // namespace icl
