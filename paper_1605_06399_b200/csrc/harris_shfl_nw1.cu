// harris_shfl_nw1.cu -- instantiation of the warp-shuffle Harris kernel for
// NW=1 warp per CTA (120-column strips: twice the CTAs of NW=2 for images that
// do not fill the GPU, e.g. BASELINE configs[1], 2048^2; separate TU for a parallel build).
#include "harris_shfl.cuh"

namespace icl {
template cudaError_t dispatch_hshfl<1>(const HarrisParams& p, int batch, int S, cudaStream_t s);
}  // namespace icl
