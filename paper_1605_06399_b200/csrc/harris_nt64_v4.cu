// harris_nt64_v4.cu -- instantiation of the streaming Harris kernel for
// NT=64 threads per CTA, VEC=4 (separate TU for a parallel build).
#include "harris_stream.cuh"

namespace icl {
template cudaError_t dispatch_hs<64, 4>(const HarrisParams& p, int batch, int S, cudaStream_t s);
}  // namespace icl
