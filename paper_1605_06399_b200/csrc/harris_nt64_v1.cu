// harris_nt64_v1.cu -- instantiation of the streaming Harris kernel for
// NT=64 threads per CTA, VEC=1 (separate TU for a parallel build).
#include "harris_stream.cuh"

namespace icl {
template cudaError_t dispatch_hs<64, 1>(const HarrisParams& p, int batch, int S, cudaStream_t s);
}  // namespace icl
