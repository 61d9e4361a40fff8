// sepconv_nt64_v1.cu -- instantiation of the streaming sepconv kernel for
// NT=64 threads per CTA, VEC=1 (separate TU for a parallel build).
#include "sepconv_stream.cuh"

namespace icl {
template cudaError_t dispatch_stream<64, 1>(const SepParams& p, int R, int batch, int S, cudaStream_t s);
}  // namespace icl
