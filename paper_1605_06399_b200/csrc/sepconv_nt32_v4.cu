// sepconv_nt32_v4.cu -- instantiation of the streaming sepconv kernel for
// NT=32 threads per CTA, VEC=4 (separate TU for a parallel build).
#include "sepconv_stream.cuh"

namespace icl {
template cudaError_t dispatch_stream<32, 4>(const SepParams& p, int R, int batch, int S, cudaStream_t s);
template cudaError_t dispatch_stream_tma<32>(const SepParams& p, int R, int batch, int S, cudaStream_t s);
}  // namespace icl
