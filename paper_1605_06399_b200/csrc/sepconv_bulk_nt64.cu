// sepconv_bulk_nt64.cu -- instantiation of the TMA-fed sepconv kernel for NT=64
// threads per CTA (separate TU for a parallel build).
#include "sepconv_bulk.cuh"

namespace icl {
template cudaError_t dispatch_bulk<64>(const SepParams& p, int R, int batch, int S, cudaStream_t s);
}  // namespace icl
