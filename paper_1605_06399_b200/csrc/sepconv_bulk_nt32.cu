// sepconv_bulk_nt32.cu -- instantiation of the TMA-fed sepconv kernel for NT=32
// threads per CTA (separate TU for a parallel build).
#include "sepconv_bulk.cuh"

namespace icl {
template cudaError_t dispatch_bulk<32>(const SepParams& p, int R, int batch, int S, cudaStream_t s);
}  // namespace icl
