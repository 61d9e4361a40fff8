// sepconv_bulk_nt128.cu -- instantiation of the TMA-fed sepconv kernel for NT=128
// threads per CTA (separate TU for a parallel build).
#include "sepconv_bulk.cuh"

namespace icl {
template cudaError_t dispatch_bulk<128>(const SepParams& p, int R, int batch, int S, cudaStream_t s);
}  // namespace icl
