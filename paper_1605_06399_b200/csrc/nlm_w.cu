// nlm_w.cu -- dispatch of the NLM variant "boxsum_w" (kernel: nlm_w.cuh) for the
// (patch, search) radii whose per-thread windows fit: S <= 5 (ox groups of <= 3).
#include "nlm_w.cuh"

namespace icl {

#define ICL_W_SET(X) X(2, 5) X(1, 3) X(2, 3) X(1, 5) X(0, 1) X(1, 1) X(2, 2) X(3, 3) X(2, 4) X(3, 5)

bool nlm_w_supported(int P, int S) {
#define ICL_W_SUP(PP, SS) if (P == PP && S == SS) return true;
  ICL_W_SET(ICL_W_SUP)
#undef ICL_W_SUP
  return false;
}

cudaError_t launch_nlm_w(const NlmCall& c, int unroll, cudaStream_t s) {
  NlmParams p = make_nlm_params(c);
  if (unroll != 1) return cudaErrorInvalidValue;  // (oy unrolled by 2 / fully: 13.1 / 12.5 ms, spills)
#define ICL_W_RUN(PP, SS) if (c.P == PP && c.S == SS) return launch_w<PP, SS>(p, c.batch, s);
  ICL_W_SET(ICL_W_RUN)
#undef ICL_W_RUN
  return cudaErrorInvalidValue;
}

}  // namespace icl
