// nlm_sym.cu -- dispatch of the NLM variant "sym_tmem" (kernel: nlm_sym.cuh).
#include "nlm_sym.cuh"

namespace icl {

#define ICL_SYM_RADII(X) X(2, 5) X(1, 3) X(2, 3) X(1, 5) X(3, 5) X(2, 7) X(3, 7) X(1, 1) X(2, 2)

bool nlm_sym_supported(int P, int S) {
#define ICL_SYM_SUP(PP, SS) if (P == PP && S == SS) return true;
  ICL_SYM_RADII(ICL_SYM_SUP)
#undef ICL_SYM_SUP
  return false;
}

// "sym_ring": the H ring in tensor memory (one CTA per SM), instantiated where it fits 512 columns
bool nlm_sym_ring_supported(int P, int S) { return (P == 2 && S == 5) || (P == 1 && S == 3); }

cudaError_t launch_nlm_sym_ring(const NlmCall& c, cudaStream_t s) {
  NlmParams p = make_nlm_params(c);
  if (c.P == 2 && c.S == 5) return launch_sym<2, 5, true>(p, c.batch, s);
  if (c.P == 1 && c.S == 3) return launch_sym<1, 3, true>(p, c.batch, s);
  return cudaErrorInvalidValue;
}

// "sym_tmem8": one 8-warp CTA per SM (the warps of an SM run each pass together)
bool nlm_sym8_supported(int P, int S) { return (P == 2 && S == 5) || (P == 1 && S == 3); }

cudaError_t launch_nlm_sym8(const NlmCall& c, cudaStream_t s) {
  NlmParams p = make_nlm_params(c);
  if (c.P == 2 && c.S == 5) return launch_sym<2, 5, false, 8>(p, c.batch, s);
  if (c.P == 1 && c.S == 3) return launch_sym<1, 3, false, 8>(p, c.batch, s);
  return cudaErrorInvalidValue;
}

cudaError_t launch_nlm_sym(const NlmCall& c, cudaStream_t s) {
  NlmParams p = make_nlm_params(c);
#define ICL_SYM_RUN(PP, SS) if (c.P == PP && c.S == SS) return launch_sym<PP, SS>(p, c.batch, s);
  ICL_SYM_RADII(ICL_SYM_RUN)
#undef ICL_SYM_RUN
  return cudaErrorInvalidValue;
}

}  // namespace icl
