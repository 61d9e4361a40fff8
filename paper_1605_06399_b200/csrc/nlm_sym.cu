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

cudaError_t launch_nlm_sym(const NlmCall& c, cudaStream_t s) {
  NlmParams p = make_nlm_params(c);
#define ICL_SYM_RUN(PP, SS) if (c.P == PP && c.S == SS) return launch_sym<PP, SS>(p, c.batch, s);
  ICL_SYM_RADII(ICL_SYM_RUN)
#undef ICL_SYM_RUN
  return cudaErrorInvalidValue;
}

}  // namespace icl
