// nlm_x2_more.cu -- further (patch, search) radii of the NLM variant "boxsum_x2"
// (nlm_x2.cuh), every combination with P <= 3 whose two-tile CTA fits two per SM
// (shared memory <= 113 KB).
#include "nlm_x2.cuh"

namespace icl {

#define ICL_X2_MORE(X) X(0, 1) X(0, 2) X(0, 3) X(0, 4) X(0, 5) X(1, 1) X(1, 2) X(1, 4) X(2, 1) X(2, 2) X(2, 4) \
  X(3, 1) X(3, 2) X(3, 3) X(3, 4)

bool nlm_x2_more_supported(int P, int S) {
#define ICL_X2_SUP(PP, SS) if (P == PP && S == SS) return true;
  ICL_X2_MORE(ICL_X2_SUP)
#undef ICL_X2_SUP
  return false;
}

cudaError_t launch_nlm_x2_more(const NlmCall& c, cudaStream_t s) {
  NlmParams p = make_nlm_params(c);
#define ICL_X2_RUN(PP, SS) if (c.P == PP && c.S == SS) return launch_x2<PP, SS>(p, c.batch, s);
  ICL_X2_MORE(ICL_X2_RUN)
#undef ICL_X2_RUN
  return cudaErrorInvalidValue;
}

}  // namespace icl
