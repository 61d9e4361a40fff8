// nlm_x2.cu -- dispatch of the NLM variant "boxsum_x2" (kernel: nlm_x2.cuh); the common
// (patch, search) radii here, more in nlm_x2_more.cu (a separate TU for a parallel build).
#include "nlm_x2.cuh"

namespace icl {

bool nlm_x2_more_supported(int P, int S);
cudaError_t launch_nlm_x2_more(const NlmCall& c, cudaStream_t s);

bool nlm_x2_supported(int P, int S) {
  return (P == 2 && S == 5) || (P == 1 && S == 3) || (P == 2 && S == 3) || (P == 1 && S == 5) ||
         nlm_x2_more_supported(P, S);
}

cudaError_t launch_nlm_x2(const NlmCall& c, cudaStream_t s) {
  NlmParams p = make_nlm_params(c);
  if (c.P == 2 && c.S == 5) return launch_x2<2, 5>(p, c.batch, s);
  if (c.P == 1 && c.S == 3) return launch_x2<1, 3>(p, c.batch, s);
  if (c.P == 2 && c.S == 3) return launch_x2<2, 3>(p, c.batch, s);
  if (c.P == 1 && c.S == 5) return launch_x2<1, 5>(p, c.batch, s);
  return launch_nlm_x2_more(c, s);
}

}  // namespace icl
