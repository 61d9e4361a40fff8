// nlm_common.cuh -- parameter block and helpers shared by the NLM kernels.
#pragma once
#include "common.cuh"
#include "internal.h"

namespace icl {

struct NlmParams {
  SrcView src;
  DstView dst;
  int P, S;
  float coef;
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

static inline NlmParams make_nlm_params(const NlmCall& c) {
  NlmParams p;
  p.src = c.src;
  p.dst = c.dst;
  p.P = c.P;
  p.S = c.S;
  p.coef = c.coef;
  return p;
}

}  // namespace icl
