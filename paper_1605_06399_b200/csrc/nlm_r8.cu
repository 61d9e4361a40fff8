// nlm_r8.cu -- NLM variant "boxsum_r8": the boxsum_32x32 structure (offset-
// major separable patch sums, 256 threads, 3 CTAs/SM) with less shared-memory
// traffic and fewer instructions per (pixel, offset) pair.  (NLM is not in
// PAPER.md; definition DESIGN.md R11-R14.)
//
// Per search row oy:
//   phase A  (thread = 4-column row segment, all 2S+1 ox) horizontal patch
//            sums H_o with a sliding sum along the 4 columns (+new^2 - old^2);
//   phase B  (thread = column x, 8 consecutive rows, one half of the ox
//            range) vertical sums with a sliding window over the 8 rows, then
//            w = 2^(-d*coef), num += w u(q), den += w.
// Shared-memory words per pair: phase A 0.6 load + 1.1 store, phase B 1.5 H
// + 1 u(q) = 4.2 (boxsum_32x32: 4.7).  FP32 per pair ~10.6 (32x32: ~15).
// The two ox halves are added at the end in a fixed order.
#include "nlm_common.cuh"

namespace icl {

template <int P, int S>
struct R8Geom {
  static constexpr int TW = 32, TH = 32, NT = 256;
  static constexpr int HR = P + S;
  static constexpr int UW0 = TW + 2 * HR;
  static constexpr int UW = ((UW0 + 30) / 32) * 32 + 1;  // == 1 (mod 32)
  static constexpr int UH = TH + 2 * HR;
  static constexpr int HROWS = TH + 2 * P;
  static constexpr int NO = 2 * S + 1;
  static constexpr int NOA = (NO + 1) / 2;  // ox handled by half 0; the rest by half 1
  static constexpr int UOFF = ((UH * UW + 3) / 4) * 4;
  static constexpr int HSZ = NO * HROWS * TW;
  static constexpr int RED = 4 * TH * TW;
  static constexpr size_t smem_bytes = (size_t)(UOFF + (HSZ > RED ? HSZ : RED)) * sizeof(float);
};

template <int P, int S>
__global__ void __launch_bounds__(256, 3) nlm_box_r8(NlmParams p) {
  using G = R8Geom<P, S>;
  constexpr int TW = G::TW, TH = G::TH, HR = G::HR, UW = G::UW, UW0 = G::UW0, UH = G::UH;
  constexpr int HROWS = G::HROWS, NO = G::NO, NOA = G::NOA, PW = 2 * P + 1;
  extern __shared__ __align__(16) float sm[];
  float* U = sm;
  float* Hs = sm + G::UOFF;
  const int tid = threadIdx.x;
  const int b = blockIdx.z;
  const int bx = blockIdx.x * TW, bly = blockIdx.y * TH;
  const int gy0 = p.dst.y0 + bly;
  for (int i = tid; i < UH * UW0; i += G::NT) {
    const int r = i / UW0, c = i % UW0;
    U[r * UW + c] = read_B(p.src, b, bx - HR + c, gy0 - HR + r);
  }
  __syncthreads();

  const int xb = tid & 31, run = (tid >> 5) & 3, half = tid >> 7;
  const int ox0 = half * NOA;  // first ox index of this half (warp-uniform)
  float num[8], den[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { num[j] = 0.0f; den[j] = 0.0f; }
  const float nc = -p.coef;

#pragma unroll 1
  for (int oy = -S; oy <= S; ++oy) {
    // ---------------- phase A
    for (int item = tid; item < HROWS * (TW / 4); item += G::NT) {
      const int hr = item / (TW / 4);
      const int x = 4 * (item % (TW / 4));
      const float* urow = U + (hr - P + HR) * UW + (x + HR - P);
      const float* qrow = U + (hr - P + oy + HR) * UW + (x + HR - P - S);
      float up[4 + 2 * P], uq[4 + 2 * P + 2 * S];
#pragma unroll
      for (int c = 0; c < 4 + 2 * P; ++c) up[c] = urow[c];
#pragma unroll
      for (int c = 0; c < 4 + 2 * P + 2 * S; ++c) uq[c] = qrow[c];
#pragma unroll
      for (int oxi = 0; oxi < NO; ++oxi) {
        float df[4 + 2 * P];
#pragma unroll
        for (int c = 0; c < 4 + 2 * P; ++c) df[c] = __fsub_rn(up[c], uq[c + oxi]);
        float h[4];
        float a = __fmul_rn(df[0], df[0]);
#pragma unroll
        for (int t = 1; t < PW; ++t) a = __fmaf_rn(df[t], df[t], a);
        h[0] = a;
#pragma unroll
        for (int j = 1; j < 4; ++j) {
          a = __fmaf_rn(df[j + 2 * P], df[j + 2 * P], a);
          a = __fmaf_rn(-df[j - 1], df[j - 1], a);
          h[j] = a;
        }
        *reinterpret_cast<float4*>(Hs + (oxi * HROWS + hr) * TW + x) = make_float4(h[0], h[1], h[2], h[3]);
      }
    }
    __syncthreads();
    // ---------------- phase B
#pragma unroll
    for (int o = 0; o < NOA; ++o) {
      const int oxi = ox0 + o;
      if (oxi < NO) {
        const float* hc = Hs + (oxi * HROWS + 8 * run) * TW + xb;
        float hv[8 + 2 * P];
#pragma unroll
        for (int k = 0; k < 8 + 2 * P; ++k) hv[k] = hc[k * TW];
        const float* qc = U + (8 * run + oy + HR) * UW + (xb + oxi - S + HR);
        float d = hv[0];
#pragma unroll
        for (int t = 1; t < PW; ++t) d = __fadd_rn(d, hv[t]);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j > 0) d = __fadd_rn(__fadd_rn(d, hv[j + 2 * P]), -hv[j - 1]);
          const float w = ex2_approx(__fmul_rn(fmaxf(d, 0.0f), nc));  // sliding sums can round below 0
          num[j] = __fmaf_rn(w, qc[j * UW], num[j]);
          den[j] = __fadd_rn(den[j], w);
        }
      }
    }
    __syncthreads();
  }
  // ---------------- combine the two ox halves (fixed order) and store
  float* red = Hs;  // [half][num|den][TH][TW]
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    red[((half * 2 + 0) * TH + 8 * run + j) * TW + xb] = num[j];
    red[((half * 2 + 1) * TH + 8 * run + j) * TW + xb] = den[j];
  }
  __syncthreads();
  for (int i = tid; i < TH * TW; i += G::NT) {
    const int y = i / TW, x = i % TW;
    const float n = __fadd_rn(red[i], red[2 * TH * TW + i]);
    const float dd = __fadd_rn(red[TH * TW + i], red[3 * TH * TW + i]);
    const int gx = bx + x, ly = bly + y;
    if (gx < p.src.W && ly < p.dst.H) dst_row(p.dst, b, ly)[gx] = __fdiv_rn(n, dd);
  }
}

template <int P, int S>
static cudaError_t launch_r8(const NlmParams& p, int batch, cudaStream_t s) {
  using G = R8Geom<P, S>;
  static_assert(G::smem_bytes <= 227 * 1024, "shared memory");
  auto kern = nlm_box_r8<P, S>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grd((p.src.W + G::TW - 1) / G::TW, (p.dst.H + G::TH - 1) / G::TH, batch);
  kern<<<grd, G::NT, G::smem_bytes, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

bool nlm_r8_supported(int P, int S) {
  return (P == 2 && S == 5) || (P == 1 && S == 3) || (P == 2 && S == 3) || (P == 1 && S == 5) ||
         (P == 3 && S == 7);
}

cudaError_t launch_nlm_r8(const NlmCall& c, cudaStream_t s) {
  NlmParams p = make_nlm_params(c);
  if (c.P == 2 && c.S == 5) return launch_r8<2, 5>(p, c.batch, s);
  if (c.P == 1 && c.S == 3) return launch_r8<1, 3>(p, c.batch, s);
  if (c.P == 2 && c.S == 3) return launch_r8<2, 3>(p, c.batch, s);
  if (c.P == 1 && c.S == 5) return launch_r8<1, 5>(p, c.batch, s);
  if (c.P == 3 && c.S == 7) return launch_r8<3, 7>(p, c.batch, s);
  return cudaErrorInvalidValue;
}

}  // namespace icl
