// nlm_r16.cu -- NLM variant "boxsum_r16": boxsum_r8 with wider phase-A
// segments and taller phase-B runs (less shared-memory traffic, which bounds
// boxsum_r8 at ~78% of the 128 B/clk/SM shared-memory bandwidth).  (NLM is
// not in PAPER.md; definition DESIGN.md R11-R14.)
//
// Per search row oy:
//   phase A  (thread = 8-column row segment, all 2S+1 ox) horizontal patch
//            sums H_o, sliding along the 8 columns;
//   phase B  (thread = column x, 16 consecutive rows, one quarter of the ox
//            range) vertical sums sliding over the 16 rows, then
//            w = 2^(-d*coef), num += w u(q), den += w.
// Shared-memory words per pair: phase A 0.39 load + 1.1 store, phase B 1.25 H
// + 1 u(q) = 3.8 (boxsum_r8: 4.2).  The 4 ox quarters are added at the end in
// a fixed order.
#include "nlm_common.cuh"

namespace icl {

template <int P, int S>
struct R16Geom {
  static constexpr int TW = 32, TH = 32, NT = 256;
  static constexpr int HR = P + S;
  static constexpr int UW0 = TW + 2 * HR;
  static constexpr int UW = ((UW0 + 30) / 32) * 32 + 1;  // == 1 (mod 32)
  static constexpr int UH = TH + 2 * HR;
  static constexpr int HROWS = TH + 2 * P;
  static constexpr int NO = 2 * S + 1;
  static constexpr int NOG = (NO + 3) / 4;  // ox per quarter (the last quarter may have fewer)
  static constexpr int UOFF = ((UH * UW + 3) / 4) * 4;
  static constexpr int HSZ = NO * HROWS * TW;
  static constexpr int RED = 8 * TH * TW;
  static constexpr size_t smem_bytes = (size_t)(UOFF + (HSZ > RED ? HSZ : RED)) * sizeof(float);
};

template <int P, int S>
__global__ void __launch_bounds__(256, 3) nlm_box_r16(NlmParams p) {
  using G = R16Geom<P, S>;
  constexpr int TW = G::TW, TH = G::TH, HR = G::HR, UW = G::UW, UW0 = G::UW0, UH = G::UH;
  constexpr int HROWS = G::HROWS, NO = G::NO, NOG = G::NOG, PW = 2 * P + 1;
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

  const int xb = tid & 31, run = (tid >> 5) & 1, grp = tid >> 6;
  const int ox0 = grp * NOG;  // first ox index of this quarter (warp-uniform)
  float num[16], den[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) { num[j] = 0.0f; den[j] = 0.0f; }
  const float nc = -p.coef;

#pragma unroll 1
  for (int oy = -S; oy <= S; ++oy) {
    // ---------------- phase A
    for (int item = tid; item < HROWS * (TW / 8); item += G::NT) {
      const int hr = item / (TW / 8);
      const int x = 8 * (item % (TW / 8));
      const float* urow = U + (hr - P + HR) * UW + (x + HR - P);
      const float* qrow = U + (hr - P + oy + HR) * UW + (x + HR - P - S);
      float up[8 + 2 * P], uq[8 + 2 * P + 2 * S];
#pragma unroll
      for (int c = 0; c < 8 + 2 * P; ++c) up[c] = urow[c];
#pragma unroll
      for (int c = 0; c < 8 + 2 * P + 2 * S; ++c) uq[c] = qrow[c];
#pragma unroll
      for (int oxi = 0; oxi < NO; ++oxi) {
        float df[8 + 2 * P];
#pragma unroll
        for (int c = 0; c < 8 + 2 * P; ++c) df[c] = __fsub_rn(up[c], uq[c + oxi]);
        float h[8];
        float a = __fmul_rn(df[0], df[0]);
#pragma unroll
        for (int t = 1; t < PW; ++t) a = __fmaf_rn(df[t], df[t], a);
        h[0] = a;
#pragma unroll
        for (int j = 1; j < 8; ++j) {
          a = __fmaf_rn(df[j + 2 * P], df[j + 2 * P], a);
          a = __fmaf_rn(-df[j - 1], df[j - 1], a);
          h[j] = a;
        }
        float* hd = Hs + (oxi * HROWS + hr) * TW + x;
        *reinterpret_cast<float4*>(hd) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(hd + 4) = make_float4(h[4], h[5], h[6], h[7]);
      }
    }
    __syncthreads();
    // ---------------- phase B
#pragma unroll
    for (int o = 0; o < NOG; ++o) {
      const int oxi = ox0 + o;
      if (oxi < NO) {
        const float* hc = Hs + (oxi * HROWS + 16 * run) * TW + xb;
        float hv[16 + 2 * P];
#pragma unroll
        for (int k = 0; k < 16 + 2 * P; ++k) hv[k] = hc[k * TW];
        const float* qc = U + (16 * run + oy + HR) * UW + (xb + oxi - S + HR);
        float d = hv[0];
#pragma unroll
        for (int t = 1; t < PW; ++t) d = __fadd_rn(d, hv[t]);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (j > 0) d = __fadd_rn(__fadd_rn(d, hv[j + 2 * P]), -hv[j - 1]);
          const float w = ex2_approx(__fmul_rn(fmaxf(d, 0.0f), nc));  // sliding sums can round below 0
          num[j] = __fmaf_rn(w, qc[j * UW], num[j]);
          den[j] = __fadd_rn(den[j], w);
        }
      }
    }
    __syncthreads();
  }
  // ---------------- combine the four ox quarters (fixed order) and store
  float* red = Hs;  // [quarter][num|den][TH][TW]
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    red[((grp * 2 + 0) * TH + 16 * run + j) * TW + xb] = num[j];
    red[((grp * 2 + 1) * TH + 16 * run + j) * TW + xb] = den[j];
  }
  __syncthreads();
  for (int i = tid; i < TH * TW; i += G::NT) {
    const int y = i / TW, x = i % TW;
    float n = red[i], dd = red[TH * TW + i];
#pragma unroll
    for (int g = 1; g < 4; ++g) {
      n = __fadd_rn(n, red[(2 * g) * TH * TW + i]);
      dd = __fadd_rn(dd, red[(2 * g + 1) * TH * TW + i]);
    }
    const int gx = bx + x, ly = bly + y;
    if (gx < p.src.W && ly < p.dst.H) dst_row(p.dst, b, ly)[gx] = __fdiv_rn(n, dd);
  }
}

template <int P, int S>
static cudaError_t launch_r16(const NlmParams& p, int batch, cudaStream_t s) {
  using G = R16Geom<P, S>;
  static_assert(G::smem_bytes <= 227 * 1024, "shared memory");
  auto kern = nlm_box_r16<P, S>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grd((p.src.W + G::TW - 1) / G::TW, (p.dst.H + G::TH - 1) / G::TH, batch);
  kern<<<grd, G::NT, G::smem_bytes, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

bool nlm_r16_supported(int P, int S) {
  return (P == 2 && S == 5) || (P == 1 && S == 3) || (P == 2 && S == 3) || (P == 1 && S == 5) ||
         (P == 3 && S == 7);
}

cudaError_t launch_nlm_r16(const NlmCall& c, cudaStream_t s) {
  NlmParams p = make_nlm_params(c);
  if (c.P == 2 && c.S == 5) return launch_r16<2, 5>(p, c.batch, s);
  if (c.P == 1 && c.S == 3) return launch_r16<1, 3>(p, c.batch, s);
  if (c.P == 2 && c.S == 3) return launch_r16<2, 3>(p, c.batch, s);
  if (c.P == 1 && c.S == 5) return launch_r16<1, 5>(p, c.batch, s);
  if (c.P == 3 && c.S == 7) return launch_r16<3, 7>(p, c.batch, s);
  return cudaErrorInvalidValue;
}

}  // namespace icl
