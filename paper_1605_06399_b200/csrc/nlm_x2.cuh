// nlm_x2.cuh -- NLM variant "boxsum_x2": the boxsum_r8 structure (offset-major
// separable patch sums through shared memory) run on TWO output tiles per CTA
// at once, every shared-memory word a float2 (tile A, tile B).  (NLM is not in
// PAPER.md; definition DESIGN.md R11-R14.)
//
// Why pairs of tiles: boxsum_r8 is co-limited by instruction issue (~17 lane-
// instructions per (pixel, offset) pair) and by shared-memory words (~4.2 per
// pair).  With the two tiles packed in the two lanes of a float2, every FP32
// operation of the box sums, the weight and the accumulation is one packed
// FADD2 / FMUL2 / FFMA2 for two pairs, and every shared-memory access is an
// LDS.64 / LDS.128 (no lane shuffles: the two tiles never mix).  Per pair:
// ~8 instructions, ~4.0 shared-memory words.
//
// Tile 32 x 28 (H rows = 28 + 2P = 32 for P = 2: one phase-A item per thread;
// phase B: 4 runs of 7 rows x 32 columns x 2 ox halves = 256 threads).
// Per search row oy:
//   phase A  thread = (H row hr, 4-column segment), all 2S+1 ox: horizontal
//            patch sums H_o(x..x+3, hr) with a sliding sum (+new^2 - old^2);
//   phase B  thread = (column x, 7-row run, ox half): vertical sliding sums,
//            w = 2^(-d*coef), num += w u(q), den += w.
// The two ox halves are added at the end in a fixed order.  Same per-element
// operations as boxsum_r8 except the run length (7 rows, restart of the
// vertical sliding sum), so results agree with it to rounding.
#pragma once
#include "nlm_common.cuh"

namespace icl {

__device__ __forceinline__ float2 f2_add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 f2_sub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

template <int P, int S>
struct X2Geom {
  static constexpr int TW = 32, TH = 28, NT = 256;
  static constexpr int HR = P + S;
  static constexpr int HROWS = TH + 2 * P;
  static constexpr int NO = 2 * S + 1;
  static constexpr int NOA = (NO + 1) / 2;
  static constexpr int UH = TH + 2 * HR;
  static constexpr int UW0 = TW + 2 * HR;                        // float2 columns
  static constexpr int UW = UW0 + ((UW0 % 4 == 2) ? 0 : (UW0 % 4 == 0 ? 2 : (UW0 % 4 == 1 ? 1 : 3)));  // == 2 (mod 4)
  static constexpr int HS = TW + 2;                              // H row stride (float2), == 2 (mod 4)
  static constexpr int HSZ = NO * HROWS * HS;
  static constexpr int RUN = TH / 4;
  static constexpr int RED = 4 * TH * TW;
  static constexpr size_t smem_bytes = (size_t)(UH * UW + (HSZ > RED ? HSZ : RED)) * sizeof(float2);
  static_assert(UW % 4 == 2 && HS % 4 == 2, "conflict-free strides");
  static_assert(TH % 4 == 0, "4 runs");
};

template <int P, int S>
__global__ void __launch_bounds__(256, 2) nlm_box_x2(NlmParams p, int ntx, int nty, int ntiles, int nhalf) {
  using G = X2Geom<P, S>;
  constexpr int TW = G::TW, TH = G::TH, HR = G::HR, UW = G::UW, UW0 = G::UW0, UH = G::UH, HS = G::HS;
  constexpr int HROWS = G::HROWS, NO = G::NO, NOA = G::NOA, RUN = G::RUN, PW = 2 * P + 1;
  constexpr int NQ = 4 + 2 * HR;  // uq window (float2), even
  extern __shared__ __align__(16) float2 sm2[];
  float2* U = sm2;
  float2* Hs = sm2 + UH * UW;
  const int tid = threadIdx.x;

  // the tile pair: A = blockIdx.x, B = blockIdx.x + nhalf (B == A when absent)
  const int per_img = ntx * nty;
  const int tA = blockIdx.x;
  const int tB = tA + nhalf < ntiles ? tA + nhalf : tA;
  const int bA = tA / per_img, bB = tB / per_img;
  const int rA = tA - bA * per_img, rB = tB - bB * per_img;
  const int yA = (rA / ntx) * TH, yB = (rB / ntx) * TH;  // local output rows
  const int xA = (rA % ntx) * TW, xB = (rB % ntx) * TW;
  const int gA = p.dst.y0 + yA, gB = p.dst.y0 + yB;

  for (int i = tid; i < UH * UW0; i += G::NT) {
    const int r = i / UW0, c = i - r * UW0;
    U[r * UW + c] = make_float2(read_B(p.src, bA, xA - HR + c, gA - HR + r), read_B(p.src, bB, xB - HR + c, gB - HR + r));
  }
  __syncthreads();

  const int xb = tid & 31, run = (tid >> 5) & 3, half = tid >> 7;
  const int ox0 = half * NOA;
  float2 num[RUN], den[RUN];
#pragma unroll
  for (int j = 0; j < RUN; ++j) { num[j] = make_float2(0.0f, 0.0f); den[j] = make_float2(0.0f, 0.0f); }
  const float2 nc = make_float2(-p.coef, -p.coef);

  // phase-A rows: consecutive threads -> consecutive H rows.  With exactly one
  // item per thread (P = 2) the oy-invariant centre row u(x-P..x+3+P, hr-P)
  // stays in registers for the whole search.
  constexpr bool ONE_ITEM = HROWS * (TW / 4) == G::NT;
  float2 up1[4 + 2 * P];
  if (ONE_ITEM) {
    const int hr = tid % HROWS, x = 4 * (tid / HROWS);
    const float2* urow = U + (hr - P + HR) * UW + (x + HR - P);
#pragma unroll
    for (int c = 0; c < 4 + 2 * P; ++c) up1[c] = urow[c];
  }

#pragma unroll 1
  for (int oy = -S; oy <= S; ++oy) {
    // ---------------- phase A: H rows hr, 4-column segments
    for (int item = tid; item < HROWS * (TW / 4); item += G::NT) {
      const int hr = item % HROWS, x = 4 * (item / HROWS);
      const float2* qrow = U + (hr - P + oy + HR) * UW + x;  // column x - P - S + HR == x
      float2 up[4 + 2 * P], uq[NQ];
      if (ONE_ITEM) {
#pragma unroll
        for (int c = 0; c < 4 + 2 * P; ++c) up[c] = up1[c];
      } else {
        const float2* urow = U + (hr - P + HR) * UW + (x + HR - P);
#pragma unroll
        for (int c = 0; c < 4 + 2 * P; ++c) up[c] = urow[c];
      }
#pragma unroll
      for (int q = 0; q < NQ / 2; ++q) {
        const float4 w = reinterpret_cast<const float4*>(qrow)[q];
        uq[2 * q] = make_float2(w.x, w.y);
        uq[2 * q + 1] = make_float2(w.z, w.w);
      }
#pragma unroll
      for (int oxi = 0; oxi < NO; ++oxi) {
        float2 df[4 + 2 * P];
#pragma unroll
        for (int c = 0; c < 4 + 2 * P; ++c) df[c] = f2_sub(up[c], uq[c + oxi]);
        float2 h[4];
        float2 a = f2_mul(df[0], df[0]);
#pragma unroll
        for (int t = 1; t < PW; ++t) a = f2_fma(df[t], df[t], a);
        h[0] = a;
#pragma unroll
        for (int j = 1; j < 4; ++j) {
          a = f2_fma(df[j + 2 * P], df[j + 2 * P], a);
          a = f2_fma(make_float2(-df[j - 1].x, -df[j - 1].y), df[j - 1], a);
          h[j] = a;
        }
        float4* dst = reinterpret_cast<float4*>(Hs + (oxi * HROWS + hr) * HS + x);
        dst[0] = make_float4(h[0].x, h[0].y, h[1].x, h[1].y);
        dst[1] = make_float4(h[2].x, h[2].y, h[3].x, h[3].y);
      }
    }
    __syncthreads();
    // ---------------- phase B: column xb, RUN rows, one half of the ox range
#pragma unroll
    for (int o = 0; o < NOA; ++o) {
      const int oxi = ox0 + o;
      if (oxi < NO) {
        const float2* hc = Hs + (oxi * HROWS + RUN * run) * HS + xb;
        float2 hv[RUN + 2 * P];
#pragma unroll
        for (int k = 0; k < RUN + 2 * P; ++k) hv[k] = hc[k * HS];
        const float2* qc = U + (RUN * run + oy + HR) * UW + (xb + oxi - S + HR);
        float2 d = hv[0];
#pragma unroll
        for (int t = 1; t < PW; ++t) d = f2_add(d, hv[t]);
#pragma unroll
        for (int j = 0; j < RUN; ++j) {
          if (j > 0) d = f2_add(f2_add(d, hv[j + 2 * P]), make_float2(-hv[j - 1].x, -hv[j - 1].y));
          // sliding sums can round below 0; a negative d with a tiny h would give w = inf
          const float2 t = f2_mul(make_float2(fmaxf(d.x, 0.0f), fmaxf(d.y, 0.0f)), nc);
          const float2 w = make_float2(ex2_approx(t.x), ex2_approx(t.y));
          num[j] = f2_fma(w, qc[j * UW], num[j]);
          den[j] = f2_add(den[j], w);
        }
      }
    }
    __syncthreads();
  }
  // ---------------- combine the two ox halves (fixed order) and store both tiles
  float2* red = Hs;  // [half][num|den][TH][TW]
#pragma unroll
  for (int j = 0; j < RUN; ++j) {
    red[((half * 2 + 0) * TH + RUN * run + j) * TW + xb] = num[j];
    red[((half * 2 + 1) * TH + RUN * run + j) * TW + xb] = den[j];
  }
  __syncthreads();
  for (int i = tid; i < TH * TW; i += G::NT) {
    const int y = i / TW, x = i % TW;
    const float2 n = f2_add(red[i], red[2 * TH * TW + i]);
    const float2 dd = f2_add(red[TH * TW + i], red[3 * TH * TW + i]);
    if (xA + x < p.src.W && yA + y < p.dst.H) dst_row(p.dst, bA, yA + y)[xA + x] = __fdiv_rn(n.x, dd.x);
    if (tB != tA && xB + x < p.src.W && yB + y < p.dst.H) dst_row(p.dst, bB, yB + y)[xB + x] = __fdiv_rn(n.y, dd.y);
  }
}

template <int P, int S>
inline cudaError_t launch_x2(const NlmParams& p, int batch, cudaStream_t s) {
  using G = X2Geom<P, S>;
  static_assert(G::smem_bytes <= 113 * 1024, "two CTAs per SM");
  auto kern = nlm_box_x2<P, S>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::smem_bytes);
  if (e != cudaSuccess) return e;
  const int ntx = (p.src.W + G::TW - 1) / G::TW, nty = (p.dst.H + G::TH - 1) / G::TH;
  const int ntiles = ntx * nty * batch;
  const int nhalf = (ntiles + 1) / 2;
  kern<<<nhalf, G::NT, G::smem_bytes, s>>>(p, ntx, nty, ntiles, nhalf);
  count_launch();
  return cudaGetLastError();
}

}  // namespace icl
