// nlm_w.cuh -- NLM variant "boxsum_w": the offset-major separable patch sums of
// boxsum_x2 (two output tiles per CTA packed in float2 lanes), restructured to
// move fewer shared-memory words per (pixel, offset) pair -- the resource that
// bounds boxsum_x2 (ncu: 81% of the smem wavefront peak at 4.57 words / pair).
// (NLM is not in PAPER.md; definition DESIGN.md R11-R14.)
//
// Per search row oy (CTA = 128 threads, tile pair of 16 x 28 outputs, 2 CTAs/SM
// at up to 255 registers per thread):
//   phase A  thread = (H row hr, 4-column segment), all 2S+1 ox: horizontal
//            patch sums H_o(x..x+3, hr) with a sliding sum (+new^2 - old^2) of
//            the scaled differences; the oy-invariant centre row stays in
//            registers; H goes to shared memory (1.14 words / pair).
//   phase B  thread = (column xb, run of 14 rows, group of <= 3 ox; one warp per
//            ox group): per ox the vertical sum slides down the 14 + 2P H rows
//            held in a register ring (each H word read ONCE: 1.29 words / pair
//            instead of 1.57), w = 2^(-d*coef), num += w u(q), den += w.  u(q) is
//            a register WINDOW per ox: column x+ox, rows y+oy for the run's 14
//            rows; from one oy to the next it shifts by one row, so a step loads
//            one new word per ox instead of 14 (0.07 words / pair instead of 1).
//   The four ox groups' partial sums are added at the end in a fixed order.
// ~2.9 shared-memory words per pair (boxsum_x2: 4.57).  Results agree with the
// other box-sum variants to rounding (runs of 14 rows instead of 7 restart the
// sliding vertical sum at different rows; ox groups of 3 instead of halves).
#pragma once
#include "nlm_common.cuh"

namespace icl {

template <int P, int S>
struct WGeom {
  static constexpr int TW = 16, TH = 28, NT = 128;
  static constexpr int HR = P + S;
  static constexpr int HROWS = TH + 2 * P;
  static constexpr int NO = 2 * S + 1;
  static constexpr int NG = 4;                      // ox groups = warps
  static constexpr int G = (NO + NG - 1) / NG;      // ox per group
  static constexpr int RUN = TH / 2;                // rows per phase-B thread
  static constexpr int UH = TH + 2 * HR;
  static constexpr int UW0 = TW + 2 * HR;           // float2 columns
  static constexpr int UW = UW0 + ((UW0 % 4 == 2) ? 0 : (UW0 % 4 == 0 ? 2 : (UW0 % 4 == 1 ? 1 : 3)));  // == 2 (mod 4)
  static constexpr int HS = TW + 2;                 // H row stride (float2), == 2 (mod 4)
  static constexpr int HSZ = NO * HROWS * HS;
  static constexpr int RED = 2 * NG * TH * TW;      // [group][num|den][TH][TW]
  static constexpr size_t smem_bytes = (size_t)(UH * UW + (HSZ > RED ? HSZ : RED)) * sizeof(float2);
  static_assert(UW % 4 == 2 && HS % 4 == 2, "conflict-free strides");
};

template <int P, int S, int UOY>
__global__ void __launch_bounds__(128, 2) nlm_box_w(NlmParams p, int ntx, int nty, int ntiles, int nhalf) {
  using G_ = WGeom<P, S>;
  constexpr int TW = G_::TW, TH = G_::TH, HR = G_::HR, UW = G_::UW, UW0 = G_::UW0, UH = G_::UH, HS = G_::HS;
  constexpr int HROWS = G_::HROWS, NO = G_::NO, G = G_::G, RUN = G_::RUN, PW = 2 * P + 1, NT = G_::NT;
  constexpr int NQ = 4 + 2 * HR;  // phase-A other-row window (float2), even
  extern __shared__ __align__(16) float2 smw[];
  float2* U = smw;
  float2* Hs = smw + UH * UW;
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

  for (int i = tid; i < UH * UW0; i += NT) {
    const int r = i / UW0, c = i - r * UW0;
    U[r * UW + c] = make_float2(read_B(p.src, bA, xA - HR + c, gA - HR + r), read_B(p.src, bB, xB - HR + c, gB - HR + r));
  }
  __syncthreads();

  // phase-B role: column xb, run, ox group = warp
  const int xb = tid & 15, run = (tid >> 4) & 1, og = tid >> 5;
  const int ox0 = og * G;  // first oxi of the group
  float2 num[RUN], den[RUN];
#pragma unroll
  for (int j = 0; j < RUN; ++j) { num[j] = make_float2(0.0f, 0.0f); den[j] = make_float2(0.0f, 0.0f); }
  const float2 nc = make_float2(-p.coef, -p.coef);

  // u(q) windows: win[o][j] = u(x + ox, y + oy + j) for the run's rows, at the current oy
  float2 win[G][RUN];
#pragma unroll
  for (int o = 0; o < G; ++o) {
    const int oxi = ox0 + o < NO ? ox0 + o : NO - 1;  // (a padded slot of the last group: never used)
#pragma unroll
    for (int j = 0; j < RUN; ++j) win[o][j] = U[(RUN * run + j - S + HR) * UW + (xb + oxi - S + HR)];
  }

  // phase-A role: consecutive threads -> consecutive H rows; with exactly one item per thread
  // the oy-invariant centre row u(x-P..x+3+P, hr-P) stays in registers for the whole search
  constexpr bool ONE_ITEM = HROWS * (TW / 4) == NT;
  float2 up1[4 + 2 * P];
  if (ONE_ITEM) {
    const int hr = tid % HROWS, x = 4 * (tid / HROWS);
    const float2* urow = U + (hr - P + HR) * UW + (x + HR - P);
#pragma unroll
    for (int c = 0; c < 4 + 2 * P; ++c) up1[c] = urow[c];
  }

  // UOY: the search-row loop unrolled (2, or 2S+1 = fully: the window shifts become renames)
#pragma unroll UOY
  for (int oy = -S; oy <= S; ++oy) {
    // ---------------- phase A: H rows hr, 4-column segments
    for (int item = tid; item < HROWS * (TW / 4); item += NT) {
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
        for (int c = 0; c < 4 + 2 * P; ++c) df[c] = __fadd2_rn(up[c], make_float2(-uq[c + oxi].x, -uq[c + oxi].y));
        float2 h[4];
        float2 a = __fmul2_rn(df[0], df[0]);
#pragma unroll
        for (int t = 1; t < PW; ++t) a = __ffma2_rn(df[t], df[t], a);
        h[0] = a;
#pragma unroll
        for (int j = 1; j < 4; ++j) {
          a = __ffma2_rn(df[j + 2 * P], df[j + 2 * P], a);
          a = __ffma2_rn(make_float2(-df[j - 1].x, -df[j - 1].y), df[j - 1], a);
          h[j] = a;
        }
        float4* dst = reinterpret_cast<float4*>(Hs + (oxi * HROWS + hr) * HS + x);
        dst[0] = make_float4(h[0].x, h[0].y, h[1].x, h[1].y);
        dst[1] = make_float4(h[2].x, h[2].y, h[3].x, h[3].y);
      }
    }
    __syncthreads();
    // ---------------- phase B: column xb, RUN rows, ox group og
#pragma unroll
    for (int o = 0; o < G; ++o) {
      const int oxi = ox0 + o;
      if (oxi < NO) {
        const float2* hc = Hs + (oxi * HROWS + RUN * run) * HS + xb;
        // ring of the last PW H rows (static indices: the run is fully unrolled)
        float2 ring[PW];
        float2 d = hc[0];
        ring[0] = d;
#pragma unroll
        for (int t = 1; t < PW; ++t) {
          ring[t] = hc[t * HS];
          d = __fadd2_rn(d, ring[t]);
        }
#pragma unroll
        for (int j = 0; j < RUN; ++j) {
          if (j > 0) {
            const float2 hn = hc[(j + 2 * P) * HS];
            d = __fadd2_rn(__fadd2_rn(d, hn), make_float2(-ring[(j - 1) % PW].x, -ring[(j - 1) % PW].y));
            ring[(j - 1) % PW] = hn;
          }
          // sliding sums can round below 0; a negative d with a tiny h would give w = inf
          const float2 t = __fmul2_rn(make_float2(fmaxf(d.x, 0.0f), fmaxf(d.y, 0.0f)), nc);
          const float2 w = make_float2(ex2_approx(t.x), ex2_approx(t.y));
          num[j] = __ffma2_rn(w, win[o][j], num[j]);
          den[j] = __fadd2_rn(den[j], w);
        }
      }
    }
    // shift the u(q) windows to oy + 1: one new row per ox
    if (oy < S) {
#pragma unroll
      for (int o = 0; o < G; ++o) {
        const int oxi = ox0 + o < NO ? ox0 + o : NO - 1;
#pragma unroll
        for (int j = 0; j + 1 < RUN; ++j) win[o][j] = win[o][j + 1];
        win[o][RUN - 1] = U[(RUN * run + RUN - 1 + oy + 1 + HR) * UW + (xb + oxi - S + HR)];
      }
    }
    __syncthreads();
  }
  // ---------------- combine the ox groups (fixed order) and store both tiles
  float2* red = Hs;  // [group][num|den][TH][TW]
#pragma unroll
  for (int j = 0; j < RUN; ++j) {
    red[((og * 2 + 0) * TH + RUN * run + j) * TW + xb] = num[j];
    red[((og * 2 + 1) * TH + RUN * run + j) * TW + xb] = den[j];
  }
  __syncthreads();
  for (int i = tid; i < TH * TW; i += NT) {
    const int y = i / TW, x = i % TW;
    float2 n = red[i], dd = red[TH * TW + i];
#pragma unroll
    for (int g = 1; g < G_::NG; ++g) {
      n = __fadd2_rn(n, red[(2 * g) * TH * TW + i]);
      dd = __fadd2_rn(dd, red[(2 * g + 1) * TH * TW + i]);
    }
    if (xA + x < p.src.W && yA + y < p.dst.H) dst_row(p.dst, bA, yA + y)[xA + x] = __fdiv_rn(n.x, dd.x);
    if (tB != tA && xB + x < p.src.W && yB + y < p.dst.H) dst_row(p.dst, bB, yB + y)[xB + x] = __fdiv_rn(n.y, dd.y);
  }
}

template <int P, int S, int UOY = 1>
inline cudaError_t launch_w(const NlmParams& p, int batch, cudaStream_t s) {
  using G = WGeom<P, S>;
  static_assert(G::smem_bytes <= 113 * 1024, "two CTAs per SM");
  auto kern = nlm_box_w<P, S, UOY>;
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
