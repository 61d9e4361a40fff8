// nlm.cu -- non-local-means variants.  NLM is not in PAPER.md; it replaces
// the paper's non-separable convolution per BASELINE.json north_star.
// Definition: DESIGN.md R11-R14 (uniform patch mean, w = exp(-d2/h^2), the
// search window includes p, boundary applied to every final read).
//
// Direct variants evaluate, per output pixel, the same fp32 sequence:
//   for oy = -S..S, ox = -S..S:            (row-major offset order)
//     d  = fma-chain over ty, tx of diff*diff, diff = u(p+t) - u(q+t)   (from 0)
//     w  = ex2.approx(-(d * coef)),  coef = log2(e) / ((2P+1)^2 h^2)   (0 if h = inf)
//     num = fma(w, u(q), num);  den = den + w
//   out = num / den
#include "common.cuh"
#include "internal.h"
#include "nlm_common.cuh"

namespace icl {

// --------------------------------------------------------------------------
// Variant "naive_direct": one logical thread per pixel, every read from
// global memory through in_B.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) nlm_naive(NlmParams p) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int ly = blockIdx.y * blockDim.y + threadIdx.y;
  const int b = blockIdx.z;
  if (x >= p.src.W || ly >= p.dst.H) return;
  const int y = p.dst.y0 + ly;
  float num = 0.0f, den = 0.0f;
  for (int oy = -p.S; oy <= p.S; ++oy)
    for (int ox = -p.S; ox <= p.S; ++ox) {
      float d = 0.0f;
      for (int ty = -p.P; ty <= p.P; ++ty)
        for (int tx = -p.P; tx <= p.P; ++tx) {
          const float diff = __fsub_rn(read_B(p.src, b, x + tx, y + ty), read_B(p.src, b, x + ox + tx, y + oy + ty));
          d = __fmaf_rn(diff, diff, d);
        }
      const float w = ex2_approx(-__fmul_rn(d, p.coef));
      num = __fmaf_rn(w, read_B(p.src, b, x + ox, y + oy), num);
      den = __fadd_rn(den, w);
    }
  dst_row(p.dst, b, ly)[x] = __fdiv_rn(num, den);
}

// --------------------------------------------------------------------------
// Variant "tiled_direct<P,S>": the paper's local-memory transformation
// (Fig. 5): the CTA's bounding-box tile (TW+2(P+S)) x
// (TH+2(P+S)) is loaded once into shared memory with the boundary applied at
// load time; each thread keeps its own patch in registers and, per search
// row oy, loads the (2P+1) x (2S+2P+1) candidate window once and slides the
// patch across it for all 2S+1 ox (full unroll => static register indices).
// --------------------------------------------------------------------------
template <int P, int S, int TW, int TH>
__global__ void __launch_bounds__(TW* TH) nlm_tiled(NlmParams p) {
  constexpr int PW = 2 * P + 1;
  constexpr int HR = P + S;
  constexpr int SW = TW + 2 * HR;
  constexpr int SH = TH + 2 * HR;
  constexpr int WW = 2 * S + PW;  // candidate window width
  __shared__ float tile[SH][SW + 1];

  const int tx0 = threadIdx.x, ty0 = threadIdx.y;
  const int b = blockIdx.z;
  const int bx = blockIdx.x * TW, bly = blockIdx.y * TH;
  const int gy0 = p.dst.y0 + bly;
  for (int i = ty0 * TW + tx0; i < SH * SW; i += TW * TH) {
    const int r = i / SW, c = i % SW;
    tile[r][c] = read_B(p.src, b, bx - HR + c, gy0 - HR + r);
  }
  __syncthreads();
  const int x = bx + tx0, ly = bly + ty0;
  if (x >= p.src.W || ly >= p.dst.H) return;

  float pp[PW][PW];
#pragma unroll
  for (int ty = 0; ty < PW; ++ty)
#pragma unroll
    for (int tx = 0; tx < PW; ++tx) pp[ty][tx] = tile[ty0 + S + ty][tx0 + S + tx];

  float num = 0.0f, den = 0.0f;
#pragma unroll 1
  for (int oy = 0; oy < 2 * S + 1; ++oy) {
    float win[PW][WW];
#pragma unroll
    for (int ty = 0; ty < PW; ++ty)
#pragma unroll
      for (int c = 0; c < WW; ++c) win[ty][c] = tile[ty0 + oy + ty][tx0 + c];
#pragma unroll
    for (int ox = 0; ox < 2 * S + 1; ++ox) {
      float d = 0.0f;
#pragma unroll
      for (int ty = 0; ty < PW; ++ty)
#pragma unroll
        for (int tx = 0; tx < PW; ++tx) {
          const float diff = __fsub_rn(pp[ty][tx], win[ty][ox + tx]);
          d = __fmaf_rn(diff, diff, d);
        }
      const float w = ex2_approx(-__fmul_rn(d, p.coef));
      num = __fmaf_rn(w, win[P][ox + P], num);
      den = __fadd_rn(den, w);
    }
  }
  dst_row(p.dst, b, ly)[x] = __fdiv_rn(num, den);
}

// ----------------------------------------------------------------- launchers
cudaError_t launch_nlm_naive(const NlmCall& c, cudaStream_t s) {
  NlmParams p = make_nlm_params(c);
  dim3 blk(32, 8), grd((c.src.W + 31) / 32, (c.dst.H + 7) / 8, c.batch);
  nlm_naive<<<grd, blk, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

template <int P, int S>
static cudaError_t launch_tiled_PS(const NlmParams& p, int batch, cudaStream_t s) {
  constexpr int TW = 32, TH = 8;
  dim3 blk(TW, TH), grd((p.src.W + TW - 1) / TW, (p.dst.H + TH - 1) / TH, batch);
  nlm_tiled<P, S, TW, TH><<<grd, blk, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

bool nlm_tiled_supported(int P, int S) {
  return (P == 2 && S == 5) || (P == 1 && S == 3) || (P == 3 && S == 7) || (P == 2 && S == 3) ||
         (P == 1 && S == 5);
}

cudaError_t launch_nlm_tiled(const NlmCall& c, int tw, int th, cudaStream_t s) {
  (void)tw;
  (void)th;
  NlmParams p = make_nlm_params(c);
  if (c.P == 2 && c.S == 5) return launch_tiled_PS<2, 5>(p, c.batch, s);
  if (c.P == 1 && c.S == 3) return launch_tiled_PS<1, 3>(p, c.batch, s);
  if (c.P == 3 && c.S == 7) return launch_tiled_PS<3, 7>(p, c.batch, s);
  if (c.P == 2 && c.S == 3) return launch_tiled_PS<2, 3>(p, c.batch, s);
  if (c.P == 1 && c.S == 5) return launch_tiled_PS<1, 5>(p, c.batch, s);
  return cudaErrorInvalidValue;
}

// --------------------------------------------------------------------------
// Variant "boxsum<P,S>": offset-major NLM.  For a fixed offset o the patch
// distance is a (2P+1)^2 box sum of D_o(x) = (u(x) - u(x+o))^2, which is
// separable: d(p,o) = sum_ty H_o(p + (0,ty)),  H_o(x,y) = sum_tx D_o(x+tx, y).
// A CTA owns a 32x32 output tile; its bounding-box input tile (halo P+S,
// boundary applied at load) sits in shared memory.  For
// each search row oy:
//   phase A  every thread computes H_o for a 4-pixel row segment and ALL
//            2S+1 ox (the candidate row is loaded once and reused across ox)
//            into shared memory, rows -P .. 32+P of the tile;
//   phase B  every thread owns one column x and 4 consecutive rows, sums
//            2P+1 H rows per output (d), and accumulates w = 2^(-d*coef),
//            num += w u(q), den += w in registers.
// Arithmetic per (pixel, offset): 2 FSUB(+halo) + (2P+1) FFMA (H) + 2P FADD
// (d) + FMUL + MUFU.EX2 + FFMA + FADD -- versus (2P+1)^2 x 3 flops direct.
// d is re-associated w.r.t. the direct form (compared by tolerance).
// --------------------------------------------------------------------------
template <int P, int S>
struct BoxGeom {
  static constexpr int TW = 32, TH = 32, NT = 256;
  static constexpr int HR = P + S;
  static constexpr int UW0 = TW + 2 * HR;
  static constexpr int UW = ((UW0 + 30) / 32) * 32 + 1;  // row stride == 1 (mod 32): conflict-free phase A
  static constexpr int UH = TH + 2 * HR;
  static constexpr int HROWS = TH + 2 * P;
  static constexpr int NO = 2 * S + 1;
  static constexpr int UOFF = ((UH * UW + 3) / 4) * 4;  // Hs starts 16-byte aligned
  static constexpr size_t smem_bytes = (size_t)(UOFF + NO * HROWS * TW) * sizeof(float);
};

template <int P, int S>
__global__ void __launch_bounds__(256) nlm_boxsum(NlmParams p) {
  using G = BoxGeom<P, S>;
  constexpr int TW = G::TW, TH = G::TH, HR = G::HR, UW = G::UW, UH = G::UH, HROWS = G::HROWS, NO = G::NO;
  constexpr int PW = 2 * P + 1;
  extern __shared__ __align__(16) float sm[];
  float* U = sm;                 // [UH][UW]
  float* Hs = sm + G::UOFF;      // [NO][HROWS][TW]
  const int tid = threadIdx.x;
  const int b = blockIdx.z;
  const int bx = blockIdx.x * TW, bly = blockIdx.y * TH;
  const int gy0 = p.dst.y0 + bly;
  for (int i = tid; i < UH * (TW + 2 * HR); i += G::NT) {
    const int r = i / (TW + 2 * HR), c = i % (TW + 2 * HR);
    U[r * UW + c] = read_B(p.src, b, bx - HR + c, gy0 - HR + r);
  }
  __syncthreads();

  // phase-B ownership: column xb, rows 4*run .. 4*run+3
  const int xb = tid & 31, run = tid >> 5;
  float num[4] = {0.f, 0.f, 0.f, 0.f}, den[4] = {0.f, 0.f, 0.f, 0.f};

#pragma unroll 1
  for (int oy = -S; oy <= S; ++oy) {
    // ---------------- phase A: H_o rows for all ox
    for (int item = tid; item < HROWS * (TW / 4); item += G::NT) {
      const int yr = item / (TW / 4);   // H row index (tile row yr - P)
      const int x = 4 * (item % (TW / 4));
      const float* urow = U + (yr - P + HR) * UW + (x + HR - P);
      const float* qrow = U + (yr - P + oy + HR) * UW + (x + HR - P - S);
      float up[4 + 2 * P], uq[4 + 2 * P + 2 * S];
#pragma unroll
      for (int c = 0; c < 4 + 2 * P; ++c) up[c] = urow[c];
#pragma unroll
      for (int c = 0; c < 4 + 2 * P + 2 * S; ++c) uq[c] = qrow[c];
#pragma unroll
      for (int ox = 0; ox < NO; ++ox) {
        float df[4 + 2 * P];
#pragma unroll
        for (int c = 0; c < 4 + 2 * P; ++c) df[c] = __fsub_rn(up[c], uq[c + ox]);
        float h[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float a = 0.0f;
#pragma unroll
          for (int t = 0; t < PW; ++t) a = __fmaf_rn(df[j + t], df[j + t], a);
          h[j] = a;
        }
        *reinterpret_cast<float4*>(Hs + (ox * HROWS + yr) * TW + x) = make_float4(h[0], h[1], h[2], h[3]);
      }
    }
    __syncthreads();
    // ---------------- phase B: vertical sums, weights, accumulation
#pragma unroll
    for (int ox = 0; ox < NO; ++ox) {
      const float* hc = Hs + (ox * HROWS + 4 * run) * TW + xb;
      float hv[4 + 2 * P];
#pragma unroll
      for (int k = 0; k < 4 + 2 * P; ++k) hv[k] = hc[k * TW];
      const float* qc = U + (4 * run + oy + HR) * UW + (xb + ox - S + HR);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float d = hv[j];
#pragma unroll
        for (int t = 1; t < PW; ++t) d = __fadd_rn(d, hv[j + t]);
        const float w = ex2_approx(-__fmul_rn(fmaxf(d, 0.0f), p.coef));
        num[j] = __fmaf_rn(w, qc[j * UW], num[j]);
        den[j] = __fadd_rn(den[j], w);
      }
    }
    __syncthreads();
  }
  const int x = bx + xb;
  if (x < p.src.W) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int ly = bly + 4 * run + j;
      if (ly < p.dst.H) dst_row(p.dst, b, ly)[x] = __fdiv_rn(num[j], den[j]);
    }
  }
}

template <int P, int S>
static cudaError_t launch_box_PS(const NlmParams& p, int batch, cudaStream_t s) {
  using G = BoxGeom<P, S>;
  static_assert(G::TH == 4 * (G::NT / 32), "phase B covers the tile");
  const size_t smem = G::smem_bytes;
  auto kern = nlm_boxsum<P, S>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grd((p.src.W + G::TW - 1) / G::TW, (p.dst.H + G::TH - 1) / G::TH, batch);
  kern<<<grd, G::NT, smem, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

bool nlm_boxsum_supported(int P, int S) { return nlm_tiled_supported(P, S); }

cudaError_t launch_nlm_boxsum(const NlmCall& c, int variant, cudaStream_t s) {
  (void)variant;
  NlmParams p = make_nlm_params(c);
  if (c.P == 2 && c.S == 5) return launch_box_PS<2, 5>(p, c.batch, s);
  if (c.P == 1 && c.S == 3) return launch_box_PS<1, 3>(p, c.batch, s);
  if (c.P == 3 && c.S == 7) return launch_box_PS<3, 7>(p, c.batch, s);
  if (c.P == 2 && c.S == 3) return launch_box_PS<2, 3>(p, c.batch, s);
  if (c.P == 1 && c.S == 5) return launch_box_PS<1, 5>(p, c.batch, s);
  return cudaErrorInvalidValue;
}

}  // namespace icl
