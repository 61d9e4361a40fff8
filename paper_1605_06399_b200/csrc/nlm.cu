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
static NlmParams make_params(const NlmCall& c) {
  NlmParams p;
  p.src = c.src;
  p.dst = c.dst;
  p.P = c.P;
  p.S = c.S;
  p.coef = c.coef;
  return p;
}

cudaError_t launch_nlm_naive(const NlmCall& c, cudaStream_t s) {
  NlmParams p = make_params(c);
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
  NlmParams p = make_params(c);
  if (c.P == 2 && c.S == 5) return launch_tiled_PS<2, 5>(p, c.batch, s);
  if (c.P == 1 && c.S == 3) return launch_tiled_PS<1, 3>(p, c.batch, s);
  if (c.P == 3 && c.S == 7) return launch_tiled_PS<3, 7>(p, c.batch, s);
  if (c.P == 2 && c.S == 3) return launch_tiled_PS<2, 3>(p, c.batch, s);
  if (c.P == 1 && c.S == 5) return launch_tiled_PS<1, 5>(p, c.batch, s);
  return cudaErrorInvalidValue;
}

cudaError_t launch_nlm_boxsum(const NlmCall& c, int variant, cudaStream_t s) {
  (void)c;
  (void)variant;
  (void)s;
  return cudaErrorNotSupported;
}

}  // namespace icl
