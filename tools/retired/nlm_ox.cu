// nlm_ox.cu -- NLM variant "boxsum_oxwarp": offset-major separable patch
// sums with one warp per horizontal search offset.  (NLM is not in PAPER.md;
// definition DESIGN.md R11-R14.)
//
// A CTA owns a 32-column x TH-row output tile and runs 2S+1 warps; warp w
// owns search offset ox = w - S and lane x one output column, for ALL TH
// rows and ALL oy.  The bounding-box input tile (halo P+S, boundary applied
// at load -- the paper's local-memory staging) sits in
// shared memory.  For each search row oy:
//   phase A  (all threads) H_o(x, r) = sum_{tx=-P..P} (u(x+tx, r) - u(x+tx+ox, r+oy))^2
//            for every ox, for 4-column row segments; the candidate row is
//            loaded once per segment and reused by all 2S+1 ox; the 4
//            outputs of a segment use a sliding sum (+new^2 - old^2).
//            Written to a double-buffered H area in shared memory.
//   phase B  (warp ox, lane x) d(y) = sum_{ty=-P..P} H_o(x, y+ty) (direct),
//            w = 2^(-d*coef), num[y] += w*u(x+ox, y+oy), den[y] += w, with
//            num/den/u(q) in registers (the oy loop is unrolled so the u(q)
//            column window is indexed statically).
// One barrier per oy (double buffering); at the end the 2S+1 partial sums
// per pixel are added in ox order through shared memory.
// Shared-memory traffic ~2.8 words per (pixel, offset) versus 4.7 for
// boxsum_32x32; FP32 ~12 ops per pair versus 3(2P+1)^2+4 = 79 direct.
#include "nlm_common.cuh"

namespace icl {

template <int P, int S, int TH>
struct OxGeom {
  static constexpr int TW = 32;
  static constexpr int NO = 2 * S + 1;
  static constexpr int NT = 32 * NO;
  static constexpr int HR = P + S;
  static constexpr int UW0 = TW + 2 * HR;
  static constexpr int UW = ((UW0 + 30) / 32) * 32 + 1;  // == 1 (mod 32): conflict-free phase A rows
  static constexpr int UH = TH + 2 * HR;
  static constexpr int HROWS = TH + 2 * P;
  static constexpr int UOFF = ((UH * UW + 3) / 4) * 4;
  static constexpr int HBUF = NO * HROWS * TW;
  static constexpr int RED = 2 * NO * TH * TW;
  static constexpr int HS = (2 * HBUF > RED ? 2 * HBUF : RED);
  static constexpr size_t smem_bytes = (size_t)(UOFF + HS) * sizeof(float);
  static constexpr int NWIN = TH + 2 * S;
  static constexpr int NITEMS = HROWS * (TW / 4);
};

template <int P, int S, int TH>
__global__ void __launch_bounds__(32 * (2 * S + 1), 1) nlm_box_ox(NlmParams p) {
  using G = OxGeom<P, S, TH>;
  constexpr int TW = G::TW, NO = G::NO, NT = G::NT, HR = G::HR, UW = G::UW, UW0 = G::UW0, UH = G::UH;
  constexpr int HROWS = G::HROWS, PW = 2 * P + 1;
  extern __shared__ __align__(16) float sm[];
  float* U = sm;
  float* Hs = sm + G::UOFF;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int b = blockIdx.z;
  const int bx = blockIdx.x * TW, bly = blockIdx.y * TH;
  const int gy0 = p.dst.y0 + bly;
  for (int i = tid; i < UH * UW0; i += NT) {
    const int r = i / UW0, c = i % UW0;
    U[r * UW + c] = read_B(p.src, b, bx - HR + c, gy0 - HR + r);
  }
  __syncthreads();

  // u(q) column window of this warp's ox: tile rows -S .. TH+S-1.
  float uwin[G::NWIN];
#pragma unroll
  for (int k = 0; k < G::NWIN; ++k) uwin[k] = U[(k - S + HR) * UW + lane + wid + P];
  float num[TH], den[TH];
#pragma unroll
  for (int y = 0; y < TH; ++y) { num[y] = 0.0f; den[y] = 0.0f; }
  const float ncoef = -p.coef;

#pragma unroll
  for (int oyi = 0; oyi < NO; ++oyi) {
    const int oy = oyi - S;
    float* Hb = Hs + (oyi & 1) * G::HBUF;
    // ---------------- phase A
    for (int item = tid; item < G::NITEMS; item += NT) {
      const int hr = item / (TW / 4);
      const int x0 = 4 * (item % (TW / 4));
      const float* urow = U + (hr - P + HR) * UW + (x0 - P + HR);
      const float* qrow = U + (hr - P + oy + HR) * UW + (x0 - P - S + HR);
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
        *reinterpret_cast<float4*>(Hb + (oxi * HROWS + hr) * TW + x0) = make_float4(h[0], h[1], h[2], h[3]);
      }
    }
    __syncthreads();
    // ---------------- phase B (warp = ox, lane = column)
    const float* hc = Hb + wid * HROWS * TW + lane;
    float ring[PW];
#pragma unroll
    for (int t = 0; t < PW - 1; ++t) ring[t] = hc[t * TW];
#pragma unroll
    for (int y = 0; y < TH; ++y) {
      ring[(y + PW - 1) % PW] = hc[(y + PW - 1) * TW];
      float d = ring[y % PW];
#pragma unroll
      for (int t = 1; t < PW; ++t) d = __fadd_rn(d, ring[(y + t) % PW]);
      const float w = ex2_approx(__fmul_rn(d, ncoef));
      num[y] = __fmaf_rn(w, uwin[y + oyi], num[y]);
      den[y] = __fadd_rn(den[y], w);
    }
    // no barrier: the next phase A writes the other H buffer (see header)
  }
  __syncthreads();
  // ---------------- reduce the 2S+1 partial sums per pixel (ox order) and store
  float* rn = Hs;                   // [NO][TH][TW]
  float* rd = Hs + NO * TH * TW;    // [NO][TH][TW]
#pragma unroll
  for (int y = 0; y < TH; ++y) {
    rn[(wid * TH + y) * TW + lane] = num[y];
    rd[(wid * TH + y) * TW + lane] = den[y];
  }
  __syncthreads();
  for (int i = tid; i < TH * TW; i += NT) {
    const int y = i / TW, x = i % TW;
    float n = rn[i], d = rd[i];
#pragma unroll
    for (int o = 1; o < NO; ++o) {
      n = __fadd_rn(n, rn[o * TH * TW + i]);
      d = __fadd_rn(d, rd[o * TH * TW + i]);
    }
    const int gx = bx + x, ly = bly + y;
    if (gx < p.src.W && ly < p.dst.H) dst_row(p.dst, b, ly)[gx] = __fdiv_rn(n, d);
  }
}

template <int P, int S, int TH>
static cudaError_t launch_ox(const NlmParams& p, int batch, cudaStream_t s) {
  using G = OxGeom<P, S, TH>;
  auto kern = nlm_box_ox<P, S, TH>;
  static_assert(G::smem_bytes <= 227 * 1024, "shared memory");
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grd((p.src.W + G::TW - 1) / G::TW, (p.dst.H + TH - 1) / TH, batch);
  kern<<<grd, G::NT, G::smem_bytes, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

bool nlm_ox_supported(int P, int S) {
  return (P == 2 && S == 5) || (P == 1 && S == 3) || (P == 2 && S == 3) || (P == 1 && S == 5) ||
         (P == 3 && S == 7);
}

cudaError_t launch_nlm_ox(const NlmCall& c, cudaStream_t s) {
  NlmParams p = make_nlm_params(c);
  if (c.P == 2 && c.S == 5) return launch_ox<2, 5, 32>(p, c.batch, s);
  if (c.P == 1 && c.S == 3) return launch_ox<1, 3, 32>(p, c.batch, s);
  if (c.P == 2 && c.S == 3) return launch_ox<2, 3, 32>(p, c.batch, s);
  if (c.P == 1 && c.S == 5) return launch_ox<1, 5, 32>(p, c.batch, s);
  if (c.P == 3 && c.S == 7) return launch_ox<3, 7, 16>(p, c.batch, s);
  return cudaErrorInvalidValue;
}

}  // namespace icl
