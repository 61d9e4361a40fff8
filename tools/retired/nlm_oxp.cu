// nlm_oxp.cu -- NLM variant "boxsum_oxp": offset-major separable patch sums
// with phase-B threads that own a whole tile column for a PAIR of horizontal
// offsets.  (NLM is not in PAPER.md; definition DESIGN.md R11-R14.)
//
// CTA = 32x32 output tile, 32 * ceil((2S+1)/2) threads (one warp per ox pair,
// lane = column).  Per search row oy:
//   phase A  (thread = 8-column row segment) horizontal patch sums H_o of all
//            2S+1 ox, sliding along the 8 columns; stored interleaved by ox
//            pair, (H_{2k}, H_{2k+1}) per column, rows padded to 80 words and
//            the column-pair order rotated per segment (conflict-free
//            16-byte stores);
//   phase B  (warp = ox pair, lane = column x, all 32 rows) one LDS.64 per H
//            row gives both offsets; vertical sums slide along the rows (fresh
//            start every 8 rows), w = 2^(-d*coef) per offset, and both offsets
//            accumulate into ONE scalar num/den per pixel (registers).
// Shared-memory words per (pixel, offset): phase A 0.39 load + 1.1 store,
// phase B 1.1 H + 1 u(q) = 3.6 (boxsum_r8: 4.2).  The per-pair partial sums
// are added in a fixed order at the end.
#include "nlm_common.cuh"

namespace icl {

template <int P, int S>
struct OxpGeom {
  static constexpr int TW = 32, TH = 32;
  static constexpr int NO = 2 * S + 1;
  static constexpr int NOP = (NO + 1) / 2;  // ox pairs (the last may be a single)
  static constexpr int NT = 32 * NOP;
  static constexpr int HR = P + S;
  static constexpr int UW0 = TW + 2 * HR;
  static constexpr int UW = ((UW0 + 30) / 32) * 32 + 1;
  static constexpr int UH = TH + 2 * HR;
  static constexpr int HROWS = TH + 2 * P;
  static constexpr int RS = 80;  // words per H row: 32 columns x 2 offsets + 16 pad
  static constexpr int UOFF = ((UH * UW + 3) / 4) * 4;
  static constexpr int HSZ = NOP * HROWS * RS;
  static constexpr int RED = 2 * NOP * TH * TW;
  static constexpr size_t smem_bytes = (size_t)(UOFF + (HSZ > RED ? HSZ : RED)) * sizeof(float);
  static constexpr int NITEMS = HROWS * (TW / 8);
};

template <int P, int S>
__global__ void __launch_bounds__(32 * ((2 * S + 2) / 2), 2) nlm_box_oxp(NlmParams p) {
  using G = OxpGeom<P, S>;
  constexpr int TW = G::TW, TH = G::TH, HR = G::HR, UW = G::UW, UW0 = G::UW0, UH = G::UH;
  constexpr int HROWS = G::HROWS, NO = G::NO, RS = G::RS, PW = 2 * P + 1;
  extern __shared__ __align__(16) float sm[];
  float* U = sm;
  float* Hs = sm + G::UOFF;
  const int tid = threadIdx.x, lane = tid & 31, pr = tid >> 5;
  const int b = blockIdx.z;
  const int bx = blockIdx.x * TW, bly = blockIdx.y * TH;
  const int gy0 = p.dst.y0 + bly;
  for (int i = tid; i < UH * UW0; i += G::NT) {
    const int r = i / UW0, c = i % UW0;
    U[r * UW + c] = read_B(p.src, b, bx - HR + c, gy0 - HR + r);
  }
  __syncthreads();

  float num[TH], den[TH];
#pragma unroll
  for (int y = 0; y < TH; ++y) { num[y] = 0.0f; den[y] = 0.0f; }
  const float nc = -p.coef;
  const bool has_y = 2 * pr + 1 < NO;  // warp-uniform: second offset of the pair exists

#pragma unroll 1
  for (int oy = -S; oy <= S; ++oy) {
    // ---------------- phase A
    if (tid < G::NITEMS) {
      const int hr = tid >> 2, seg = tid & 3;
      const int x = 8 * seg;
      const float* urow = U + (hr - P + HR) * UW + (x + HR - P);
      const float* qrow = U + (hr - P + oy + HR) * UW + (x + HR - P - S);
      float up[8 + 2 * P], uq[8 + 2 * P + 2 * S];
#pragma unroll
      for (int c = 0; c < 8 + 2 * P; ++c) up[c] = urow[c];
#pragma unroll
      for (int c = 0; c < 8 + 2 * P + 2 * S; ++c) uq[c] = qrow[c];
      float* hrow = Hs + hr * RS + 2 * x;  // + pair * HROWS * RS
#pragma unroll
      for (int k = 0; k < (NO + 1) / 2; ++k) {
        float h[2][8];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int oxi = 2 * k + e;
          if (oxi < NO) {
            float df[8 + 2 * P];
#pragma unroll
            for (int c = 0; c < 8 + 2 * P; ++c) df[c] = __fsub_rn(up[c], uq[c + oxi]);
            float a = __fmul_rn(df[0], df[0]);
#pragma unroll
            for (int t = 1; t < PW; ++t) a = __fmaf_rn(df[t], df[t], a);
            h[e][0] = a;
#pragma unroll
            for (int j = 1; j < 8; ++j) {
              a = __fmaf_rn(df[j + 2 * P], df[j + 2 * P], a);
              a = __fmaf_rn(-df[j - 1], df[j - 1], a);
              h[e][j] = a;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) h[e][j] = 0.0f;
          }
        }
        float* hp = hrow + k * HROWS * RS;
#pragma unroll
        for (int st = 0; st < 4; ++st) {
          const int cp = (st + seg) & 3;  // rotated column pair: conflict-free 16-byte stores
          // select with static indices (cp is runtime): 4-way
          float a0, a1, a2, a3;
          if (cp == 0) { a0 = h[0][0]; a1 = h[1][0]; a2 = h[0][1]; a3 = h[1][1]; }
          else if (cp == 1) { a0 = h[0][2]; a1 = h[1][2]; a2 = h[0][3]; a3 = h[1][3]; }
          else if (cp == 2) { a0 = h[0][4]; a1 = h[1][4]; a2 = h[0][5]; a3 = h[1][5]; }
          else { a0 = h[0][6]; a1 = h[1][6]; a2 = h[0][7]; a3 = h[1][7]; }
          *reinterpret_cast<float4*>(hp + 4 * cp) = make_float4(a0, a1, a2, a3);
        }
      }
    }
    __syncthreads();
    // ---------------- phase B: warp = ox pair, lane = column, all TH rows
    {
      const float* hc = Hs + pr * HROWS * RS + 2 * lane;
      const int ox0 = 2 * pr - S;
      const float* q0 = U + (oy + HR) * UW + (lane + ox0 + HR);
      float2 ring[PW];
      float2 d = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int y = 0; y < TH; ++y) {
        if (y % 8 == 0) {  // fresh sum every 8 rows (bounded rounding drift)
#pragma unroll
          for (int t = 0; t < PW; ++t) ring[(y + t) % PW] = *reinterpret_cast<const float2*>(hc + (y + t) * RS);
          d = ring[y % PW];
#pragma unroll
          for (int t = 1; t < PW; ++t) d = __fadd2_rn(d, ring[(y + t) % PW]);
        } else {
          const float2 hn = *reinterpret_cast<const float2*>(hc + (y + PW - 1) * RS);
          d = __fadd2_rn(__fadd2_rn(d, hn), make_float2(-ring[(y - 1) % PW].x, -ring[(y - 1) % PW].y));
          ring[(y + PW - 1) % PW] = hn;
        }
        const float2 xv = __fmul2_rn(d, make_float2(nc, nc));
        const float w0 = ex2_approx(xv.x);
        const float u0 = q0[y * UW];
        num[y] = __fmaf_rn(w0, u0, num[y]);
        den[y] = __fadd_rn(den[y], w0);
        if (has_y) {
          const float w1 = ex2_approx(xv.y);
          const float u1 = q0[y * UW + 1];
          num[y] = __fmaf_rn(w1, u1, num[y]);
          den[y] = __fadd_rn(den[y], w1);
        }
      }
    }
    __syncthreads();
  }
  // ---------------- combine the ox pairs (fixed order) and store
  float* rn = Hs;                        // [pair][TH][TW]
  float* rd = Hs + G::NOP * TH * TW;
#pragma unroll
  for (int y = 0; y < TH; ++y) {
    rn[(pr * TH + y) * TW + lane] = num[y];
    rd[(pr * TH + y) * TW + lane] = den[y];
  }
  __syncthreads();
  for (int i = tid; i < TH * TW; i += G::NT) {
    const int y = i / TW, x = i % TW;
    float n = rn[i], dd = rd[i];
#pragma unroll
    for (int o = 1; o < G::NOP; ++o) {
      n = __fadd_rn(n, rn[o * TH * TW + i]);
      dd = __fadd_rn(dd, rd[o * TH * TW + i]);
    }
    const int gx = bx + x, ly = bly + y;
    if (gx < p.src.W && ly < p.dst.H) dst_row(p.dst, b, ly)[gx] = __fdiv_rn(n, dd);
  }
}

template <int P, int S>
static cudaError_t launch_oxp(const NlmParams& p, int batch, cudaStream_t s) {
  using G = OxpGeom<P, S>;
  static_assert(G::smem_bytes <= 227 * 1024, "shared memory");
  auto kern = nlm_box_oxp<P, S>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grd((p.src.W + G::TW - 1) / G::TW, (p.dst.H + G::TH - 1) / G::TH, batch);
  kern<<<grd, G::NT, G::smem_bytes, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

bool nlm_oxp_supported(int P, int S) {
  return (P == 2 && S == 5) || (P == 1 && S == 3) || (P == 2 && S == 3) || (P == 1 && S == 5);
}

cudaError_t launch_nlm_oxp(const NlmCall& c, cudaStream_t s) {
  NlmParams p = make_nlm_params(c);
  if (c.P == 2 && c.S == 5) return launch_oxp<2, 5>(p, c.batch, s);
  if (c.P == 1 && c.S == 3) return launch_oxp<1, 3>(p, c.batch, s);
  if (c.P == 2 && c.S == 3) return launch_oxp<2, 3>(p, c.batch, s);
  if (c.P == 1 && c.S == 5) return launch_oxp<1, 5>(p, c.batch, s);
  return cudaErrorInvalidValue;
}

}  // namespace icl
