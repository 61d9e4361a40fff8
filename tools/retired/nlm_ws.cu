// nlm_ws.cu -- NLM variant "boxsum_ws": warp-specialised offset-major
// separable box sums.  (NLM is not in PAPER.md; definition DESIGN.md R11-R14.)
//
// CTA = 16 warps over a 32-column x TH-row output tile, TH = 32 - 2P, its
// bounding-box input tile U (halo P+S, boundary applied at load -- the
// paper's local-memory staging) in shared memory.
//
//  producers (warpgroup 0, 128 threads, setmaxnreg 88): thread (k, seg)
//    computes, for every search row oy and every ox, the horizontal patch
//    sums  H_o(x, r) = sum_{tx=-P..P} (u(x+tx, r) - u(x+tx+ox, r+oy))^2
//    of 4 columns and the ROW PAIR (r_k, r_k + 16), packed in FFMA2/FADD2
//    lanes; H rows r in [-P, TH+P) = 32 rows = 16 pairs.  Sliding sums along
//    the 4 columns.  Stored as float2 (H(k), H(k+16)) per column in a
//    double-buffered shared-memory area (layout below, conflict-free).
//  consumers (warpgroups 1-3, 12 warps, setmaxnreg 136): warp w owns
//    ox = w - S, lane x one output column, for all TH rows and all oy; rows
//    (y, y+16) are packed in float2 lanes: d = sum of 2P+1 H rows,
//    w = 2^(-d*coef), num = fma(w, u(q), num), den += w, with num/den and the
//    u(q) column window in registers (the oy loop is unrolled).
//  The two roles hand H buffers over with named barriers (FULL: producers
//    arrive / consumers sync; EMPTY: consumers arrive / producers sync), so
//    phase A of oy+1 overlaps phase B of oy.
//  At the end the 2S+1 per-ox partial sums of each pixel are added in ox
//    order through shared memory (deterministic), divided and stored.
#include "nlm_common.cuh"

namespace icl {

template <int P, int S>
struct WsGeom {
  static constexpr int TW = 32;
  static constexpr int TH = 32 - 2 * P;      // producer rows = 32 = 16 pairs
  static constexpr int NO = 2 * S + 1;       // consumer warps used (<= 12)
  static constexpr int NT = 512;
  static constexpr int HR = P + S;
  static constexpr int UW0 = TW + 2 * HR;
  static constexpr int UW = ((UW0 + 30) / 32) * 32 + 1;
  static constexpr int UH = TH + 2 * HR;
  static constexpr int UOFF = ((UH * UW + 3) / 4) * 4;
  static constexpr int HBUF = NO * 16 * TW * 2;   // floats per H buffer
  static constexpr int RED = 2 * NO * TH * TW;    // num/den partials
  static constexpr size_t smem_bytes = (size_t)(UOFF + 2 * HBUF + RED) * sizeof(float);
  static constexpr int NPK = 16 - 2 * P;          // packed consumer row pairs (y, y+16)
  static constexpr int NW2 = 16 + 2 * S;          // u(q) window pairs
};

// H buffer layout: float index of (ox, k, column x = 4*seg + 2*j + e, r2)
__device__ __forceinline__ int hidx(int ox, int k, int j, int seg, int e) {
  return ((((ox * 16 + k) * 2 + j) * 8 + seg) * 4) + 2 * e;
}

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n)); }

template <int P, int S>
__global__ void __launch_bounds__(512, 1) nlm_ws(NlmParams p) {
  using G = WsGeom<P, S>;
  constexpr int TW = G::TW, TH = G::TH, NO = G::NO, HR = G::HR, UW = G::UW, UW0 = G::UW0, UH = G::UH;
  constexpr int PW = 2 * P + 1, NPK = G::NPK, NW2 = G::NW2;
  extern __shared__ __align__(16) float sm[];
  float* U = sm;
  float* Hs = sm + G::UOFF;
  float* red = Hs + 2 * G::HBUF;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int b = blockIdx.z;
  const int bx = blockIdx.x * TW, bly = blockIdx.y * TH;
  const int gy0 = p.dst.y0 + bly;
  for (int i = tid; i < UH * UW0; i += G::NT) {
    const int r = i / UW0, c = i % UW0;
    U[r * UW + c] = read_B(p.src, b, bx - HR + c, gy0 - HR + r);
  }
  __syncthreads();

  if (wid < 4) {
    // =========================== producers ===========================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n");
    const int k = tid >> 3, seg = tid & 7, x0 = 4 * seg;
    const float* ua = U + (k - P + HR) * UW + (x0 - P + HR);
    const float* ub = ua + 16 * UW;
    float2 nup[4 + 2 * P];
#pragma unroll
    for (int c = 0; c < 4 + 2 * P; ++c) nup[c] = make_float2(-ua[c], -ub[c]);
#pragma unroll 1
    for (int oyi = 0; oyi < NO; ++oyi) {
      const int buf = oyi & 1;
      if (oyi >= 2) named_sync(3 + buf, 512);  // EMPTY[buf]: consumers done with oy-2
      float* Hb = Hs + buf * G::HBUF;
      const float* qa = ua + (oyi - S) * UW - S;
      const float* qb = qa + 16 * UW;
      float2 uq[4 + 2 * P + 2 * S];
#pragma unroll
      for (int c = 0; c < 4 + 2 * P + 2 * S; ++c) uq[c] = make_float2(qa[c], qb[c]);
#pragma unroll
      for (int oxi = 0; oxi < NO; ++oxi) {
        float2 df[4 + 2 * P];
#pragma unroll
        for (int c = 0; c < 4 + 2 * P; ++c) df[c] = __fadd2_rn(uq[c + oxi], nup[c]);
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
        *reinterpret_cast<float4*>(Hb + hidx(oxi, k, 0, seg, 0)) = make_float4(h[0].x, h[0].y, h[1].x, h[1].y);
        *reinterpret_cast<float4*>(Hb + hidx(oxi, k, 1, seg, 0)) = make_float4(h[2].x, h[2].y, h[3].x, h[3].y);
      }
      named_arrive(1 + buf, 512);  // FULL[buf]
    }
  } else {
    // =========================== consumers ===========================
    asm volatile("setmaxnreg.inc.sync.aligned.u32 136;\n");
    const int w = wid - 4;             // ox index (warps >= NO idle but keep the handshake)
    const bool act = w < NO;
    const int wo = act ? w : 0;
    // u(q) column window: pair m = (tile row m-S, tile row m-S+16) at column lane+ox
    float2 uw[NW2];
    {
      const float* col = U + lane + wo + P;  // (lane + ox + HR) with ox = wo - S
#pragma unroll
      for (int m = 0; m < NW2; ++m) {
        const float lo = col[(m - S + HR) * UW];
        const float hi = (m < NPK + 2 * S) ? col[(m - S + 16 + HR) * UW] : 0.0f;
        uw[m] = make_float2(lo, hi);
      }
    }
    float2 num[NPK], den[NPK];
    float nums[2 * P], dens[2 * P];
#pragma unroll
    for (int y = 0; y < NPK; ++y) { num[y] = make_float2(0.f, 0.f); den[y] = make_float2(0.f, 0.f); }
#pragma unroll
    for (int y = 0; y < 2 * P; ++y) { nums[y] = 0.f; dens[y] = 0.f; }
    const float nc = -p.coef;
    const int seg = lane >> 2, jj = (lane >> 1) & 1, e = lane & 1;
#pragma unroll
    for (int oyi = 0; oyi < NO; ++oyi) {
      const int buf = oyi & 1;
      named_sync(1 + buf, 512);  // FULL[buf]
      if (act) {
        const float* hb = Hs + buf * G::HBUF + hidx(wo, 0, jj, seg, e);
        constexpr int KST = 2 * 8 * 4;  // float stride between consecutive k
        float2 hk[16];
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) hk[kk] = *reinterpret_cast<const float2*>(hb + kk * KST);
        // packed rows (y, y+16), y < NPK: d = H(y..y+2P) (.x) and H(y+16..y+16+2P) (.y)
#pragma unroll
        for (int y = 0; y < NPK; ++y) {
          float2 d = hk[y];
#pragma unroll
          for (int t = 1; t < PW; ++t) d = __fadd2_rn(d, hk[y + t]);
          const float2 x2 = __fmul2_rn(d, make_float2(nc, nc));
          const float2 w2 = make_float2(ex2_approx(x2.x), ex2_approx(x2.y));
          num[y] = __ffma2_rn(w2, uw[y + oyi], num[y]);
          den[y] = __fadd2_rn(den[y], w2);
        }
        // scalar rows y = NPK .. 15: H rows y..y+2P straddle the pair boundary
#pragma unroll
        for (int yy = 0; yy < 2 * P; ++yy) {
          const int y = NPK + yy;
          float d = hk[y].x;
#pragma unroll
          for (int t = 1; t < PW; ++t) d = __fadd_rn(d, (y + t < 16) ? hk[y + t].x : hk[y + t - 16].y);
          const float wv = ex2_approx(__fmul_rn(d, nc));
          nums[yy] = __fmaf_rn(wv, uw[y + oyi].x, nums[yy]);
          dens[yy] = __fadd_rn(dens[yy], wv);
        }
      }
      if (oyi + 2 < NO) named_arrive(3 + buf, 512);  // EMPTY[buf] (the last two are never awaited)
    }
    if (act) {
      // partials -> red[ox][row][col]
      float* rn = red;
      float* rd = red + NO * TH * TW;
#pragma unroll
      for (int y = 0; y < NPK; ++y) {
        rn[(wo * TH + y) * TW + lane] = num[y].x;
        rd[(wo * TH + y) * TW + lane] = den[y].x;
        rn[(wo * TH + y + 16) * TW + lane] = num[y].y;
        rd[(wo * TH + y + 16) * TW + lane] = den[y].y;
      }
#pragma unroll
      for (int yy = 0; yy < 2 * P; ++yy) {
        rn[(wo * TH + NPK + yy) * TW + lane] = nums[yy];
        rd[(wo * TH + NPK + yy) * TW + lane] = dens[yy];
      }
    }
  }
  __syncthreads();
  {
    const float* rn = red;
    const float* rd = red + NO * TH * TW;
    for (int i = tid; i < TH * TW; i += G::NT) {
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
}

template <int P, int S>
static cudaError_t launch_ws(const NlmParams& p, int batch, cudaStream_t s) {
  using G = WsGeom<P, S>;
  static_assert(G::NO <= 12, "at most 12 consumer warps");
  static_assert(G::smem_bytes <= 227 * 1024, "shared memory");
  auto kern = nlm_ws<P, S>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grd((p.src.W + G::TW - 1) / G::TW, (p.dst.H + G::TH - 1) / G::TH, batch);
  kern<<<grd, G::NT, G::smem_bytes, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

bool nlm_ws_supported(int P, int S) {
  return (P == 2 && S == 5) || (P == 1 && S == 3) || (P == 2 && S == 3) || (P == 1 && S == 5);
}

cudaError_t launch_nlm_ws(const NlmCall& c, cudaStream_t s) {
  NlmParams p = make_nlm_params(c);
  if (c.P == 2 && c.S == 5) return launch_ws<2, 5>(p, c.batch, s);
  if (c.P == 1 && c.S == 3) return launch_ws<1, 3>(p, c.batch, s);
  if (c.P == 2 && c.S == 3) return launch_ws<2, 3>(p, c.batch, s);
  if (c.P == 1 && c.S == 5) return launch_ws<1, 5>(p, c.batch, s);
  return cudaErrorInvalidValue;
}

}  // namespace icl
