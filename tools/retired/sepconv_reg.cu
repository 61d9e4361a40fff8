// sepconv_reg.cu -- variant family "reg<R,NW>" (R <= 4): fused single-pass
// separable convolution streamed through REGISTERS (§6 lines
// 588-592, fusion per PAPER.md:701-704).
//
// Each warp owns a 128-column strip (lane = 4 columns, float4 = "blocked"
// mapping) and S output rows; a CTA is NW side-by-side strips.  Per input row
// a lane issues one 16-byte global load (lanes 0 / 31 one more for the strip
// halo), P = 2R+1 rows ahead of use (a register prefetch queue of one ring
// period), gets the R neighbour columns from lanes +-1 with warp shuffles,
// computes the row pass into a register ring of P rows and emits one output
// row per input row with a 16-byte streaming store.  No shared memory, no
// barriers.  Same per-output fp32 operation order as every other sepconv
// variant (bit-identical).
#include "common.cuh"
#include "internal.h"
#include "sepconv_stream.cuh"

namespace icl {

struct RowQ {
  float4 c;  // this lane's 4 columns
  float4 h;  // lane 0: 4 columns left of the strip; lane 31: 4 columns right of it
};

__device__ __forceinline__ float ldB1(const float* row, int x, int W, bool clampb, float cval) {
  if (x < 0) return clampb ? __ldg(row) : cval;
  if (x >= W) return clampb ? __ldg(row + W - 1) : cval;
  return __ldg(row + x);
}

// 4 consecutive columns x..x+3 of `row` with the boundary applied (x % 4 == 0).
__device__ __forceinline__ float4 ld4B(const float* row, int x, int W, bool clampb, float cval) {
  if (x >= 0 && x + 3 < W) return __ldg(reinterpret_cast<const float4*>(row + x));
  return make_float4(ldB1(row, x, W, clampb, cval), ldB1(row, x + 1, W, clampb, cval),
                     ldB1(row, x + 2, W, clampb, cval), ldB1(row, x + 3, W, clampb, cval));
}

template <int R, int NW>
__global__ void __launch_bounds__(32 * NW) sep_reg(SepParams p, int S) {
  constexpr int P = 2 * R + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.z;
  const int x0 = (blockIdx.x * NW + warp) * 128;
  const int xc = x0 + 4 * lane;
  const int ly0 = blockIdx.y * S;
  const int ly1 = min(ly0 + S, p.dst.H);
  const int g0 = p.dst.y0 + ly0;
  const int NI = (ly1 - ly0) + 2 * R;
  const int W = p.src.W, Hg = p.src.Hg;
  const bool clampb = p.src.border == kBorderClamp;
  const float cval = p.src.cval;
  if (x0 >= W) return;  // whole warp outside (warp-uniform; no barriers in this kernel)
  const int hx = lane == 0 ? x0 - 4 : x0 + 128;
  const bool hl = (lane == 0 || lane == 31) && R > 0;

  auto load = [&](int k) {
    RowQ q;
    int gi = g0 - R + k;
    if ((gi < 0 || gi >= Hg) && !clampb) {
      q.c = make_float4(cval, cval, cval, cval);
      q.h = q.c;
      return q;
    }
    gi = clampi(gi, 0, Hg - 1);
    const float* row = src_row(p.src, b, gi);
    q.c = ld4B(row, xc, W, clampb, cval);
    q.h = hl ? ld4B(row, hx, W, clampb, cval) : q.c;
    return q;
  };

  RowQ q[P];
#pragma unroll
  for (int u = 0; u < P; ++u)
    if (u < NI) q[u] = load(u);
  float4 ring[P];

  for (int kb = 0; kb < NI; kb += P) {
#pragma unroll
    for (int u = 0; u < P; ++u) {
      const int k = kb + u;
      if (k < NI) {
        const RowQ cur = q[u];
        if (k + P < NI) q[u] = load(k + P);
        // window: 4 columns left (lane-1), own 4, 4 right (lane+1)
        float v[12];
        v[4] = cur.c.x; v[5] = cur.c.y; v[6] = cur.c.z; v[7] = cur.c.w;
        if (R > 0) {
          float4 L, Rt;
          L.x = __shfl_up_sync(0xffffffffu, cur.c.x, 1);
          L.y = __shfl_up_sync(0xffffffffu, cur.c.y, 1);
          L.z = __shfl_up_sync(0xffffffffu, cur.c.z, 1);
          L.w = __shfl_up_sync(0xffffffffu, cur.c.w, 1);
          Rt.x = __shfl_down_sync(0xffffffffu, cur.c.x, 1);
          Rt.y = __shfl_down_sync(0xffffffffu, cur.c.y, 1);
          Rt.z = __shfl_down_sync(0xffffffffu, cur.c.z, 1);
          Rt.w = __shfl_down_sync(0xffffffffu, cur.c.w, 1);
          if (lane == 0) L = cur.h;
          if (lane == 31) Rt = cur.h;
          v[0] = L.x; v[1] = L.y; v[2] = L.z; v[3] = L.w;
          v[8] = Rt.x; v[9] = Rt.y; v[10] = Rt.z; v[11] = Rt.w;
        }
        float t[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float a = 0.0f;
#pragma unroll
          for (int i = 0; i < P; ++i) a = __fmaf_rn(p.fx[i], v[4 - R + c + i], a);
          t[c] = a;
        }
        ring[u] = make_float4(t[0], t[1], t[2], t[3]);
        if (k >= 2 * R) {
          float o[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
          for (int j = 0; j < P; ++j) {
            const float4 rr = ring[(u + 1 + j) % P];
            o[0] = __fmaf_rn(p.gy[j], rr.x, o[0]);
            o[1] = __fmaf_rn(p.gy[j], rr.y, o[1]);
            o[2] = __fmaf_rn(p.gy[j], rr.z, o[2]);
            o[3] = __fmaf_rn(p.gy[j], rr.w, o[3]);
          }
          float* drow = dst_row(p.dst, b, ly0 + k - 2 * R);
          if (xc + 3 < W) {
            st_cs4(drow + xc, make_float4(o[0], o[1], o[2], o[3]));
          } else {
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (xc + c < W) drow[xc + c] = o[c];
          }
        }
      }
    }
  }
}

template <int R, int NW>
static cudaError_t launch_reg_R(const SepParams& p, int batch, int S, cudaStream_t s) {
  dim3 grd((p.src.W + 128 * NW - 1) / (128 * NW), (p.dst.H + S - 1) / S, batch);
  sep_reg<R, NW><<<grd, 32 * NW, 0, s>>>(p, S);
  count_launch();
  return cudaGetLastError();
}

template <int NW>
static cudaError_t dispatch_reg(const SepParams& p, int R, int batch, int S, cudaStream_t s) {
  switch (R) {
    case 0: return launch_reg_R<0, NW>(p, batch, S, s);
    case 1: return launch_reg_R<1, NW>(p, batch, S, s);
    case 2: return launch_reg_R<2, NW>(p, batch, S, s);
    case 3: return launch_reg_R<3, NW>(p, batch, S, s);
    case 4: return launch_reg_R<4, NW>(p, batch, S, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_sep_reg(const SepCall& c, int nw, int S, cudaStream_t s) {
  SepParams p = make_sep_params(c, true);
  const int R = c.rx > c.ry ? c.rx : c.ry;
  if (nw == 2) return dispatch_reg<2>(p, R, c.batch, S, s);
  if (nw == 4) return dispatch_reg<4>(p, R, c.batch, S, s);
  return cudaErrorInvalidValue;
}

}  // namespace icl
