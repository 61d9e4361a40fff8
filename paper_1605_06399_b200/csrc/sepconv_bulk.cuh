// sepconv_bulk.cuh -- variant family "bulk<R,NT>": fused single-pass separable
// convolution fed by the TMA engine (§6; fusion per
// PAPER.md:701-704; local-memory staging PAPER.md:484-525).
//
// A CTA owns a strip of TW = 4*NT columns x S output rows.  Input rows (TW +
// 2*HP columns) arrive in shared memory by 1-D bulk copies (cp.async.bulk,
// SASS UBLKCP) issued by one thread, in stages of P = 2R+1 rows, completion
// tracked by one mbarrier per stage slot (expect_tx bytes).  Threads never
// issue loads; one __syncthreads per stage (P rows) releases the previous
// slot, so the per-row barrier of stream<> disappears.  Each thread computes
// the row pass of its 4 columns into a register ring of P rows (static
// indices: a stage is exactly one ring period) and emits one output row per
// input row with 16-byte streaming stores.
// Boundary: interior CTAs copy whole rows; CTAs touching the left/right image
// edge copy the 16-byte-aligned in-image part and fix the halo columns (and
// a 1-3 column ragged tail) from global memory; constant-border rows outside
// the image are filled with c by the threads (no copy).  Same per-output fp32
// operation order as every other sepconv variant (bit-identical).
#pragma once
#include "common.cuh"
#include "internal.h"
#include "sepconv_stream.cuh"

namespace icl {

template <int R, int NT>
struct BulkGeom {
  static constexpr int HP = SepGeom<R>::HP;
  static constexpr int P = SepGeom<R>::P;
  static constexpr int TW = 4 * NT;
  static constexpr int ROWLEN = TW + 2 * HP;
  static constexpr int STAGE = P * ROWLEN;  // floats
  static constexpr int NS0 = 49152 / (STAGE * 4);
  static constexpr int NS = NS0 < 2 ? 2 : (NS0 > 8 ? 8 : NS0);
  static constexpr size_t smem_bytes = (size_t)NS * STAGE * 4 + 64;
};

template <int R, int NT>
__global__ void __launch_bounds__(NT) sep_bulk(SepParams p, int S) {
  using G = BulkGeom<R, NT>;
  constexpr int HP = G::HP, P = G::P, TW = G::TW, ROWLEN = G::ROWLEN, NS = G::NS;
  extern __shared__ __align__(16) float smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * G::STAGE);

  const int tid = threadIdx.x;
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TW;
  const int ly0 = blockIdx.y * S;
  const int ly1 = min(ly0 + S, p.dst.H);
  const int g0 = p.dst.y0 + ly0;
  const int NI = (ly1 - ly0) + 2 * R;
  const int NSTG = (NI + P - 1) / P;
  const int W = p.src.W, Hg = p.src.Hg;
  const bool clampb = p.src.border == kBorderClamp;
  const bool edge = (x0 - HP < 0) || (x0 + TW + HP > W);
  const int W4 = W & ~3;
  // bulk-copied column range [clo, chi) (absolute columns), 16-byte aligned
  const int clo = edge ? max(x0 - HP, 0) : x0 - HP;
  const int chi = edge ? min(x0 + TW + HP, W4) : x0 + TW + HP;
  const bool any_copy = chi > clo;

  auto issue = [&](int s) {  // thread 0 only
    float* slot = smem + (s % NS) * G::STAGE;
    uint32_t bytes = 0;
    const float* srcs[P];
#pragma unroll
    for (int u = 0; u < P; ++u) {
      srcs[u] = nullptr;
      const int k = s * P + u;
      if (k >= NI || !any_copy) continue;
      int gi = g0 - R + k;
      if (gi < 0 || gi >= Hg) {
        if (!clampb) continue;
        gi = clampi(gi, 0, Hg - 1);
      }
      srcs[u] = src_row(p.src, b, gi) + clo;
      bytes += (uint32_t)(chi - clo) * 4u;
    }
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&bars[s % NS], bytes);
#pragma unroll
    for (int u = 0; u < P; ++u)
      if (srcs[u]) bulk_g2s(slot + u * ROWLEN + (clo - (x0 - HP)), srcs[u], (uint32_t)(chi - clo) * 4u, &bars[s % NS]);
  };
  // Does stage s need thread-side filling (edge columns / constant rows)?
  auto needfix = [&](int s) {
    if (edge) return true;
    if (clampb) return false;
    const int gfirst = g0 - R + s * P, glast = gfirst + P - 1;
    return gfirst < 0 || glast >= Hg;
  };
  auto fixup = [&](int s) {
    float* slot = smem + (s % NS) * G::STAGE;
#pragma unroll 1
    for (int u = 0; u < P; ++u) {
      const int k = s * P + u;
      if (k >= NI) break;
      int gi = g0 - R + k;
      const bool outrow = gi < 0 || gi >= Hg;
      const bool crow = outrow && !clampb;
      gi = clampi(gi, 0, Hg - 1);
      const float* row = src_row(p.src, b, gi);
      float* dst = slot + u * ROWLEN;
      for (int c = tid; c < ROWLEN; c += NT) {
        const int xe = x0 - HP + c;
        if (crow) dst[c] = p.src.cval;
        else if (xe < 0) dst[c] = clampb ? __ldg(row) : p.src.cval;
        else if (xe >= W) dst[c] = clampb ? __ldg(row + W - 1) : p.src.cval;
        else if (xe < clo || xe >= chi) dst[c] = __ldg(row + xe);
      }
    }
  };

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&bars[i], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < NS && s < NSTG; ++s) issue(s);

  float4 ring[P];
  const int xc = x0 + 4 * tid;
#pragma unroll 1
  for (int s = 0; s < NSTG; ++s) {
    mbar_wait(&bars[s % NS], (uint32_t)((s / NS) & 1));
    __syncthreads();  // everyone finished stage s-1: its slot may be refilled
    if (tid == 0 && s >= 1 && s - 1 + NS < NSTG) issue(s - 1 + NS);
    if (needfix(s)) {
      fixup(s);
      __syncthreads();
    }
    const float* slot = smem + (s % NS) * G::STAGE;
#pragma unroll
    for (int u = 0; u < P; ++u) {
      const int k = s * P + u;
      if (k < NI) {
        const float* st = slot + u * ROWLEN;
        float v[4 + 2 * HP];
#pragma unroll
        for (int q = 0; q < (4 + 2 * HP) / 4; ++q) {
          const float4 w = reinterpret_cast<const float4*>(st + 4 * tid)[q];
          v[4 * q] = w.x; v[4 * q + 1] = w.y; v[4 * q + 2] = w.z; v[4 * q + 3] = w.w;
        }
        float t[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float a = 0.0f;
#pragma unroll
          for (int i = 0; i < P; ++i) a = __fmaf_rn(p.fx[i], v[HP - R + c + i], a);
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

template <int R, int NT>
static inline cudaError_t launch_bulk_R(const SepParams& p, int batch, int S, cudaStream_t s) {
  using G = BulkGeom<R, NT>;
  auto kern = sep_bulk<R, NT>;
  if (G::smem_bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::smem_bytes);
    if (e != cudaSuccess) return e;
  }
  dim3 grd((p.src.W + G::TW - 1) / G::TW, (p.dst.H + S - 1) / S, batch);
  kern<<<grd, NT, G::smem_bytes, s>>>(p, S);
  count_launch();
  return cudaGetLastError();
}

template <int NT>
cudaError_t dispatch_bulk(const SepParams& p, int R, int batch, int S, cudaStream_t s) {
  switch (R) {
#define ICL_BULK_CASE(r) \
  case r:                \
    return launch_bulk_R<r, NT>(p, batch, S, s);
    ICL_BULK_CASE(0) ICL_BULK_CASE(1) ICL_BULK_CASE(2) ICL_BULK_CASE(3) ICL_BULK_CASE(4) ICL_BULK_CASE(5)
    ICL_BULK_CASE(6) ICL_BULK_CASE(7) ICL_BULK_CASE(8) ICL_BULK_CASE(9) ICL_BULK_CASE(10) ICL_BULK_CASE(11)
    ICL_BULK_CASE(12) ICL_BULK_CASE(13) ICL_BULK_CASE(14) ICL_BULK_CASE(15)
#undef ICL_BULK_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace icl
