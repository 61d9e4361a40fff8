// blur_harris.cu -- a two-filter pipeline in one pass: separable (Gaussian)
// pre-smoothing followed by Harris (FAST-style filter
// chains, §2.2 lines 128-142 -- "connecting together pre-implemented
// filters to form a pipeline", each filter taking and producing images).
//
// Semantics (R24): the chain of the two library calls
//     blurred = icl_sepconv(src, taps, sep border)        (fp32 image)
//     R, mask = icl_harris(blurred, block, k, harris border)
// computed without the intermediate image in HBM: 9 B/px instead of 8 + 9.
// The blurred value of every pixel is the sepconv fp32 chain
//     t_j = fma-chain_i fx[i] * src_B(x+i, y+j),  b = fma-chain_j gy[j] * t_j
// and the Harris stage is harris_shfl_fast's, so the result equals the two
// calls bit for bit (tests/test_gpu_chain.py).
//
// Structure: the harris_shfl<B,NW> kernel with its cp.async input loader
// replaced by a blur producer.  Thread s owns ring columns 4s..4s+3 of the
// CTA's blurred rows; it keeps the row-pass results t of the last 2R+1 raw
// rows for those columns in registers (a sliding window: one new raw row per
// blurred row, three 16-byte loads), and writes each blurred row into the
// shared-memory ring the Harris stage reads, one ring block (RB rows) ahead.
#include "common.cuh"
#include "harris_shfl.cuh"
#include "internal.h"

namespace icl {

struct BlurHarrisParams {
  HarrisParams h;  // h.src: the source image with the HARRIS boundary (applied to the blurred image)
  SrcView raw;     // the same image with the SEPCONV boundary
  float fx[2 * kMaxRadius + 1];
  float gy[2 * kMaxRadius + 1];
};

template <int R, int B, int NW>
__global__ void __launch_bounds__(32 * NW) blur_harris_kernel(BlurHarrisParams bp, int S) {
  extern __shared__ __align__(16) float smem[];
  const HarrisParams& p = bp.h;
  constexpr int A = B / 2;
  constexpr int BB = B - 1 - A;
  constexpr int NT = 32 * NW;
  constexpr int HP = 8;
  constexpr int TW = 120 * NW;
  constexpr int ROWLEN = TW + 2 * HP;
  constexpr int NSLOT = ROWLEN / 4;
  constexpr int RB = HarFastGeom<B>::RB, NBLKS = HarFastGeom<B>::NBLKS, NSR = HarFastGeom<B>::NSR;
  constexpr int K = 2 * R + 1;
  static_assert(NSLOT <= NT, "one producer slot per thread");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TW;
  const int ly0 = blockIdx.y * S;
  const int ly1 = min(ly0 + S, p.dst.H);
  const int g0 = p.dst.y0 + ly0;
  const int NY = (ly1 - ly0) + B - 1;
  const int NL = NY + 2;
  const int NBI = (NY + RB - 1) / RB;
  const int NBL = (NL + RB - 1) / RB;
  const int W = p.src.W;
  const int Hg = p.src.Hg;
  const bool clampb = p.src.border == kBorderClamp;
  const bool edge = x0 - HP < 0 || x0 + TW + HP > W;

  // ---------------- raw-row ring: raw rows stream in by cp.async one ring block ahead of the
  // producer (RAWLEN columns: the CTA's ring columns plus 4 each side for the blur footprint)
  constexpr int RAWLEN = ROWLEN + 8;
  constexpr int NRAW = 2 * RB + 2 * R + 1;  // rows of the producing block + the block being loaded
  float* raw = smem + NSR * ROWLEN;
  const int xr0 = x0 - HP - 4;               // global column of raw ring column 0
  const bool raw_edge = xr0 < 0 || xr0 + RAWLEN > W;
  auto raw_slot = [&](int r) { return raw + (((r % NRAW) + NRAW) % NRAW) * RAWLEN; };
  auto load_raw = [&](int r) {
    float* st = raw_slot(r);
    const bool out_row = r < 0 || r >= Hg;
    if (out_row && bp.raw.border == kBorderConstant) {
      for (int c = tid; c < RAWLEN; c += NT) st[c] = bp.raw.cval;
      return;
    }
    const float* row = src_row(bp.raw, b, clampi(r, 0, Hg - 1));
    if (!raw_edge) {
      for (int c = tid; c < RAWLEN / 4; c += NT) cp_async16(st + 4 * c, row + xr0 + 4 * c, 16);
    } else {  // sepconv boundary on the columns (synchronous; edge strips only)
      for (int c = tid; c < RAWLEN; c += NT) {
        int x = xr0 + c;
        if (x < 0 || x >= W) {
          if (bp.raw.border == kBorderConstant) {
            st[c] = bp.raw.cval;
            continue;
          }
          x = clampi(x, 0, W - 1);
        }
        st[c] = __ldg(row + x);
      }
    }
  };
  // raw rows block m's blurred rows need: up to clamp(last input row of m) + R
  int rl = clampi(g0 - A - 1, 0, Hg - 1) - R;  // next raw row to load
  auto load_for_block = [&](int m) {
    const int kl = min(m * RB + RB - 1, NL - 1);
    const int hi = clampi(g0 - A - 1 + kl, 0, Hg - 1) + R;
    for (; rl <= hi; ++rl) load_raw(rl);
    cp_async_commit();
  };

  // ---------------- blur producer state (thread = ring slot)
  float tw[K][4];
  int tc = INT_MIN;  // centre raw row of the window
  // row pass of raw row r (global) for the slot's 4 columns -> t[4]
  auto trow = [&](int r, float (&t)[4]) {
    const float4* rr = reinterpret_cast<const float4*>(raw_slot(r) + 4 * tid);
    const float4 w0 = rr[0], w1 = rr[1], w2 = rr[2];
    const float v12[12] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w, w2.x, w2.y, w2.z, w2.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float a = 0.0f;
#pragma unroll
      for (int i = 0; i < K; ++i) a = __fmaf_rn(bp.fx[i], v12[4 - R + q + i], a);
      t[q] = a;
    }
  };
  // blurred Harris-input rows of ring block m (Harris boundary: clamp -> the
  // blurred row at clamp(gi); constant -> the constant)
  auto produce_block = [&](int m) {
    if (tid >= NSLOT) return;
#pragma unroll 1
    for (int u = 0; u < RB; ++u) {
      const int kl = m * RB + u;
      if (kl >= NL) break;
      float* st = smem + (kl % NSR) * ROWLEN + 4 * tid;
      int gi = g0 - A - 1 + kl;
      if (gi < 0 || gi >= Hg) {
        if (!clampb) {
          *reinterpret_cast<float4*>(st) = make_float4(p.src.cval, p.src.cval, p.src.cval, p.src.cval);
          continue;
        }
        gi = clampi(gi, 0, Hg - 1);
      }
      if (gi == tc + 1) {  // slide the window by one raw row
#pragma unroll
        for (int j = 0; j + 1 < K; ++j)
#pragma unroll
          for (int q = 0; q < 4; ++q) tw[j][q] = tw[j + 1][q];
        trow(gi + R, tw[K - 1]);
        tc = gi;
      } else if (gi != tc) {
#pragma unroll
        for (int j = 0; j < K; ++j) trow(gi - R + j, tw[j]);
        tc = gi;
      }
      float o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float a = 0.0f;
#pragma unroll
        for (int j = 0; j < K; ++j) a = __fmaf_rn(bp.gy[j], tw[j][q], a);
        o[q] = a;
      }
      *reinterpret_cast<float4*>(st) = make_float4(o[0], o[1], o[2], o[3]);
    }
  };
  // Harris input boundary of the halo columns outside [0, W) of ring block m
  auto fix_block = [&](int m) {
    for (int u = 0; u < RB; ++u) {
      const int kl = m * RB + u;
      if (kl >= NL) break;
      float* st = smem + (kl % NSR) * ROWLEN;
      const int il = HP - x0, ir = (W - 1) - x0 + HP;
      const float vl = (il >= 0 && il < ROWLEN) ? st[il] : 0.0f;
      const float vr = (ir >= 0 && ir < ROWLEN) ? st[ir] : 0.0f;
      for (int c = tid; c < ROWLEN; c += NT) {
        const int xe = x0 - HP + c;
        if (xe < 0) st[c] = clampb ? vl : p.src.cval;
        else if (xe >= W) st[c] = clampb ? vr : p.src.cval;
      }
    }
  };
  // prologue: ring blocks 0 .. NBLKS-2, raw rows double-buffered one block ahead
  load_for_block(0);
  for (int m = 0; m < NBLKS - 1; ++m) {
    if (m + 1 < NBL) load_for_block(m + 1);
    else cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (m < NBL) produce_block(m);
    __syncthreads();  // the producer is done with these raw rows before they are overwritten
  }
  if (NBLKS - 1 < NBL) load_for_block(NBLKS - 1);
  else cp_async_commit();

  // ---------------- Harris stage (harris_shfl_fast, reading the blurred ring)
  const int xl = x0 + 120 * warp + 4 * (lane - 1);
  const int si = xl - (x0 - HP);
  const bool emit = lane >= 1 && lane <= 30 && xl < W;
  const int xw = x0 + 120 * warp - 4;
  const int ll = (0 - xw) >> 2, el = (0 - xw) & 3;
  const int lr = (W - 1 - xw) >> 2, er = (W - 1 - xw) & 3;
  float2 hr2[B][4];
  float hrxy[B][4];
  float* drow = dst_row(p.dst, b, ly0);
  const int64_t dpitch = p.dst.pitch >> 2;
  char* mrow = p.mask ? p.mask + (int64_t)b * p.mbstride + (int64_t)ly0 * p.mpitch : nullptr;

#pragma unroll 1
  for (int i = 0; i < NBI; ++i) {
    cp_async_wait<0>();  // raw rows of block i + NBLKS - 1
    __syncthreads();     // ... and the ring blocks produced so far are visible
    if (edge) {
      if (i == 0) fix_block(0);
      if (i + 1 < NBL) fix_block(i + 1);
      __syncthreads();
    }
    if (i + NBLKS - 1 < NBL) produce_block(i + NBLKS - 1);
    if (i + NBLKS < NBL) load_for_block(i + NBLKS);  // (ring of 2 blocks + 2R rows: no overlap)
    const int base = (i % NBLKS) * RB;
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const int step = i * RB + u;
      if (step < NY) {
        const int yy = g0 - A + step;
        const int dz = yy < 0 ? -yy : (yy >= Hg ? (Hg - 1) - yy : 0);
        float in[3][6];
#pragma unroll
        for (int rr = 0; rr < 3; ++rr) {
          int sr = base + u + rr + dz;
          if (sr >= NSR) sr -= NSR;
          if (sr < 0) sr += NSR;
          const float* st = smem + sr * ROWLEN + si;
          const float4 w = *reinterpret_cast<const float4*>(st);
          in[rr][0] = __shfl_up_sync(0xffffffffu, w.w, 1);
          in[rr][1] = w.x; in[rr][2] = w.y; in[rr][3] = w.z; in[rr][4] = w.w;
          in[rr][5] = __shfl_down_sync(0xffffffffu, w.x, 1);
        }
        float vd[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) vd[c] = __fsub_rn(in[2][c], in[0][c]);
        float2 g[8];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float h0 = __fsub_rn(in[0][c + 2], in[0][c]);
          const float h1 = __fsub_rn(in[1][c + 2], in[1][c]);
          const float h2 = __fsub_rn(in[2][c + 2], in[2][c]);
          g[c + 2].x = __fmaf_rn(2.0f, h1, __fadd_rn(h0, h2));
          g[c + 2].y = __fmaf_rn(2.0f, vd[c + 1], __fadd_rn(vd[c], vd[c + 2]));
        }
        if (edge) {
          const float2 e0 = el == 0 ? g[2] : el == 1 ? g[3] : el == 2 ? g[4] : g[5];
          const float2 e1 = er == 0 ? g[2] : er == 1 ? g[3] : er == 2 ? g[4] : g[5];
          float2 gl, gr;
          gl.x = __shfl_sync(0xffffffffu, e0.x, ll & 31);
          gl.y = __shfl_sync(0xffffffffu, e0.y, ll & 31);
          gr.x = __shfl_sync(0xffffffffu, e1.x, lr & 31);
          gr.y = __shfl_sync(0xffffffffu, e1.y, lr & 31);
          if (!clampb) gl = gr = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int xe = xl + c;
            if (xe < 0) g[c + 2] = gl;
            else if (xe >= W) g[c + 2] = gr;
          }
        }
        g[0].x = __shfl_up_sync(0xffffffffu, g[4].x, 1);
        g[0].y = __shfl_up_sync(0xffffffffu, g[4].y, 1);
        g[1].x = __shfl_up_sync(0xffffffffu, g[5].x, 1);
        g[1].y = __shfl_up_sync(0xffffffffu, g[5].y, 1);
        g[6].x = __shfl_down_sync(0xffffffffu, g[2].x, 1);
        g[6].y = __shfl_down_sync(0xffffffffu, g[2].y, 1);
        g[7].x = __shfl_down_sync(0xffffffffu, g[3].x, 1);
        g[7].y = __shfl_down_sync(0xffffffffu, g[3].y, 1);
        const int slot = u % B;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float2 hxxyy = make_float2(0.0f, 0.0f);
          float hxy = 0.0f;
#pragma unroll
          for (int t = -A; t <= BB; ++t) {
            const float2 gg = g[2 + q + t];
            hxxyy = __ffma2_rn(gg, gg, hxxyy);
            hxy = __fmaf_rn(gg.x, gg.y, hxy);
          }
          hr2[slot][q] = hxxyy;
          hrxy[slot][q] = hxy;
        }
        if (dz != 0 && !clampb) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            hr2[slot][q] = make_float2(0.0f, 0.0f);
            hrxy[slot][q] = 0.0f;
          }
        }
        if (step >= B - 1) {
          float R4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float2 s2 = hr2[(u + 1) % B][q];
            float sxy = hrxy[(u + 1) % B][q];
#pragma unroll
            for (int j = 1; j < B; ++j) {
              s2 = __fadd2_rn(s2, hr2[(u + 1 + j) % B][q]);
              sxy = __fadd_rn(sxy, hrxy[(u + 1 + j) % B][q]);
            }
            R4[q] = harris_R(s2.x, sxy, s2.y, p.k);
          }
          if (emit) {
            if (xl + 3 < W) {
              st_cs4(drow + xl, make_float4(R4[0], R4[1], R4[2], R4[3]));
              if (mrow)
                *reinterpret_cast<uchar4*>(mrow + xl) = make_uchar4(R4[0] > p.threshold, R4[1] > p.threshold,
                                                                    R4[2] > p.threshold, R4[3] > p.threshold);
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (xl + q < W) {
                  drow[xl + q] = R4[q];
                  if (mrow) mrow[xl + q] = R4[q] > p.threshold ? 1 : 0;
                }
            }
          }
          drow += dpitch;
          if (mrow) mrow += p.mpitch;
        }
      }
    }
  }
}

template <int R, int B>
static cudaError_t launch_bh(const BlurHarrisParams& bp, int batch, int S, cudaStream_t s) {
  constexpr int NW = 2;
  constexpr int TW = 120 * NW;
  const size_t smem = ((size_t)HarFastGeom<B>::NSR * (TW + 16) +
                       (size_t)(2 * HarFastGeom<B>::RB + 2 * R + 1) * (TW + 24)) * sizeof(float);
  auto kern = blur_harris_kernel<R, B, NW>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grd((bp.h.src.W + TW - 1) / TW, (bp.h.dst.H + S - 1) / S, batch);
  kern<<<grd, 32 * NW, smem, s>>>(bp, S);
  count_launch();
  return cudaGetLastError();
}

template <int R>
static cudaError_t dispatch_bh_b(const BlurHarrisParams& bp, int batch, int S, cudaStream_t s) {
  switch (bp.h.block) {
    case 1: return launch_bh<R, 1>(bp, batch, S, s);
    case 2: return launch_bh<R, 2>(bp, batch, S, s);
    case 3: return launch_bh<R, 3>(bp, batch, S, s);
    case 4: return launch_bh<R, 4>(bp, batch, S, s);
    case 5: return launch_bh<R, 5>(bp, batch, S, s);
    default: return cudaErrorInvalidValue;
  }
}

bool blur_harris_supported(int R, int block) { return R >= 0 && R <= 3 && block >= 1 && block <= 5; }

cudaError_t launch_blur_harris(const HarrisCall& h, const SrcView& raw, const float* fx, int rx, const float* gy,
                               int ry, int S, cudaStream_t s) {
  BlurHarrisParams bp;
  bp.h.src = h.src;
  bp.h.dst = h.dst;
  bp.h.mask = h.mask;
  bp.h.mpitch = h.mpitch;
  bp.h.mbstride = h.mbstride;
  bp.h.block = h.block;
  bp.h.k = h.k;
  bp.h.threshold = h.threshold;
  bp.raw = raw;
  const int R = rx > ry ? rx : ry;  // taps zero-padded to R (fma(0, v, a) == a: same values)
  for (int i = 0; i < 2 * kMaxRadius + 1; ++i) bp.fx[i] = bp.gy[i] = 0.0f;
  for (int i = -rx; i <= rx; ++i) bp.fx[R + i] = fx[rx + i];
  for (int j = -ry; j <= ry; ++j) bp.gy[R + j] = gy[ry + j];
  switch (R) {
    case 0: return dispatch_bh_b<0>(bp, h.batch, S, s);
    case 1: return dispatch_bh_b<1>(bp, h.batch, S, s);
    case 2: return dispatch_bh_b<2>(bp, h.batch, S, s);
    case 3: return dispatch_bh_b<3>(bp, h.batch, S, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace icl
