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

// Ring of blurred rows: RB rows per block as harris_shfl (a multiple of B, so the general
// path's window slots are static), but only 3 blocks -- the producer writes block i+2 while
// the consumer reads block i and the first rows of block i+1, and rows are produced by the
// CTA itself (no load latency to hide), so a deeper ring would only cost occupancy.
template <int B>
struct ChainGeom {
  static constexpr int RB = HarFastGeom<B>::RB;
  static constexpr int NBLKS = 3;
  static constexpr int NSR = RB * NBLKS;
};

struct BlurHarrisParams {
  HarrisParams h;  // h.src: the source image with the HARRIS boundary (applied to the blurred image)
  SrcView raw;     // the same image with the SEPCONV boundary
  float fx[2 * kMaxRadius + 1];
  float gy[2 * kMaxRadius + 1];
};

template <int R, int B, int NW>
__device__ __forceinline__ void blur_harris_general(const BlurHarrisParams& bp, int S, float* smem) {
  const HarrisParams& p = bp.h;
  constexpr int A = B / 2;
  constexpr int BB = B - 1 - A;
  constexpr int NT = 32 * NW;
  constexpr int HP = 8;
  constexpr int TW = 120 * NW;
  constexpr int ROWLEN = TW + 2 * HP;
  constexpr int NSLOT = ROWLEN / 4;
  constexpr int RB = ChainGeom<B>::RB, NBLKS = ChainGeom<B>::NBLKS, NSR = ChainGeom<B>::NSR;
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

// Interior CTAs (every raw row and column the chain touches inside the image): the
// harris_shfl_interior consumer (mirror ring rows, compile-time offsets, running
// vertical sums) fed by the blur producer.  The producer keeps its row-pass rows t
// in a per-slot shared-memory ring (K rows x 4 columns per thread) instead of
// registers, so the consumer keeps its register budget.  Same values as the
// general path (bit-identical).
template <int R, int B, int NW>
__device__ __forceinline__ void blur_harris_interior(const BlurHarrisParams& bp, int S, float* smem) {
  const HarrisParams& p = bp.h;
  constexpr int A = B / 2;
  constexpr int BB = B - 1 - A;
  constexpr int HP = 8;
  constexpr int TW = 120 * NW;
  constexpr int ROWLEN = TW + 2 * HP;
  constexpr int NSLOT = ROWLEN / 4;
  constexpr int RB = ChainGeom<B>::RB, NBLKS = ChainGeom<B>::NBLKS, NSR = ChainGeom<B>::NSR;
  constexpr int K = 2 * R + 1;
  constexpr int RAWLEN = ROWLEN + 8;
  constexpr int NRAW = 2 * RB + 2 * R + 1;
  static_assert(RB >= 2, "mirror rows cover the two rows a step reads past its block");
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
  float* raw = smem + (NSR + 2) * ROWLEN;
  float* tring = raw + NRAW * RAWLEN;  // [K][NSLOT][4]
  const int xr0 = x0 - HP - 4;
  const int64_t spitch = bp.raw.pitch >> 2;
  const float* rbase = src_row(bp.raw, b, 0) + xr0;  // raw row 0, ring column 0

  // raw rows: cp.async, one ring block ahead of the producer
  int rl = g0 - A - 1 - R;  // next raw row to load
  auto load_for_block = [&](int m) {
    const int hi = g0 - A - 1 + min(m * RB + RB - 1, NL - 1) + R;
    for (; rl <= hi; ++rl) {
      float* st = raw + (rl % NRAW) * RAWLEN;
      const float* g = rbase + (int64_t)rl * spitch;
      for (int c = tid; c < RAWLEN / 4; c += 32 * NW) cp_async16(st + 4 * c, g + 4 * c, 16);
    }
    cp_async_commit();
  };
  // Ring indices are carried incrementally (no constant-divisor modulo in the row loop): the
  // raw row gi + R of produced row kl sits in raw slot rs, its row pass goes to t slot ts, and
  // the window's oldest t row (gi - R) is t slot to.
  const float* rawt = raw + 4 * tid;
  float* trt = tring + 4 * tid;
  auto row_pass = [&](const float* rrow, float* tdst) {
    const float4* rr = reinterpret_cast<const float4*>(rrow);
    const float4 w0 = rr[0], w1 = rr[1], w2 = rr[2];
    const float v12[12] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w, w2.x, w2.y, w2.z, w2.w};
    float o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float acc = 0.0f;
#pragma unroll
      for (int i = 0; i < K; ++i) acc = __fmaf_rn(bp.fx[i], v12[4 - R + q + i], acc);
      o[q] = acc;
    }
    *reinterpret_cast<float4*>(tdst) = make_float4(o[0], o[1], o[2], o[3]);
  };
  const int r_first = g0 - A - 1 - R;  // first raw row of the CTA (>= 0 here)
  int rs = (r_first + 2 * R) % NRAW;   // raw slot of row (gi + R) for kl = 0
  int ts = (2 * R) % K;                // t slot of that row
  int to = 0;                          // t slot of row gi - R
  int kr = 0;                          // blurred ring row of kl
  auto produce_block = [&](int m) {
    if (tid >= NSLOT) return;
    if (m == 0) {  // the window's first 2R rows
      int s = r_first % NRAW;
#pragma unroll 1
      for (int j = 0; j < 2 * R; ++j) {
        row_pass(rawt + s * RAWLEN, trt + j * NSLOT * 4);
        s = s + 1 == NRAW ? 0 : s + 1;
      }
    }
    const int nu = min(RB, NL - m * RB);
#pragma unroll 1
    for (int u = 0; u < nu; ++u) {
      row_pass(rawt + rs * RAWLEN, trt + ts * NSLOT * 4);
      float4 acc = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const int sj = to + j < K ? to + j : to + j - K;
        const float4 tv = *reinterpret_cast<const float4*>(trt + sj * NSLOT * 4);
        acc.x = __fmaf_rn(bp.gy[j], tv.x, acc.x);
        acc.y = __fmaf_rn(bp.gy[j], tv.y, acc.y);
        acc.z = __fmaf_rn(bp.gy[j], tv.z, acc.z);
        acc.w = __fmaf_rn(bp.gy[j], tv.w, acc.w);
      }
      *reinterpret_cast<float4*>(smem + kr * ROWLEN + 4 * tid) = acc;
      if (kr < 2) *reinterpret_cast<float4*>(smem + (NSR + kr) * ROWLEN + 4 * tid) = acc;  // mirror
      rs = rs + 1 == NRAW ? 0 : rs + 1;
      ts = ts + 1 == K ? 0 : ts + 1;
      to = to + 1 == K ? 0 : to + 1;
      kr = kr + 1 == NSR ? 0 : kr + 1;
    }
  };
  load_for_block(0);
  for (int m = 0; m < NBLKS - 1; ++m) {
    if (m + 1 < NBL) load_for_block(m + 1);
    else cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (m < NBL) produce_block(m);
    __syncthreads();
  }
  if (NBLKS - 1 < NBL) load_for_block(NBLKS - 1);
  else cp_async_commit();

  const int xl = x0 + 120 * warp + 4 * (lane - 1);
  const float* stb = smem + (xl - (x0 - HP));
  const bool emit = lane >= 1 && lane <= 30;
  constexpr int NC = B > 1 ? B - 1 : 1;
  float2 c2[NC][4];
  float2 cxy[NC][2];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
#pragma unroll
    for (int q = 0; q < 4; ++q) c2[k][q] = make_float2(0.0f, 0.0f);
    cxy[k][0] = cxy[k][1] = make_float2(0.0f, 0.0f);
  }
  float* drow = dst_row(p.dst, b, ly0) + xl;
  const int64_t dpitch = p.dst.pitch >> 2;
  const bool has_mask = p.mask != nullptr;
  char* mrow = has_mask ? p.mask + (int64_t)b * p.mbstride + (int64_t)ly0 * p.mpitch + xl : nullptr;

#pragma unroll 1
  for (int i = 0; i < NBI; ++i) {
    cp_async_wait<0>();
    __syncthreads();
    if (i + NBLKS - 1 < NBL) produce_block(i + NBLKS - 1);
    if (i + NBLKS < NBL) load_for_block(i + NBLKS);
    const float* sb = stb + (i % NBLKS) * RB * ROWLEN;
#pragma unroll 1
    for (int u = 0; u < RB; ++u) {
      const int step = i * RB + u;
      if (step < NY) {
        float4 w[3];
        float il[3], ir[3];
        float hd[3][4];
#pragma unroll
        for (int rr = 0; rr < 3; ++rr) {
          w[rr] = *reinterpret_cast<const float4*>(sb + (u + rr) * ROWLEN);
          il[rr] = __shfl_up_sync(0xffffffffu, w[rr].w, 1);
          ir[rr] = __shfl_down_sync(0xffffffffu, w[rr].x, 1);
          const float2 m = __fadd2_rn(make_float2(w[rr].z, w[rr].w), make_float2(-w[rr].x, -w[rr].y));
          hd[rr][0] = __fsub_rn(w[rr].y, il[rr]);
          hd[rr][1] = m.x;
          hd[rr][2] = m.y;
          hd[rr][3] = __fsub_rn(ir[rr], w[rr].z);
        }
        float vd[6];
        {
          const float2 v12 = __fadd2_rn(make_float2(w[2].x, w[2].y), make_float2(-w[0].x, -w[0].y));
          const float2 v34 = __fadd2_rn(make_float2(w[2].z, w[2].w), make_float2(-w[0].z, -w[0].w));
          vd[0] = __fsub_rn(il[2], il[0]);
          vd[1] = v12.x; vd[2] = v12.y; vd[3] = v34.x; vd[4] = v34.y;
          vd[5] = __fsub_rn(ir[2], ir[0]);
        }
        float2 g[8];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          g[c + 2].x = __fmaf_rn(2.0f, hd[1][c], __fadd_rn(hd[0][c], hd[2][c]));
          g[c + 2].y = __fmaf_rn(2.0f, vd[c + 1], __fadd_rn(vd[c], vd[c + 2]));
        }
        g[0].x = __shfl_up_sync(0xffffffffu, g[4].x, 1);
        g[0].y = __shfl_up_sync(0xffffffffu, g[4].y, 1);
        g[1].x = __shfl_up_sync(0xffffffffu, g[5].x, 1);
        g[1].y = __shfl_up_sync(0xffffffffu, g[5].y, 1);
        g[6].x = __shfl_down_sync(0xffffffffu, g[2].x, 1);
        g[6].y = __shfl_down_sync(0xffffffffu, g[2].y, 1);
        g[7].x = __shfl_down_sync(0xffffffffu, g[3].x, 1);
        g[7].y = __shfl_down_sync(0xffffffffu, g[3].y, 1);
        float2 h2[4];
        float2 hxy[2];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float2 hxxyy = make_float2(0.0f, 0.0f);
          float hh = 0.0f;
#pragma unroll
          for (int t2 = -A; t2 <= BB; ++t2) {
            const float2 gg = g[2 + q + t2];
            hxxyy = __ffma2_rn(gg, gg, hxxyy);
            hh = __fmaf_rn(gg.x, gg.y, hh);
          }
          h2[q] = hxxyy;
          if (q & 1) hxy[q >> 1].y = hh;
          else hxy[q >> 1].x = hh;
        }
        float2 s2o[4];
        float2 sxyo[2];
        if (B > 1) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            s2o[q] = __fadd2_rn(c2[0][q], h2[q]);
#pragma unroll
            for (int k = 0; k + 1 < NC; ++k) c2[k][q] = __fadd2_rn(c2[k + 1][q], h2[q]);
            c2[NC - 1][q] = h2[q];
          }
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            sxyo[m] = __fadd2_rn(cxy[0][m], hxy[m]);
#pragma unroll
            for (int k = 0; k + 1 < NC; ++k) cxy[k][m] = __fadd2_rn(cxy[k + 1][m], hxy[m]);
            cxy[NC - 1][m] = hxy[m];
          }
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) s2o[q] = h2[q];
          sxyo[0] = hxy[0];
          sxyo[1] = hxy[1];
        }
        if (step >= B - 1) {
          float R4[4];
          R4[0] = harris_R(s2o[0].x, sxyo[0].x, s2o[0].y, p.k);
          R4[1] = harris_R(s2o[1].x, sxyo[0].y, s2o[1].y, p.k);
          R4[2] = harris_R(s2o[2].x, sxyo[1].x, s2o[2].y, p.k);
          R4[3] = harris_R(s2o[3].x, sxyo[1].y, s2o[3].y, p.k);
          if (emit) {
            st_cs4(drow, make_float4(R4[0], R4[1], R4[2], R4[3]));
            if (has_mask)
              *reinterpret_cast<uchar4*>(mrow) = make_uchar4(R4[0] > p.threshold, R4[1] > p.threshold,
                                                             R4[2] > p.threshold, R4[3] > p.threshold);
          }
          drow += dpitch;
          mrow += has_mask ? p.mpitch : 0;
        }
      }
    }
  }
  cp_async_wait<0>();
}

template <int R, int B, int NW>
__global__ void __launch_bounds__(32 * NW, 16 / NW) blur_harris_kernel(BlurHarrisParams bp, int S) {
  extern __shared__ __align__(16) float smem[];
  constexpr int TW = 120 * NW, HP = 8, A = B / 2, BB = B - 1 - A;
  const int x0 = blockIdx.x * TW, ly0 = blockIdx.y * S;
  const int ly1 = min(ly0 + S, bp.h.dst.H);
  const int g0 = bp.h.dst.y0 + ly0;
  // every raw row and column the CTA touches (Harris halo + blur radius) inside the image
  const bool interior = x0 - HP - 4 >= 0 && x0 + TW + HP + 4 <= bp.h.src.W && g0 - A - 1 - R >= 0 &&
                        bp.h.dst.y0 + ly1 + BB + 1 + R <= bp.h.src.Hg && g0 - A - 1 - R >= bp.h.src.y0 &&
                        bp.h.dst.y0 + ly1 + BB + 1 + R <= bp.h.src.y0 + bp.h.src.Hl &&
                        ((bp.raw.pitch | (int64_t)bp.raw.base) & 15) == 0;
  if (interior) blur_harris_interior<R, B, NW>(bp, S, smem);
  else blur_harris_general<R, B, NW>(bp, S, smem);
}

template <int R, int B>
static cudaError_t launch_bh(const BlurHarrisParams& bp, int batch, int S, cudaStream_t s) {
  constexpr int NW = 4;
  constexpr int TW = 120 * NW;
  const size_t smem = ((size_t)(ChainGeom<B>::NSR + 2) * (TW + 16) +   // blurred ring + mirror rows
                       (size_t)(2 * ChainGeom<B>::RB + 2 * R + 1) * (TW + 24) +  // raw rows
                       (size_t)(2 * R + 1) * (TW + 16)) * sizeof(float);  // row-pass ring (interior)
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
