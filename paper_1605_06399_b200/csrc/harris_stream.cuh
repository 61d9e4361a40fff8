// harris_stream.cuh -- the fused streaming Harris kernel template and its
// launch helpers; instantiated per CTA width in harris_nt*.cu (parallel build).
#pragma once
#include "common.cuh"
#include "internal.h"

namespace icl {

struct HarrisParams {
  SrcView src;
  DstView dst;
  char* mask;
  int64_t mpitch, mbstride;
  int block;
  float k;
  float threshold;
};

__device__ __forceinline__ float harris_R(float sxx, float sxy, float syy, float k) {
  const float det = __fmaf_rn(sxx, syy, -__fmul_rn(sxy, sxy));
  const float tr = __fadd_rn(sxx, syy);
  return __fmaf_rn(-k, __fmul_rn(tr, tr), det);
}

// --------------------------------------------------------------------------
// Variant family "stream<B,NT,VEC>": fused Sobel + structure tensor +
// response (+ mask) in one pass.  A CTA owns a strip of TW = 4*NT columns and
// S output rows; input rows (with 4 halo columns each side) stream through an
// NS-stage cp.async ring in shared memory.  For every H-row yy (the rows the
// window sums touch) the thread reads the 3 input rows around
// r = clamp(yy, 0, Hg-1) from the ring, computes hd/vd -> dx/dy -> the three
// horizontal product sums for its 4 columns, and keeps the last B of them in
// a register ring; each step emits one output row.  For clamp, yy outside the
// image reuses row r's values (== dx(clamp(q))); for constant they are 0.
// --------------------------------------------------------------------------
constexpr int kHarStages = 10;

// Border path: CTAs whose strip touches the left/right image edge or whose
// rows touch the top/bottom (clamp/constant logic per H-row, one barrier per
// input row).
// TW_/HP_: output columns per CTA and halo columns per side (the warp-shuffle
// kernel of harris_shfl.cuh uses 120*NW and 8); threads with 4*tid >= TW only
// help with the loads.
template <int B, int NT, int VEC, int TW_ = 4 * NT, int HP_ = 4>
__device__ __forceinline__ void harris_slow(const HarrisParams& p, int S, float* smem) {
  constexpr int NS = kHarStages;
  constexpr int A = B / 2;
  constexpr int BB = B - 1 - A;
  constexpr int HP = HP_;  // >= A + 1 (4 suffices for B <= 7), multiple of 4
  constexpr int TW = TW_;
  constexpr int ROWLEN = TW + 2 * HP;
  constexpr int NSLOT = ROWLEN / 4;
  constexpr int NC = 4 + B - 1;  // dx/dy columns per thread: xc-A .. xc+3+BB

  const int tid = threadIdx.x;
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TW;
  const int ly0 = blockIdx.y * S;
  const int ly1 = min(ly0 + S, p.dst.H);
  const int g0 = p.dst.y0 + ly0;
  const int g1 = p.dst.y0 + ly1;
  const int W = p.src.W;
  const int Hg = p.src.Hg;
  const bool clampb = p.src.border == kBorderClamp;
  const bool edge = (x0 - HP < 0) || (x0 + TW + HP > W);
  const int r0 = clampi(g0 - A, 0, Hg - 1);
  const int rl = clampi(g1 - 1 + BB, 0, Hg - 1);
  const int NL = rl - r0 + 3;  // loads: global rows r0-1 .. rl+1

  auto load_row = [&](int kl) {
    if (kl >= NL) return;
    float* st = smem + (kl % NS) * ROWLEN;
    int gi = r0 - 1 + kl;
    if (gi < 0 || gi >= Hg) {
      if (!clampb) {
        for (int s = tid; s < NSLOT; s += NT)
          reinterpret_cast<float4*>(st)[s] = make_float4(p.src.cval, p.src.cval, p.src.cval, p.src.cval);
        return;
      }
      gi = clampi(gi, 0, Hg - 1);
    }
    const float* row = src_row(p.src, b, gi);
    for (int s = tid; s < NSLOT; s += NT) {
      const int xs = x0 - HP + 4 * s;
      if (VEC == 4) {
        int nb = (xs < 0) ? 0 : min(max(W - xs, 0), 4) * 4;
        cp_async16(st + 4 * s, nb ? (const void*)(row + xs) : (const void*)row, nb);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int xe = xs + e;
          const bool in = xe >= 0 && xe < W;
          cp_async4(st + 4 * s + e, in ? (const void*)(row + xe) : (const void*)row, in ? 4 : 0);
        }
      }
    }
  };
  // Boundary fix-up of the halo columns of load kl (input image boundary).
  auto fix_row = [&](int kl) {
    float* st = smem + (kl % NS) * ROWLEN;
    const int il = HP - x0;
    const int ir = (W - 1) - x0 + HP;
    const float vl = (il >= 0 && il < ROWLEN) ? st[il] : 0.0f;  // column 0, if in this row
    const float vr = (ir >= 0 && ir < ROWLEN) ? st[ir] : 0.0f;  // column W-1, if in this row
    for (int s = tid; s < NSLOT; s += NT) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int xe = x0 - HP + 4 * s + e;
        if (xe < 0) st[4 * s + e] = clampb ? vl : p.src.cval;
        else if (xe >= W) st[4 * s + e] = clampb ? vr : p.src.cval;
      }
    }
  };

  // Prologue: loads 0..NS-3.
  for (int kl = 0; kl < NS - 2; ++kl) {
    load_row(kl);
    cp_async_commit();
  }

  const int xc = x0 + 4 * tid;
  const bool active = xc < W && 4 * tid < TW;
  float hring[B][12];  // [slot][ {xx[4], xy[4], yy[4]} ]
  int cidx = 0;        // load index of the current centre row (0 = none yet)
  const int NY = (ly1 - ly0) + B - 1;

  for (int kb = 0; kb < NY; kb += B) {
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int step = kb + u;
      if (step < NY) {
        const int yy = g0 - A + step;
        const int r = clampi(yy, 0, Hg - 1);
        const int want = r - r0 + 1;  // load index of row r
        if (want != cidx) {           // advance the window by one input row (uniform)
          cidx = want;
          cp_async_wait<NS - 5>();  // loads 0..cidx+1 complete
          __syncthreads();
          if (edge) {
            if (cidx == 1) { fix_row(0); fix_row(1); }
            fix_row(cidx + 1);
            __syncthreads();
          }
          load_row(cidx + NS - 3);
          cp_async_commit();
        }
        float* hs = hring[u];
        const bool zero = (!clampb) && (yy < 0 || yy >= Hg);
        if (zero || !active) {
#pragma unroll
          for (int q = 0; q < 12; ++q) hs[q] = 0.0f;
        } else {
          float in[3][12];
#pragma unroll
          for (int rr = 0; rr < 3; ++rr) {
            const float* st = smem + ((cidx - 1 + rr) % NS) * ROWLEN + 4 * tid + (HP - 4);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              const float4 w = reinterpret_cast<const float4*>(st)[q];
              in[rr][4 * q] = w.x; in[rr][4 * q + 1] = w.y; in[rr][4 * q + 2] = w.z; in[rr][4 * q + 3] = w.w;
            }
          }
          // window column c <-> global column xc - 4 + c
          float vd[12];
#pragma unroll
          for (int c = 3 - A; c <= 8 + BB; ++c) vd[c] = __fsub_rn(in[2][c], in[0][c]);
          float dx[12], dy[12];
#pragma unroll
          for (int c = 4 - A; c <= 7 + BB; ++c) {
            const float h0 = __fsub_rn(in[0][c + 1], in[0][c - 1]);
            const float h1 = __fsub_rn(in[1][c + 1], in[1][c - 1]);
            const float h2 = __fsub_rn(in[2][c + 1], in[2][c - 1]);
            dx[c] = __fmaf_rn(2.0f, h1, __fadd_rn(h0, h2));
            dy[c] = __fmaf_rn(2.0f, vd[c], __fadd_rn(vd[c - 1], vd[c + 1]));
          }
          if (edge) {  // per-stage boundary of dx/dy at columns outside [0, W)
            float lx = 0.0f, ly = 0.0f, rx = 0.0f, ry = 0.0f;
#pragma unroll
            for (int c = 4 - A; c <= 7 + BB; ++c) {
              if (xc - 4 + c == 0) { lx = dx[c]; ly = dy[c]; }
              if (xc - 4 + c == W - 1) { rx = dx[c]; ry = dy[c]; }
            }
#pragma unroll
            for (int c = 4 - A; c <= 7 + BB; ++c) {
              const int xe = xc - 4 + c;
              if (xe < 0) { dx[c] = clampb ? lx : 0.0f; dy[c] = clampb ? ly : 0.0f; }
              else if (xe >= W) { dx[c] = clampb ? rx : 0.0f; dy[c] = clampb ? ry : 0.0f; }
            }
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float hxx = 0.0f, hxy = 0.0f, hyy = 0.0f;
#pragma unroll
            for (int t = -A; t <= BB; ++t) {
              const float gx = dx[4 + q + t], gy = dy[4 + q + t];
              hxx = __fmaf_rn(gx, gx, hxx);
              hxy = __fmaf_rn(gx, gy, hxy);
              hyy = __fmaf_rn(gy, gy, hyy);
            }
            hs[q] = hxx; hs[4 + q] = hxy; hs[8 + q] = hyy;
          }
        }
        (void)NC;
        if (step >= B - 1 && active) {
          const int ly = ly0 + step - (B - 1);
          float R[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float sxx = hring[(u + 1) % B][q], sxy = hring[(u + 1) % B][4 + q], syy = hring[(u + 1) % B][8 + q];
#pragma unroll
            for (int j = 1; j < B; ++j) {
              sxx = __fadd_rn(sxx, hring[(u + 1 + j) % B][q]);
              sxy = __fadd_rn(sxy, hring[(u + 1 + j) % B][4 + q]);
              syy = __fadd_rn(syy, hring[(u + 1 + j) % B][8 + q]);
            }
            R[q] = harris_R(sxx, sxy, syy, p.k);
          }
          float* drow = dst_row(p.dst, b, ly);
          const bool full = xc + 3 < W;
          if (VEC == 4 && full) st_cs4(drow + xc, make_float4(R[0], R[1], R[2], R[3]));
          else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (xc + q < W) drow[xc + q] = R[q];
          }
          if (p.mask) {
            char* mrow = p.mask + (int64_t)b * p.mbstride + (int64_t)ly * p.mpitch;
            unsigned char m[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) m[q] = R[q] > p.threshold ? 1 : 0;
            if (VEC == 4 && full) {
              *reinterpret_cast<uchar4*>(mrow + xc) = make_uchar4(m[0], m[1], m[2], m[3]);
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (xc + q < W) mrow[xc + q] = m[q];
            }
          }
        }
      }
    }
  }
  cp_async_wait<0>();
}


// --------------------------------------------------------------------------
// Interior fast path: every input row and column the CTA touches is inside
// the image, so r == yy for every H-row, no boundary logic runs, copy
// addresses are fixed per thread (running row pointers), and one barrier
// serves a block of RB H-rows (RB a multiple of B: static ring indices).
// Identical fp32 operation order to the border path and the naive variant.
// --------------------------------------------------------------------------
template <int B>
struct HarFastGeom {
  static constexpr int RB = B * ((4 + B - 1) / B);
  static constexpr int NBLKS = RB <= 8 ? 5 : 4;
  static constexpr int NSR = RB * NBLKS;
};

template <int B, int NT>
__device__ __forceinline__ void harris_fast(const HarrisParams& p, int S, float* smem) {
  constexpr int A = B / 2;
  constexpr int BB = B - 1 - A;
  constexpr int HP = 4;
  constexpr int TW = 4 * NT;
  constexpr int ROWLEN = TW + 2 * HP;
  constexpr int NSLOT = ROWLEN / 4;
  constexpr int RB = HarFastGeom<B>::RB, NBLKS = HarFastGeom<B>::NBLKS, NSR = HarFastGeom<B>::NSR;
  const int tid = threadIdx.x;
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TW;
  const int ly0 = blockIdx.y * S;
  const int ly1 = min(ly0 + S, p.dst.H);
  const int g0 = p.dst.y0 + ly0;
  const int NY = (ly1 - ly0) + B - 1;  // H-rows: global g0-A .. g0-A+NY-1
  const int NL = NY + 2;               // input rows: global g0-A-1 .. g0-A+NY
  const int NBI = (NY + RB - 1) / RB;  // step blocks
  const int NBL = (NL + RB - 1) / RB;  // load blocks
  const float* row0 = src_row(p.src, b, g0 - A - 1) + (x0 - HP);
  const int64_t spitch = p.src.pitch >> 2;
  const int s1 = tid + NT;

  auto load_block = [&](int m) {
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const int kl = m * RB + u;
      if (kl < NL) {
        float* st = smem + (kl % NSR) * ROWLEN;
        const float* row = row0 + (int64_t)kl * spitch;
        cp_async16(st + 4 * tid, row + 4 * tid, 16);
        if (s1 < NSLOT) cp_async16(st + 4 * s1, row + 4 * s1, 16);
      }
    }
  };
  for (int m = 0; m < NBLKS - 1; ++m) {
    if (m < NBL) load_block(m);
    cp_async_commit();
  }

  const int xc = x0 + 4 * tid;
  // ring of the last B H-rows: (Hxx, Hyy) packed per column + Hxy
  float2 hr2[B][4];
  float hrxy[B][4];
  float* drow = dst_row(p.dst, b, ly0);
  const int64_t dpitch = p.dst.pitch >> 2;
  char* mrow = p.mask ? p.mask + (int64_t)b * p.mbstride + (int64_t)ly0 * p.mpitch : nullptr;

#pragma unroll 1
  for (int i = 0; i < NBI; ++i) {
    cp_async_wait<NBLKS - 3>();  // load blocks 0 .. i+1 complete
    __syncthreads();             // ... for all threads; load block i-1 is free
    if (i + NBLKS - 1 < NBL) load_block(i + NBLKS - 1);
    cp_async_commit();
    const int base = (i % NBLKS) * RB;  // smem row of load index i*RB
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const int step = i * RB + u;
      if (step < NY) {
        float in[3][12];
#pragma unroll
        for (int rr = 0; rr < 3; ++rr) {
          int sr = base + u + rr;
          if (sr >= NSR) sr -= NSR;
          const float* st = smem + sr * ROWLEN + 4 * tid;
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const float4 w = reinterpret_cast<const float4*>(st)[q];
            in[rr][4 * q] = w.x; in[rr][4 * q + 1] = w.y; in[rr][4 * q + 2] = w.z; in[rr][4 * q + 3] = w.w;
          }
        }
        float vd[12];
#pragma unroll
        for (int c = 3 - A; c <= 8 + BB; ++c) vd[c] = __fsub_rn(in[2][c], in[0][c]);
        float2 g[12];  // (dx, dy) per column: operands of the packed products
#pragma unroll
        for (int c = 4 - A; c <= 7 + BB; ++c) {
          const float h0 = __fsub_rn(in[0][c + 1], in[0][c - 1]);
          const float h1 = __fsub_rn(in[1][c + 1], in[1][c - 1]);
          const float h2 = __fsub_rn(in[2][c + 1], in[2][c - 1]);
          g[c].x = __fmaf_rn(2.0f, h1, __fadd_rn(h0, h2));
          g[c].y = __fmaf_rn(2.0f, vd[c], __fadd_rn(vd[c - 1], vd[c + 1]));
        }
        const int slot = u % B;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float2 hxxyy = make_float2(0.0f, 0.0f);
          float hxy = 0.0f;
#pragma unroll
          for (int t = -A; t <= BB; ++t) {
            const float2 gg = g[4 + q + t];
            hxxyy = __ffma2_rn(gg, gg, hxxyy);  // (dx^2 + Hxx, dy^2 + Hyy): same rounding as 2 FFMA
            hxy = __fmaf_rn(gg.x, gg.y, hxy);
          }
          hr2[slot][q] = hxxyy;
          hrxy[slot][q] = hxy;
        }
        if (step >= B - 1) {
          float R[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float2 s2 = hr2[(u + 1) % B][q];
            float sxy = hrxy[(u + 1) % B][q];
#pragma unroll
            for (int j = 1; j < B; ++j) {
              s2 = __fadd2_rn(s2, hr2[(u + 1 + j) % B][q]);
              sxy = __fadd_rn(sxy, hrxy[(u + 1 + j) % B][q]);
            }
            R[q] = harris_R(s2.x, sxy, s2.y, p.k);
          }
          st_cs4(drow + xc, make_float4(R[0], R[1], R[2], R[3]));
          drow += dpitch;
          if (mrow) {
            *reinterpret_cast<uchar4*>(mrow + xc) =
                make_uchar4(R[0] > p.threshold, R[1] > p.threshold, R[2] > p.threshold, R[3] > p.threshold);
            mrow += p.mpitch;
          }
        }
      }
    }
  }
  cp_async_wait<0>();
}

template <int B, int NT, int VEC>
__global__ void __launch_bounds__(NT) harris_stream(HarrisParams p, int S) {
  extern __shared__ __align__(16) float smem[];
  constexpr int A = B / 2, BB = B - 1 - A, TW = 4 * NT;
  const int x0 = blockIdx.x * TW;
  const int ly0 = blockIdx.y * S;
  const int ly1 = min(ly0 + S, p.dst.H);
  const int g0 = p.dst.y0 + ly0;
  const bool fast = VEC == 4 && x0 - 4 >= 0 && x0 + TW + 4 <= p.src.W && g0 - A - 1 >= 0 &&
                    g0 + (ly1 - ly0) + BB + 1 <= p.src.Hg;
  if (fast) harris_fast<B, NT>(p, S, smem);
  else harris_slow<B, NT, VEC>(p, S, smem);
}

template <int B, int NT, int VEC>
static inline cudaError_t launch_hs(const HarrisParams& p, int batch, int S, cudaStream_t s) {
  constexpr int ROWLEN = 4 * NT + 8;
  const int rows = kHarStages > HarFastGeom<B>::NSR ? kHarStages : HarFastGeom<B>::NSR;
  const size_t smem = (size_t)rows * ROWLEN * sizeof(float);
  auto kern = harris_stream<B, NT, VEC>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grd((p.src.W + 4 * NT - 1) / (4 * NT), (p.dst.H + S - 1) / S, batch);
  kern<<<grd, NT, smem, s>>>(p, S);
  count_launch();
  return cudaGetLastError();
}

template <int NT, int VEC>
cudaError_t dispatch_hs(const HarrisParams& p, int batch, int S, cudaStream_t s) {
  switch (p.block) {
    case 1: return launch_hs<1, NT, VEC>(p, batch, S, s);
    case 2: return launch_hs<2, NT, VEC>(p, batch, S, s);
    case 3: return launch_hs<3, NT, VEC>(p, batch, S, s);
    case 4: return launch_hs<4, NT, VEC>(p, batch, S, s);
    case 5: return launch_hs<5, NT, VEC>(p, batch, S, s);
    case 6: return launch_hs<6, NT, VEC>(p, batch, S, s);
    case 7: return launch_hs<7, NT, VEC>(p, batch, S, s);
    default: return cudaErrorInvalidValue;
  }
}


}  // namespace icl
