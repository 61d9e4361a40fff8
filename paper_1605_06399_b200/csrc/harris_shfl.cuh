// harris_shfl.cuh -- Harris variant family "shfl<B,NW>": the fused streaming
// Harris kernel (§6; Tables 4-5) with the window halo
// exchanged by warp shuffles instead of recomputed.
//
// Each lane computes (dx, dy) only for its own 4 columns (differences-first
// Sobel, R19) and fetches the B-1 neighbour columns the window sums
// need from lanes -1 / +1 (__shfl_up/down, 8 shuffles per H-row for B <= 5).
// Warps overlap by one lane on each side: lanes 0 and 31 only supply halo
// columns, lanes 1..30 emit outputs, so a warp produces 120 columns and a
// CTA of NW warps a strip of TW = 120*NW columns.  The Sobel stage costs
// ~34 FP32 ops per H-row instead of ~74 (no 2x halo recomputation); the rest
// (FFMA2-packed (Sxx,Syy) window sums, ring of B H-rows, response, mask) is
// the stream<> fast path.  Image borders are handled in the same kernel:
// left/right edges by per-element fix-ups (CTA-uniform flag), top/bottom by
// loading clamped (or constant) rows and recomputing H at the clamped centre
// row (== H(clamp(yy)), per-stage semantics).  Same per-output fp32 operation
// order as every other Harris variant (bit-identical).
#pragma once
#include <cuda.h>

#include "harris_stream.cuh"

#ifndef ICL_HSHFL_MINB
#define ICL_HSHFL_MINB (16 / NW)
#endif

namespace icl {

// Row segment of this CTA.  The last segment (bottom border, general path) is launched first: in a
// grid of about one wave (e.g. BASELINE configs[1], 2048^2) the slower border CTAs then run beside
// the interior ones instead of forming the tail.
__device__ __forceinline__ int hshfl_segment() {
  return blockIdx.y == 0 ? (int)gridDim.y - 1 : (int)blockIdx.y - 1;
}

template <int B, int NW>
__device__ __forceinline__ void harris_shfl_fast(const HarrisParams& p, int S, float* smem) {
  constexpr int A = B / 2;
  constexpr int BB = B - 1 - A;
  static_assert(A <= 2 && BB <= 2, "shuffle halo covers windows up to 5x5");
  constexpr int NT = 32 * NW;
  constexpr int HP = 8;
  constexpr int TW = 120 * NW;
  constexpr int ROWLEN = TW + 2 * HP;
  constexpr int NSLOT = ROWLEN / 4;
  constexpr int RB = HarFastGeom<B>::RB, NBLKS = HarFastGeom<B>::NBLKS, NSR = HarFastGeom<B>::NSR;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TW;
  const int ly0 = hshfl_segment() * S;
  const int ly1 = min(ly0 + S, p.dst.H);
  const int g0 = p.dst.y0 + ly0;
  const int NY = (ly1 - ly0) + B - 1;
  const int NL = NY + 2;
  const int NBI = (NY + RB - 1) / RB;
  const int NBL = (NL + RB - 1) / RB;
  const int W = p.src.W;
  const int Hg = p.src.Hg;
  const bool clampb = p.src.border == kBorderClamp;
  // left/right image edge inside this strip: per-element boundary work (uniform flag)
  const bool edge = x0 - HP < 0 || x0 + TW + HP > W;
  const float* rowb = src_row(p.src, b, g0 - A - 1);  // input row of load index 0, column 0
  const int64_t spitch = p.src.pitch >> 2;

  auto load_block = [&](int m) {
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const int kl = m * RB + u;
      if (kl < NL) {
        float* st = smem + (kl % NSR) * ROWLEN;
        int gi = g0 - A - 1 + kl;
        if (gi < 0 || gi >= Hg) {  // input row outside the image (top / bottom segments only)
          if (!clampb) {
            for (int c = tid; c < ROWLEN; c += NT) st[c] = p.src.cval;
            continue;
          }
          gi = clampi(gi, 0, Hg - 1);
        }
        const float* row = rowb + (int64_t)(gi - (g0 - A - 1)) * spitch;
        for (int s = tid; s < NSLOT; s += NT) {
          const int xs = x0 - HP + 4 * s;
          if (!edge) {
            cp_async16(st + 4 * s, row + xs, 16);
          } else {  // zero-fill outside [0, W); fixed below (Fig. 3)
            const int nb = (xs < 0) ? 0 : min(max(W - xs, 0), 4) * 4;
            cp_async16(st + 4 * s, nb ? (const void*)(row + xs) : (const void*)row, nb);
          }
        }
      }
    }
  };
  // Input boundary of the halo columns outside [0, W) of load block m.
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
  for (int m = 0; m < NBLKS - 1; ++m) {
    if (m < NBL) load_block(m);
    cp_async_commit();
  }

  // own columns: xl .. xl+3, xl = x0 + 120*warp + 4*(lane-1); smem index of xl:
  const int xl = x0 + 120 * warp + 4 * (lane - 1);
  const int si = xl - (x0 - HP);
  const bool emit = lane >= 1 && lane <= 30 && xl < W;
  // a warp whose columns (and left halo lane) all lie right of the image produces nothing: it only
  // helps load the ring (right edge strip: e.g. 16 of 240 columns in the image at W = 4096)
  const bool warp_live = x0 + 120 * warp - 4 < W;
  // lanes of this warp owning image columns 0 and W-1 (for the dx/dy boundary)
  const int xw = x0 + 120 * warp - 4;  // first column of lane 0
  const int ll = (0 - xw) >> 2, el = (0 - xw) & 3;
  const int lr = (W - 1 - xw) >> 2, er = (W - 1 - xw) & 3;
  float2 hr2[B][4];
  float hrxy[B][4];
  float* drow = dst_row(p.dst, b, ly0);
  const int64_t dpitch = p.dst.pitch >> 2;
  char* mrow = p.mask ? p.mask + (int64_t)b * p.mbstride + (int64_t)ly0 * p.mpitch : nullptr;

#pragma unroll 1
  for (int i = 0; i < NBI; ++i) {
    cp_async_wait<NBLKS - 3>();
    __syncthreads();
    if (edge) {  // rows of load blocks i (first time only) and i+1 become visible now
      if (i == 0) fix_block(0);
      if (i + 1 < NBL) fix_block(i + 1);
      __syncthreads();
    }
    if (i + NBLKS - 1 < NBL) load_block(i + NBLKS - 1);
    cp_async_commit();
    const int base = (i % NBLKS) * RB;
    if (!warp_live) continue;
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      const int step = i * RB + u;
      if (step < NY) {
        // H-row yy outside the image: clamp -> recompute H at r = clamp(yy) from the
        // same smem rows (== H(clamp(yy)), per-stage semantics); constant -> 0 below.
        const int yy = g0 - A + step;
        const int dz = yy < 0 ? -yy : (yy >= Hg ? (Hg - 1) - yy : 0);
        // columns xl-1 .. xl+4 of the three input rows (index c+1 <-> column xl+c)
        float in[3][6];
#pragma unroll
        for (int rr = 0; rr < 3; ++rr) {
          int sr = base + u + rr + dz;
          if (sr >= NSR) sr -= NSR;
          if (sr < 0) sr += NSR;
          const float* st = smem + sr * ROWLEN + si;
          const float4 w = *reinterpret_cast<const float4*>(st);
          // columns xl-1 / xl+4 belong to lanes -1 / +1 (lanes 0 / 31 get junk there,
          // which only feeds their own non-emitted, non-shared columns)
          in[rr][0] = __shfl_up_sync(0xffffffffu, w.w, 1);
          in[rr][1] = w.x; in[rr][2] = w.y; in[rr][3] = w.z; in[rr][4] = w.w;
          in[rr][5] = __shfl_down_sync(0xffffffffu, w.x, 1);
        }
        float vd[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) vd[c] = __fsub_rn(in[2][c], in[0][c]);
        // g[j] = (dx, dy) of column xl-2+j, j = 0..7 (own columns j = 2..5)
        float2 g[8];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float h0 = __fsub_rn(in[0][c + 2], in[0][c]);
          const float h1 = __fsub_rn(in[1][c + 2], in[1][c]);
          const float h2 = __fsub_rn(in[2][c + 2], in[2][c]);
          g[c + 2].x = __fmaf_rn(2.0f, h1, __fadd_rn(h0, h2));
          g[c + 2].y = __fmaf_rn(2.0f, vd[c + 1], __fadd_rn(vd[c], vd[c + 2]));
        }
        if (edge) {  // per-stage boundary of dx/dy: outside [0, W) -> dx(clamp(q)) or 0
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
          if (emit) {
            if (xl + 3 < W) {
              st_cs4(drow + xl, make_float4(R[0], R[1], R[2], R[3]));
              if (mrow)
                *reinterpret_cast<uchar4*>(mrow + xl) =
                    make_uchar4(R[0] > p.threshold, R[1] > p.threshold, R[2] > p.threshold, R[3] > p.threshold);
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (xl + q < W) {
                  drow[xl + q] = R[q];
                  if (mrow) mrow[xl + q] = R[q] > p.threshold ? 1 : 0;
                }
            }
          }
          drow += dpitch;
          if (mrow) mrow += p.mpitch;
        }
      }
    }
  }
  cp_async_wait<0>();
}

// Interior CTAs (strip and all its input rows inside the image: no dz, no
// edge fix-ups) -- the same FP32 operations as harris_shfl_fast with all
// index work hoisted: the smem ring carries two mirror rows after its last
// row (ring rows 0 and 1 are also written at NSR and NSR+1), so the three
// input rows of a step are base + (u + rr) with compile-time offsets; the
// loader walks a row pointer by the pitch; every emitting lane stores a full
// float4.  Bit-identical to the general path.
// EDGE: the strip touches the left / right image edge (its rows are still inside the image): the
// loader zero-fills columns outside [0, W), fix_block applies the input boundary there (mirror rows
// included), dx/dy outside [0, W) take the per-stage boundary, and stores are guarded -- the
// general path's column logic without its row logic.
// TMA (the "shfl_tma_*" variants, NW <= 2): each block of RB ring rows arrives as ONE
// cp.async.bulk.tensor box (tm_blk: ROWLEN x RB) issued by thread 0 -- plus a 2-row box (tm_mir)
// for the mirror rows when the block lands in ring slot 0 -- completing on that slot's mbarrier;
// columns outside the image are zero-filled by the TMA unit exactly as by the zero-byte cp.async.
template <int B, int NW, bool EDGE, bool TMA = false>
__device__ __forceinline__ void harris_shfl_interior(const HarrisParams& p, int S, float* smem,
                                                     const CUtensorMap* tm_blk = nullptr,
                                                     const CUtensorMap* tm_mir = nullptr,
                                                     uint64_t* bars = nullptr) {
  constexpr int A = B / 2;
  constexpr int BB = B - 1 - A;
  constexpr int NT = 32 * NW;
  constexpr int HP = 8;
  constexpr int TW = 120 * NW;
  constexpr int ROWLEN = TW + 2 * HP;
  constexpr int NSLOT = ROWLEN / 4;
  constexpr int RB = HarFastGeom<B>::RB, NBLKS = HarFastGeom<B>::NBLKS, NSR = HarFastGeom<B>::NSR;
  static_assert(RB >= 2, "mirror rows cover the two rows a step reads past its block");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TW;
  const int ly0 = hshfl_segment() * S;
  const int ly1 = min(ly0 + S, p.dst.H);
  const int g0 = p.dst.y0 + ly0;
  const int NY = (ly1 - ly0) + B - 1;
  const int NL = NY + 2;
  const int NBI = (NY + RB - 1) / RB;
  const int NBL = (NL + RB - 1) / RB;
  const int64_t spitch = p.src.pitch >> 2;
  const bool loader = tid < NSLOT;
  const int W = p.src.W;
  const int xs = x0 - HP + 4 * tid;  // first column of this loader slot
  // EDGE: bytes of the slot inside [0, W) (zero-filled beyond), from an in-row address
  const int nb = !EDGE ? 16 : (xs < 0 ? 0 : min(max(W - xs, 0), 4) * 4);
  const float* gsrc = src_row(p.src, b, g0 - A - 1) + (EDGE && nb == 0 ? 0 : xs);
  float* sdst = smem + 4 * tid;

  // a one-warp CTA (NW = 1) has more 16-byte slots per row than threads: lanes 0..NSLOT-NT-1 also
  // load a second slot
  constexpr bool TWO_SLOTS = NSLOT > NT;
  static_assert(NSLOT <= 2 * NT, "at most two loader slots per thread");
  const int tid2 = tid + NT;
  const bool loader2 = TWO_SLOTS && tid2 < NSLOT;
  const int xs2 = x0 - HP + 4 * tid2;
  const int nb2 = !EDGE ? 16 : (xs2 < 0 ? 0 : min(max(W - xs2, 0), 4) * 4);
  const float* gsrc2 = src_row(p.src, b, g0 - A - 1) + (EDGE && nb2 == 0 ? 0 : xs2);
  float* sdst2 = smem + 4 * tid2;

  const int trow0 = g0 - A - 1 - p.src.y0;  // band-buffer row of load index 0
  auto load_block = [&](int m) {
    if constexpr (TMA) {
      if (tid == 0) {
        const int r0 = (m % NBLKS) * RB;
        uint64_t* bar = &bars[m % NBLKS];
        mbar_arrive_expect_tx(bar, (uint32_t)((RB + (r0 == 0 ? 2 : 0)) * ROWLEN * sizeof(float)));
        tma_load_3d(smem + r0 * ROWLEN, tm_blk, x0 - HP, trow0 + m * RB, b, bar);
        if (r0 == 0) tma_load_3d(smem + NSR * ROWLEN, tm_mir, x0 - HP, trow0 + m * RB, b, bar);  // mirror
      }
      return;
    }
    if (!loader) return;
    const float* g = gsrc + (int64_t)(m * RB) * spitch;
    const float* g2 = gsrc2 + (int64_t)(m * RB) * spitch;
    const int r0 = (m % NBLKS) * RB;
#pragma unroll
    for (int u = 0; u < RB; ++u) {
      if (m * RB + u < NL) {
        cp_async16(sdst + (r0 + u) * ROWLEN, g, nb);
        if (u < 2 && r0 == 0) cp_async16(sdst + (NSR + u) * ROWLEN, g, nb);  // mirror
        if (TWO_SLOTS && loader2) {
          cp_async16(sdst2 + (r0 + u) * ROWLEN, g2, nb2);
          if (u < 2 && r0 == 0) cp_async16(sdst2 + (NSR + u) * ROWLEN, g2, nb2);
        }
      }
      g += spitch;
      g2 += spitch;
    }
  };
  // EDGE: input boundary of the halo columns outside [0, W) of load block m (and of its mirror rows)
  const bool clampb = p.src.border == kBorderClamp;
  auto fix_block = [&](int m) {
    for (int u = 0; u < RB; ++u) {
      const int kl = m * RB + u;
      if (kl >= NL) break;
      const int rr = kl % NSR;
      for (int mirror = 0; mirror < (rr < 2 ? 2 : 1); ++mirror) {
        float* st = smem + (mirror ? NSR + rr : rr) * ROWLEN;
        const int il = HP - x0, ir = (W - 1) - x0 + HP;
        const float vl = (il >= 0 && il < ROWLEN) ? st[il] : 0.0f;
        const float vr = (ir >= 0 && ir < ROWLEN) ? st[ir] : 0.0f;
        for (int c = tid; c < ROWLEN; c += NT) {
          const int xe = x0 - HP + c;
          if (xe < 0) st[c] = clampb ? vl : p.src.cval;
          else if (xe >= W) st[c] = clampb ? vr : p.src.cval;
        }
      }
    }
  };
  if constexpr (TMA) {
    if (tid == 0) {
#pragma unroll
      for (int m = 0; m < NBLKS; ++m) mbar_init(&bars[m], 1);
      mbar_fence_init();
    }
    __syncthreads();
  }
  for (int m = 0; m < NBLKS - 1; ++m) {
    if (m < NBL) load_block(m);
    if constexpr (!TMA) cp_async_commit();
  }

  const int xl = x0 + 120 * warp + 4 * (lane - 1);
  const float* stb = smem + (xl - (x0 - HP));
  const bool emit = lane >= 1 && lane <= 30 && (!EDGE || xl < W);
  const bool warp_live = !EDGE || x0 + 120 * warp - 4 < W;  // (see harris_shfl_fast)
  // lanes of this warp owning image columns 0 and W-1 (for the dx/dy boundary)
  const int xw = x0 + 120 * warp - 4;
  const int ll = (0 - xw) >> 2, el = (0 - xw) & 3;
  const int lr = (W - 1 - xw) >> 2, er = (W - 1 - xw) & 3;
  // running vertical window sums instead of a ring of B H-rows: when H-row n arrives, the
  // oldest chain completes output n-B+1 (c[0] + h), the others take h as their next term and
  // h starts a new chain -- every output is summed oldest row first, the ring's order
  // Sxy chains of the output pairs (q = 2m, 2m+1) share float2 lanes (FADD2): the same per-lane adds
  constexpr int NC = B > 1 ? B - 1 : 1;
  float2 c2[NC][4];
  float2 cxy[NC][2];
#pragma unroll
  for (int k = 0; k < NC; ++k) {  // (read only by outputs that are never emitted)
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
    if constexpr (TMA) {  // blocks i and i+1 (a step reads up to two rows past its block)
      mbar_wait(&bars[i % NBLKS], (uint32_t)((i / NBLKS) & 1));
      if (i + 1 < NBL) mbar_wait(&bars[(i + 1) % NBLKS], (uint32_t)(((i + 1) / NBLKS) & 1));
    } else {
      cp_async_wait<NBLKS - 3>();
    }
    __syncthreads();
    if (EDGE) {  // rows of load blocks i (first time only) and i+1 become visible now
      if (i == 0) fix_block(0);
      if (i + 1 < NBL) fix_block(i + 1);
      __syncthreads();
    }
    if (i + NBLKS - 1 < NBL) load_block(i + NBLKS - 1);
    if constexpr (!TMA) cp_async_commit();
    if (!warp_live) continue;
    const float* sb = stb + (i % NBLKS) * RB * ROWLEN;
#pragma unroll 1
    for (int u = 0; u < RB; ++u) {
      const int step = i * RB + u;
      if (step < NY) {
        // columns xl-1 .. xl+4 of the three rows; the differences of the two middle column pairs
        // run as FADD2 on the aligned halves of the LDS.128 (same per-lane subtractions)
        float4 w[3];
        float il[3], ir[3];
        float hd[3][4];
#pragma unroll
        for (int rr = 0; rr < 3; ++rr) {
          w[rr] = *reinterpret_cast<const float4*>(sb + (u + rr) * ROWLEN);
          il[rr] = __shfl_up_sync(0xffffffffu, w[rr].w, 1);    // column xl-1
          ir[rr] = __shfl_down_sync(0xffffffffu, w[rr].x, 1);  // column xl+4
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
        if (EDGE) {  // per-stage boundary of dx/dy: outside [0, W) -> dx(clamp(q)) or 0
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
        float2 h2[4];
        float2 hxy[2];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float2 hxxyy = make_float2(0.0f, 0.0f);
          float hh = 0.0f;
#pragma unroll
          for (int t = -A; t <= BB; ++t) {
            const float2 gg = g[2 + q + t];
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
            s2o[q] = __fadd2_rn(c2[0][q], h2[q]);  // completes output row step-B+1
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
          float R[4];
          R[0] = harris_R(s2o[0].x, sxyo[0].x, s2o[0].y, p.k);
          R[1] = harris_R(s2o[1].x, sxyo[0].y, s2o[1].y, p.k);
          R[2] = harris_R(s2o[2].x, sxyo[1].x, s2o[2].y, p.k);
          R[3] = harris_R(s2o[3].x, sxyo[1].y, s2o[3].y, p.k);
          if (emit) {
            if (!EDGE || xl + 3 < W) {
              st_cs4(drow, make_float4(R[0], R[1], R[2], R[3]));
              if (has_mask)
                *reinterpret_cast<uchar4*>(mrow) =
                    make_uchar4(R[0] > p.threshold, R[1] > p.threshold, R[2] > p.threshold, R[3] > p.threshold);
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (xl + q < W) {
                  drow[q] = R[q];
                  if (has_mask) mrow[q] = R[q] > p.threshold ? 1 : 0;
                }
            }
          }
          drow += dpitch;
          mrow += has_mask ? p.mpitch : 0;
        }
      }
    }
  }
  if constexpr (TMA) {  // boxes issued past the last computed block land before the CTA exits
    for (int m = NBI + 1; m < NBL; ++m) mbar_wait(&bars[m % NBLKS], (uint32_t)((m / NBLKS) & 1));
  } else {
    cp_async_wait<0>();
  }
}

template <int B, int NW>
__global__ void __launch_bounds__(32 * NW, ICL_HSHFL_MINB) harris_shfl(HarrisParams p, int S) {
  extern __shared__ __align__(16) float smem[];
  constexpr int TW = 120 * NW, HP = 8, A = B / 2, BB = B - 1 - A;
  const int x0 = blockIdx.x * TW, ly0 = hshfl_segment() * S;
  const int ly1 = min(ly0 + S, p.dst.H);
  const int g0 = p.dst.y0 + ly0;
  // every input row (g0-A-1 .. last output row + BB + 1) and column inside the image
  const bool interior = x0 - HP >= 0 && x0 + TW + HP <= p.src.W && g0 - A - 1 >= 0 &&
                        p.dst.y0 + ly1 + BB + 1 <= p.src.Hg;
  // rows inside the image: the interior path (with the column boundary logic on the edge strips)
  const bool rows_in = g0 - A - 1 >= 0 && p.dst.y0 + ly1 + BB + 1 <= p.src.Hg;
  if (interior) harris_shfl_interior<B, NW, false>(p, S, smem);
  else if (rows_in) harris_shfl_interior<B, NW, true>(p, S, smem);
  else harris_shfl_fast<B, NW>(p, S, smem);
}

// the "shfl_tma_*" variants: the interior paths fed by TMA boxes (NW <= 2: a ring row of 120*NW + 16
// columns fits one box); the general path (top / bottom segments) keeps the per-thread loader
template <int B, int NW>
__global__ void __launch_bounds__(32 * NW, ICL_HSHFL_MINB) harris_shfl_tma(HarrisParams p, int S,
                                                                            const __grid_constant__ CUtensorMap tm_blk,
                                                                            const __grid_constant__ CUtensorMap tm_mir) {
  extern __shared__ __align__(128) float hsmem_tma[];  // TMA destinations: 128-byte aligned ring
  __shared__ __align__(8) uint64_t bars[HarFastGeom<B>::NBLKS];
  float* smem = hsmem_tma;
  constexpr int TW = 120 * NW, HP = 8, A = B / 2, BB = B - 1 - A;
  const int x0 = blockIdx.x * TW, ly0 = hshfl_segment() * S;
  const int ly1 = min(ly0 + S, p.dst.H);
  const int g0 = p.dst.y0 + ly0;
  const bool interior = x0 - HP >= 0 && x0 + TW + HP <= p.src.W && g0 - A - 1 >= 0 &&
                        p.dst.y0 + ly1 + BB + 1 <= p.src.Hg;
  const bool rows_in = g0 - A - 1 >= 0 && p.dst.y0 + ly1 + BB + 1 <= p.src.Hg;
  if (interior) harris_shfl_interior<B, NW, false, true>(p, S, smem, &tm_blk, &tm_mir, bars);
  else if (rows_in) harris_shfl_interior<B, NW, true, true>(p, S, smem, &tm_blk, &tm_mir, bars);
  else harris_shfl_fast<B, NW>(p, S, smem);
}

bool make_view_tmap(const SrcView& src, int batch, int box_w, int box_h, CUtensorMap* map);

template <int B, int NW>
static inline cudaError_t launch_hshfl_tma(const HarrisParams& p, int batch, int S, cudaStream_t s) {
  constexpr int TW = 120 * NW;
  constexpr int ROWLEN = TW + 16;
  static_assert(ROWLEN <= 256, "one tensor box per ring row");
  const size_t smem = (size_t)(HarFastGeom<B>::NSR + 2) * ROWLEN * sizeof(float);  // + 2 mirror rows
  CUtensorMap mb, mm;
  if (!make_view_tmap(p.src, batch, ROWLEN, HarFastGeom<B>::RB, &mb) || !make_view_tmap(p.src, batch, ROWLEN, 2, &mm))
    return cudaErrorNotSupported;
  auto kern = harris_shfl_tma<B, NW>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grd((p.src.W + TW - 1) / TW, (p.dst.H + S - 1) / S, batch);
  kern<<<grd, 32 * NW, smem, s>>>(p, S, mb, mm);
  count_launch();
  return cudaGetLastError();
}

template <int NW>
cudaError_t dispatch_hshfl_tma(const HarrisParams& p, int batch, int S, cudaStream_t s) {
  switch (p.block) {
    case 1: return launch_hshfl_tma<1, NW>(p, batch, S, s);
    case 2: return launch_hshfl_tma<2, NW>(p, batch, S, s);
    case 3: return launch_hshfl_tma<3, NW>(p, batch, S, s);
    case 4: return launch_hshfl_tma<4, NW>(p, batch, S, s);
    case 5: return launch_hshfl_tma<5, NW>(p, batch, S, s);
    default: return cudaErrorInvalidValue;
  }
}

template <int B, int NW>
static inline cudaError_t launch_hshfl(const HarrisParams& p, int batch, int S, cudaStream_t s) {
  constexpr int TW = 120 * NW;
  constexpr int ROWLEN = TW + 16;
  const size_t smem = (size_t)(HarFastGeom<B>::NSR + 2) * ROWLEN * sizeof(float);  // + 2 mirror rows
  auto kern = harris_shfl<B, NW>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grd((p.src.W + TW - 1) / TW, (p.dst.H + S - 1) / S, batch);
  kern<<<grd, 32 * NW, smem, s>>>(p, S);
  count_launch();
  return cudaGetLastError();
}

template <int NW>
cudaError_t dispatch_hshfl(const HarrisParams& p, int batch, int S, cudaStream_t s) {
  switch (p.block) {
    case 1: return launch_hshfl<1, NW>(p, batch, S, s);
    case 2: return launch_hshfl<2, NW>(p, batch, S, s);
    case 3: return launch_hshfl<3, NW>(p, batch, S, s);
    case 4: return launch_hshfl<4, NW>(p, batch, S, s);
    case 5: return launch_hshfl<5, NW>(p, batch, S, s);
    default: return cudaErrorInvalidValue;  // B = 6, 7 need a wider shuffle halo
  }
}

}  // namespace icl
