// sepconv_stream.cuh -- the fused streaming sepconv kernel template and its
// launch helpers; instantiated per CTA width in sepconv_nt*.cu (parallel build).
#pragma once
#include <cuda.h>

#include <type_traits>

#include "common.cuh"
#include "internal.h"

namespace icl {

struct SepParams {
  SrcView src;
  DstView dst;
  int rx, ry;
  float fx[2 * kMaxRadius + 1];
  float gy[2 * kMaxRadius + 1];
  // tap pairs (fx[i], fx[i-1]) for two adjacent outputs fed by one input element (FFMA2 with a
  // broadcast input); i = 1..2R used -- the first / last element of a pair runs as scalar FFMA
  float2 fxp[2 * kMaxRadius + 2];
};

// --------------------------------------------------------------------------
// Variant family "stream<R,NT,VEC>": fused single pass (A20).  A CTA owns a
// column strip of TW = 4*NT pixels and a segment of S output rows.  It
// streams the S + 2R input rows of its strip (plus HP halo columns on each
// side) top-down through an NS-stage cp.async ring in shared memory (the
// paper's "local memory" staging, Fig. 5, made a pipeline);
// each thread computes the row pass for its 4 columns ("blocked" mapping,
// float4) into a register ring of 2R+1 intermediate rows and emits one
// output row per input row.  HBM traffic ~= 8 B/px + vertical halo 2R/S.
// VEC=4: 16-byte cp.async (needs 16B-aligned data/pitch); VEC=1: 4-byte.
// --------------------------------------------------------------------------
template <int R>
struct SepGeom {
  static constexpr int HP = ((R + 3) / 4) * 4;  // halo columns, padded to float4
  static constexpr int P = 2 * R + 1;           // ring depth
};

// Rows per pipeline block (a multiple of the ring period P, >= 4) and blocks
// of shared memory (NBLK-1 blocks in flight while one is computed).
template <int R>
struct StreamGeom {
  static constexpr int P = SepGeom<R>::P;
  static constexpr int RB = P * ((4 + P - 1) / P);
  static constexpr int NBLK = RB <= 8 ? 3 : 2;
  static constexpr int NSR = RB * NBLK;  // rows of shared memory
  // floats per block slot for a row length L, padded to 128 bytes (a TMA tile destination)
  static constexpr int blk(int L) { return ((RB * L * 4 + 127) / 128) * 128 / 4; }
};


// TMA (round 2, the "tma_*" variants, NT = 32: a 144-column row fits one tensor box): interior
// CTAs stage each block of RB input rows with ONE cp.async.bulk.tensor issued by thread 0 (a
// 144 x RB x 1 box of the source's tensor map -- rows past the band buffer are zero-filled by the
// TMA unit, never read from memory) and wait on that block's mbarrier instead of per-thread
// cp.async groups; border CTAs keep the per-thread loader.  Same arithmetic (bit-identical).
template <int R, int NT, int VEC, bool TMA = false>
__device__ __forceinline__ void sep_stream_body(const SepParams& p, int S, const CUtensorMap* tmap) {
  constexpr int HP = SepGeom<R>::HP;
  constexpr int P = SepGeom<R>::P;
  constexpr int RB = StreamGeom<R>::RB, NBLK = StreamGeom<R>::NBLK, NSR = StreamGeom<R>::NSR;
  constexpr int TW = 4 * NT;
  constexpr int ROWLEN = TW + 2 * HP;
  constexpr int NSLOT = ROWLEN / 4;
  extern __shared__ __align__(128) float smem[];
  constexpr int BLKF = StreamGeom<R>::blk(ROWLEN);  // floats per block slot (128-byte multiple)
  // smem row of input row k: block slot (k / RB) % NBLK, row k % RB inside it
  auto srow = [&](int k) { return smem + ((k / RB) % NBLK) * BLKF + (k % RB) * ROWLEN; };

  const int tid = threadIdx.x;
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TW;
  const int ly0 = blockIdx.y * S;
  const int ly1 = min(ly0 + S, p.dst.H);
  const int g0 = p.dst.y0 + ly0;
  const int NI = (ly1 - ly0) + 2 * R;
  const int NB = (NI + RB - 1) / RB;
  const int W = p.src.W;
  const int Hg = p.src.Hg;
  const bool clampb = p.src.border == kBorderClamp;
  const bool edge = (x0 - HP < 0) || (x0 + TW + HP > W);
  const bool vint = (g0 - R >= 0) && (g0 - R + NI <= Hg);
  const bool fast = !edge && vint && VEC == 4;  // no boundary work anywhere in this CTA
  const bool tma = TMA && fast;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NBLK * BLKF);  // NBLK mbarriers (TMA)
  if (TMA) {
    if (tid == 0) {
      for (int i = 0; i < NBLK; ++i) mbar_init(&bars[i], 1);
      mbar_fence_init();
    }
    __syncthreads();
  }

  // fast-path copy descriptors (columns never change across rows)
  const float* row0 = src_row(p.src, b, fast ? g0 - R : 0);  // row of input k = 0
  const int s1 = tid + NT;
  const int c0 = x0 - HP + 4 * tid, c1 = x0 - HP + 4 * s1;

  // Issue the loads of rows [kb, kb + RB) into their smem rows (k % NSR).
  auto load_block = [&](int kb) {
    if (tma) {
      if (tid == 0) {
        uint64_t* bar = &bars[(kb / RB) % NBLK];
        mbar_arrive_expect_tx(bar, (uint32_t)(RB * ROWLEN * sizeof(float)));
        tma_load_3d(srow(kb), tmap, x0 - HP, g0 - R + kb - p.src.y0, b, bar);
      }
      return;
    }
    if (fast) {
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        const int k = kb + u;
        if (k < NI) {
          float* st = srow(k);
          const float* row = row0 + (int64_t)k * (p.src.pitch >> 2);
          cp_async16(st + 4 * tid, row + c0, 16);
          if (s1 < NSLOT) cp_async16(st + 4 * s1, row + c1, 16);
        }
      }
      return;
    }
    for (int u = 0; u < RB; ++u) {
      const int k = kb + u;
      if (k >= NI) break;
      float* st = srow(k);
      int gi = g0 - R + k;
      if (gi < 0 || gi >= Hg) {
        if (!clampb) {  // constant border: a full row of c
          for (int s = tid; s < NSLOT; s += NT)
            reinterpret_cast<float4*>(st)[s] = make_float4(p.src.cval, p.src.cval, p.src.cval, p.src.cval);
          continue;
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
    }
  };
  // Boundary fix-up of the halo columns outside [0, W) of rows [kb, kb+RB).
  auto fix_block = [&](int kb) {
    const int il = HP - x0;
    const int ir = (W - 1) - x0 + HP;
    for (int u = 0; u < RB; ++u) {
      const int k = kb + u;
      if (k >= NI) break;
      float* st = srow(k);
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
    }
  };

  // Prologue: blocks 0 .. NBLK-2 in flight (one cp.async group per block).
  for (int i = 0; i < NBLK - 1; ++i) {
    if (i < NB) load_block(i * RB);
    cp_async_commit();
  }

  float4 ring[P];
  const int xc = x0 + 4 * tid;
  float* drow = dst_row(p.dst, b, ly0);
  const int64_t dpitch = p.dst.pitch >> 2;

#pragma unroll 1
  for (int i = 0; i < NB; ++i) {
    if (tma) mbar_wait(&bars[i % NBLK], (uint32_t)((i / NBLK) & 1));  // block i's TMA landed
    else cp_async_wait<NBLK - 2>();  // block i complete
    __syncthreads();            // ... for every thread; block i-1's rows are free
    if (edge) {
      fix_block(i * RB);
      __syncthreads();
    }
    if (i + NBLK - 1 < NB) load_block((i + NBLK - 1) * RB);
    cp_async_commit();
    // a block whose RB steps all exist and all emit, in a strip away from the image edges, runs
    // as ONE basic block (no per-step branches), so the compiler can overlap the row pass of a
    // step with the column chain of the previous one; the first / last blocks and edge strips keep
    // the checked form.  Same operations in the same order (bit-identical).  Only for R <= 4: above,
    // the duplicated block body costs more in instruction fetch than the overlap gains (16384^2:
    // R = 4 0.359 vs 0.387 ms; R = 6 / 8 / 10 0.468 / 0.636 / 0.877 vs 0.433 / 0.574 / 0.771 ms).
    constexpr bool kFastBlocks = R <= 4;
    constexpr bool kPredBlocks = R >= 5;
    const bool full = kFastBlocks && VEC == 4 && !edge && (i + 1) * RB <= NI && i * RB >= 2 * R;
    auto step = [&](const int u, const int k, auto fast_tag) {
      constexpr bool FAST = decltype(fast_tag)::value;

        const float* st = srow(k);
        float v[4 + 2 * HP];
#pragma unroll
        for (int q = 0; q < (4 + 2 * HP) / 4; ++q) {
          const float4 w = reinterpret_cast<const float4*>(st + 4 * tid)[q];
          v[4 * q] = w.x; v[4 * q + 1] = w.y; v[4 * q + 2] = w.z; v[4 * q + 3] = w.w;
        }
        // row pass, two outputs per FFMA2: input v[k] feeds output c with tap k-c and output c+1
        // with tap k-c-1 -- the tap pair (fx[i], fx[i-1]) from the parameter bank, the input
        // broadcast.  Each lane runs exactly its output's FMA chain over i = 0..2R (from 0.0f), so
        // the result is the scalar chain's, bit for bit; the chain ends run as scalar FFMAs.
        float2 t01, t23;
        {
          constexpr int B0 = HP - R;
          t01.x = __fmaf_rn(p.fx[0], v[B0], 0.0f);
          t23.x = __fmaf_rn(p.fx[0], v[B0 + 2], 0.0f);
          t01.y = 0.0f;
          t23.y = 0.0f;
          if (R == 0) {
            t01.y = __fmaf_rn(p.fx[0], v[B0 + 1], 0.0f);
            t23.y = __fmaf_rn(p.fx[0], v[B0 + 3], 0.0f);
          } else {
#pragma unroll
            for (int i = 1; i <= 2 * R; ++i) {
              const float va = v[B0 + i], vb = v[B0 + 2 + i];
              t01 = __ffma2_rn(make_float2(va, va), p.fxp[i], t01);
              t23 = __ffma2_rn(make_float2(vb, vb), p.fxp[i], t23);
            }
            t01.y = __fmaf_rn(p.fx[2 * R], v[B0 + 2 * R + 1], t01.y);
            t23.y = __fmaf_rn(p.fx[2 * R], v[B0 + 2 * R + 3], t23.y);
          }
        }
        ring[u % P] = make_float4(t01.x, t01.y, t23.x, t23.y);
        if constexpr (kPredBlocks) {
          // R >= 5: the column pass for every step (a partly filled ring before step 2R only
          // feeds discarded outputs) and emission by predicate, so every block is one basic block
          // without duplicating the body (16384^2 R = 5 / 6 / 7 / 8 / 9 / 10: 0.397 / 0.427 /
          // 0.476 / 0.509 / 0.625 / 0.730 vs 0.408 / 0.441 / 0.497 / 0.587 / 0.708 / 0.778 ms)
          const bool em = FAST || (k >= 2 * R && k < NI);
          float2 o01 = make_float2(0.0f, 0.0f), o23 = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int j = 0; j < P; ++j) {
            const float4 rr = ring[(u + 1 + j) % P];
            const float2 g = make_float2(p.gy[j], p.gy[j]);
            o01 = __ffma2_rn(g, make_float2(rr.x, rr.y), o01);
            o23 = __ffma2_rn(g, make_float2(rr.z, rr.w), o23);
          }
          const float o[4] = {o01.x, o01.y, o23.x, o23.y};
          const bool v4 = FAST || (VEC == 4 && xc + 3 < W);
          if (em && v4) st_cs4(drow + xc, make_float4(o[0], o[1], o[2], o[3]));
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (!FAST && em && !v4 && xc + c < W) drow[xc + c] = o[c];
          drow += em ? dpitch : 0;
        } else {
        if (FAST || k >= 2 * R) {
          // column pass: two columns per FFMA2 (the tap broadcast), each lane its scalar chain
          float2 o01 = make_float2(0.0f, 0.0f), o23 = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int j = 0; j < P; ++j) {
            const float4 rr = ring[(u + 1 + j) % P];
            const float2 g = make_float2(p.gy[j], p.gy[j]);
            o01 = __ffma2_rn(g, make_float2(rr.x, rr.y), o01);
            o23 = __ffma2_rn(g, make_float2(rr.z, rr.w), o23);
          }
          const float o[4] = {o01.x, o01.y, o23.x, o23.y};
          if (FAST || (VEC == 4 && xc + 3 < W)) {
            st_cs4(drow + xc, make_float4(o[0], o[1], o[2], o[3]));
          } else {
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (xc + c < W) drow[xc + c] = o[c];
          }
          drow += dpitch;
        }
        }
    };
    if constexpr (kFastBlocks) {
      if (full) {
#pragma unroll
        for (int u = 0; u < RB; ++u) step(u, i * RB + u, std::true_type{});
        continue;
      }
    }
    {
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        const int k = i * RB + u;
        if (kPredBlocks || k < NI) step(u, k, std::false_type{});
      }
    }
  }
  cp_async_wait<0>();
}

template <int R, int NT, int VEC>
__global__ void __launch_bounds__(NT) sep_stream(SepParams p, int S) {
  sep_stream_body<R, NT, VEC, false>(p, S, nullptr);
}

template <int R, int NT>
__global__ void __launch_bounds__(NT) sep_stream_tma(SepParams p, int S, const __grid_constant__ CUtensorMap tmap) {
  sep_stream_body<R, NT, 4, true>(p, S, &tmap);
}
// Pipeline invariant: before block i, NBLK-1+i cp.async groups are committed
// (one per block, empty past the end), so wait_group(NBLK-2) completes block
// i while block i+1 .. stays in flight; block i+NBLK-1 is issued into the
// smem rows block i-1 used, which every thread released at this barrier.
// RB is a multiple of P, so ring slot u % P == k % P (static indices).

template <int R, int NT, int VEC>
static inline cudaError_t launch_stream_R(const SepParams& p, int batch, int S, cudaStream_t s) {
  constexpr int ROWLEN = 4 * NT + 2 * SepGeom<R>::HP;
  const size_t smem = (size_t)StreamGeom<R>::NBLK * StreamGeom<R>::blk(ROWLEN) * sizeof(float);
  auto kern = sep_stream<R, NT, VEC>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grd((p.src.W + 4 * NT - 1) / (4 * NT), (p.dst.H + S - 1) / S, batch);
  kern<<<grd, NT, smem, s>>>(p, S);
  count_launch();
  return cudaGetLastError();
}

// The source as a 3-D tensor map (x = W columns, y = the rows held locally, z = images), box
// ROWLEN x RB x 1, zero fill out of bounds (cuTensorMapEncodeTiled through the runtime's driver
// entry point: no link-time libcuda dependency).
bool make_src_tmap(const SepParams& p, int batch, int box_w, int box_h, CUtensorMap* map);

template <int R, int NT>
static inline cudaError_t launch_stream_tma_R(const SepParams& p, int batch, int S, cudaStream_t s) {
  constexpr int ROWLEN = 4 * NT + 2 * SepGeom<R>::HP;
  static_assert(ROWLEN <= 256, "one tensor box per row block");
  const size_t smem = (size_t)StreamGeom<R>::NBLK * StreamGeom<R>::blk(ROWLEN) * sizeof(float) +
                      8 * StreamGeom<R>::NBLK;
  CUtensorMap map;
  if (!make_src_tmap(p, batch, ROWLEN, StreamGeom<R>::RB, &map)) return cudaErrorNotSupported;
  auto kern = sep_stream_tma<R, NT>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grd((p.src.W + 4 * NT - 1) / (4 * NT), (p.dst.H + S - 1) / S, batch);
  kern<<<grd, NT, smem, s>>>(p, S, map);
  count_launch();
  return cudaGetLastError();
}

template <int NT>
cudaError_t dispatch_stream_tma(const SepParams& p, int R, int batch, int S, cudaStream_t s) {
  switch (R) {
#define ICL_SEPT_CASE(r) \
  case r:                \
    return launch_stream_tma_R<r, NT>(p, batch, S, s);
    ICL_SEPT_CASE(0) ICL_SEPT_CASE(1) ICL_SEPT_CASE(2) ICL_SEPT_CASE(3) ICL_SEPT_CASE(4) ICL_SEPT_CASE(5)
    ICL_SEPT_CASE(6) ICL_SEPT_CASE(7) ICL_SEPT_CASE(8) ICL_SEPT_CASE(9) ICL_SEPT_CASE(10) ICL_SEPT_CASE(11)
    ICL_SEPT_CASE(12) ICL_SEPT_CASE(13) ICL_SEPT_CASE(14) ICL_SEPT_CASE(15)
#undef ICL_SEPT_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

template <int NT, int VEC>
cudaError_t dispatch_stream(const SepParams& p, int R, int batch, int S, cudaStream_t s) {
  switch (R) {
#define ICL_SEP_CASE(r) \
  case r:               \
    return launch_stream_R<r, NT, VEC>(p, batch, S, s);
    ICL_SEP_CASE(0) ICL_SEP_CASE(1) ICL_SEP_CASE(2) ICL_SEP_CASE(3) ICL_SEP_CASE(4) ICL_SEP_CASE(5)
    ICL_SEP_CASE(6) ICL_SEP_CASE(7) ICL_SEP_CASE(8) ICL_SEP_CASE(9) ICL_SEP_CASE(10) ICL_SEP_CASE(11)
    ICL_SEP_CASE(12) ICL_SEP_CASE(13) ICL_SEP_CASE(14) ICL_SEP_CASE(15)
#undef ICL_SEP_CASE
    default:
      return cudaErrorInvalidValue;
  }
}


static inline SepParams make_sep_params(const SepCall& c, bool pad) {
  SepParams p;
  p.src = c.src;
  p.dst = c.dst;
  p.rx = c.rx;
  p.ry = c.ry;
  for (int i = 0; i < 2 * kMaxRadius + 1; ++i) { p.fx[i] = 0.0f; p.gy[i] = 0.0f; }
  if (pad) {
    const int R = c.rx > c.ry ? c.rx : c.ry;
    for (int i = 0; i < 2 * c.rx + 1; ++i) p.fx[R - c.rx + i] = c.fx[i];
    for (int j = 0; j < 2 * c.ry + 1; ++j) p.gy[R - c.ry + j] = c.gy[j];
  } else {
    for (int i = 0; i < 2 * c.rx + 1; ++i) p.fx[i] = c.fx[i];
    for (int j = 0; j < 2 * c.ry + 1; ++j) p.gy[j] = c.gy[j];
  }
  for (int i = 0; i < 2 * kMaxRadius + 2; ++i)
    p.fxp[i] = make_float2(i < 2 * kMaxRadius + 1 ? p.fx[i] : 0.0f, i >= 1 ? p.fx[i - 1] : 0.0f);
  return p;
}

}  // namespace icl
