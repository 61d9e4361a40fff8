// sepconv_tile.cu -- variant family "tile<R>" for large radii: fused separable
// convolution with both passes inside one CTA through shared memory
// (§6; local-memory staging PAPER.md:484-525; the
// Halide-style fusion of PAPER.md:701-704).
//
// The register ring of stream<R> holds 2R+1 rows of row-pass results per
// thread (124 registers at R = 15), which caps occupancy and leaves the kernel
// latency-bound for R >~ 6.  Here a CTA owns a 64x64 output tile:
//   load    input tile rows g0-R .. g0+63+R, columns x0-HP .. x0+63+HP
//           (16-byte vector loads for interior tiles; in_B per element at
//           the image border);
//   pass H  t(r, c) = fma-chain over i of fx[i] * in(r, c-R+i), 8 columns per
//           thread from an aligned 8+2HP super-window (LDS.128), consecutive
//           threads on consecutive rows (conflict-free), stored to smem;
//   pass V  out(y, c) = fma-chain over j of gy[j] * t(y+j, c), 2 columns x 8
//           rows per thread, the two columns packed in FFMA2 lanes (LDS.64).
// Same per-output fp32 operation order as every sepconv variant
// (bit-identical).  FP32 work 2(2R+1) FMA/px at ~1 smem word per FMA pair.
#include "common.cuh"
#include "internal.h"
#include "sepconv_stream.cuh"

namespace icl {

template <int R, int TH_ = 64>
struct TileGeom {
  static constexpr int TW = 64, TH = TH_, NT = 4 * TH_;  // pass V: 32 column pairs x (NT/32) runs of 8 rows
  static constexpr int HP = ((R + 3) / 4) * 4;
  static constexpr int P = 2 * R + 1;
  static constexpr int IR = TH + 2 * R;          // input / t rows
  static constexpr int IW0 = TW + 2 * HP;        // input columns
  static constexpr int IW = ((IW0 + 31) / 32) * 32 + 4;  // row stride == 4 (mod 32) words
  static constexpr int TWS = TW + 4;              // t row stride (== 4 mod 32)
  static constexpr size_t smem_bytes = (size_t)(IR * IW + IR * TWS) * sizeof(float);
};

template <int R>
__global__ void __launch_bounds__(256) sep_tile(SepParams p) {
  using G = TileGeom<R>;
  constexpr int TW = G::TW, TH = G::TH, HP = G::HP, P = G::P, IR = G::IR, IW = G::IW, IW0 = G::IW0;
  constexpr int TWS = G::TWS, NT = G::NT;
  extern __shared__ __align__(16) float smem[];
  float* In = smem;             // [IR][IW]
  float* T = smem + IR * IW;    // [IR][TWS]
  const int tid = threadIdx.x;
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TW;
  const int ly0 = blockIdx.y * TH;
  const int g0 = p.dst.y0 + ly0;
  const int W = p.src.W, Hg = p.src.Hg;
  const bool interior = x0 - HP >= 0 && x0 + TW + HP <= W && g0 - R >= 0 && g0 + TH + R <= Hg &&
                        g0 - R >= p.src.y0 && g0 + TH + R <= p.src.y0 + p.src.Hl;  // (16-byte-aligned images; rows held)

  // ---------------- load the input tile
  if (interior) {
    constexpr int NV = IW0 / 4;
    for (int i = tid; i < IR * NV; i += NT) {
      const int r = i / NV, v = i % NV;
      const float4 w = __ldg(reinterpret_cast<const float4*>(src_row(p.src, b, g0 - R + r) + (x0 - HP + 4 * v)));
      *reinterpret_cast<float4*>(In + r * IW + 4 * v) = w;
    }
  } else {
    for (int i = tid; i < IR * IW0; i += NT) {
      const int r = i / IW0, c = i % IW0;
      In[r * IW + c] = read_B(p.src, b, x0 - HP + c, g0 - R + r);
    }
  }
  __syncthreads();

  // ---------------- pass H: rows r = 0..IR-1, 8-column runs (8 per row)
  for (int item = tid; item < IR * (TW / 8); item += NT) {
    const int r = item % IR, k = item / IR;  // consecutive threads -> consecutive rows
    const float* src = In + r * IW + 8 * k;
    float v[8 + 2 * HP];
#pragma unroll
    for (int q = 0; q < (8 + 2 * HP) / 4; ++q) {
      const float4 w = reinterpret_cast<const float4*>(src)[q];
      v[4 * q] = w.x; v[4 * q + 1] = w.y; v[4 * q + 2] = w.z; v[4 * q + 3] = w.w;
    }
    float t[8];
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      float a = 0.0f;
#pragma unroll
      for (int i = 0; i < P; ++i) a = __fmaf_rn(p.fx[i], v[HP - R + o + i], a);
      t[o] = a;
    }
    float* dst = T + r * TWS + 8 * k;
    reinterpret_cast<float4*>(dst)[0] = make_float4(t[0], t[1], t[2], t[3]);
    reinterpret_cast<float4*>(dst)[1] = make_float4(t[4], t[5], t[6], t[7]);
  }
  __syncthreads();

  // ---------------- pass V: 2 columns x 8 rows per thread, FFMA2 over the column pair
  {
    const int cp = tid & 31, run = tid >> 5;  // 32 column pairs x 8 runs of 8 rows
    const float* tc = T + (8 * run) * TWS + 2 * cp;
    float2 o[8];
#pragma unroll
    for (int y = 0; y < 8; ++y) o[y] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int rr = 0; rr < 8 + 2 * R; ++rr) {
      const float2 tv = *reinterpret_cast<const float2*>(tc + rr * TWS);
#pragma unroll
      for (int y = 0; y < 8; ++y) {
        const int j = rr - y;  // tap index for output row y
        if (j >= 0 && j < P) o[y] = __ffma2_rn(make_float2(p.gy[j], p.gy[j]), tv, o[y]);
      }
    }
    const int gx = x0 + 2 * cp;
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      const int ly = ly0 + 8 * run + y;
      if (ly < p.dst.H) {
        float* drow = dst_row(p.dst, b, ly);
        if (gx + 1 < W && ((reinterpret_cast<uintptr_t>(drow + gx) & 7) == 0)) {
          *reinterpret_cast<float2*>(drow + gx) = o[y];
        } else {
          if (gx < W) drow[gx] = o[y].x;
          if (gx + 1 < W) drow[gx + 1] = o[y].y;
        }
      }
    }
  }
}

// Persistent form: grid = 2 CTAs per SM, each walks tiles t = blockIdx.x,
// blockIdx.x + gridDim.x, ...; the NEXT tile's input is prefetched with
// cp.async into a second input buffer while the current tile runs passes H/V,
// hiding the global-load latency the one-tile-per-CTA form exposes.  Same
// arithmetic (bit-identical).
// TH_ = 128 (round 2, "tile128p_v4"): 128-row tiles with 512 threads (1 CTA/SM, the same 16
// warps): the pass-H halo recompute drops from (64+2R)/64 to (128+2R)/128 (1.47 -> 1.23 at R = 15)
// and each barrier covers twice the work.
template <int R, int TH_ = 64>
struct TilePGeom {
  using G = TileGeom<R, TH_>;
  static constexpr size_t smem_bytes = (size_t)(2 * G::IR * G::IW + G::IR * G::TWS) * sizeof(float);
};

template <int R, int TH_ = 64>
__global__ void __launch_bounds__(4 * TH_, TH_ == 64 ? 2 : 1) sep_tile_p(SepParams p, int ntx, int nty, int ntiles) {
  using G = TileGeom<R, TH_>;
  constexpr int TW = G::TW, TH = G::TH, HP = G::HP, P = G::P, IR = G::IR, IW = G::IW, IW0 = G::IW0;
  constexpr int TWS = G::TWS, NT = G::NT;
  constexpr int NV = IW0 / 4;  // 16-byte vectors per input row (<= 24 for R <= 15: one lane each)
  static_assert(NV <= 32, "one warp lane per input vector");
  constexpr int NI = (IR * (TW / 8) + NT - 1) / NT;  // pass-H items per thread
  extern __shared__ __align__(16) float smem[];
  float* T = smem + 2 * IR * IW;  // input buffers at smem + k * IR * IW, k = 0, 1
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W = p.src.W, Hg = p.src.Hg;
  const int per_img = ntx * nty;

  struct Tile { int b, x0, ly0; bool interior; };
  auto tile_of = [&](int t) {
    Tile c;
    c.b = t / per_img;
    const int r = t - c.b * per_img;
    const int ty = r / ntx;
    c.ly0 = ty * TH;
    c.x0 = (r - ty * ntx) * TW;
    const int g0 = p.dst.y0 + c.ly0;
    c.interior = c.x0 - HP >= 0 && c.x0 + TW + HP <= W && g0 - R >= 0 && g0 + TH + R <= Hg &&
                 g0 - R >= p.src.y0 && g0 + TH + R <= p.src.y0 + p.src.Hl;
    return c;
  };
  // interior tile: warp w copies rows w, w+NWARP, ... ; lane v copies 16-byte vector v
  constexpr int NWARP = NT / 32;
  auto load_async = [&](const Tile& c, float* In) {
    if (lane < NV) {
      const char* g = reinterpret_cast<const char*>(src_row(p.src, c.b, p.dst.y0 + c.ly0 - R + warp) +
                                                    (c.x0 - HP + 4 * lane));
      const int64_t step = NWARP * p.src.pitch;
      uint32_t sa = smem_u32(In + warp * IW + 4 * lane);
#pragma unroll 4
      for (int r = warp; r < IR; r += NWARP) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g) : "memory");
        g += step;
        sa += NWARP * IW * sizeof(float);
      }
    }
  };
  // border tile: in_B per element (Fig. 3)
  auto load_border = [&](const Tile& c, float* In) {
    const int g0 = p.dst.y0 + c.ly0;
    for (int i = tid; i < IR * IW0; i += NT) {
      const int r = i / IW0, col = i - r * IW0;
      In[r * IW + col] = read_B(p.src, c.b, c.x0 - HP + col, g0 - R + r);
    }
  };

  // per-thread pass-H item offsets do not depend on the tile
  int hin[NI], hout[NI];
#pragma unroll
  for (int k = 0; k < NI; ++k) {
    const int item = tid + k * NT;
    const int r = item % IR, q = item / IR;  // consecutive threads -> consecutive rows
    hin[k] = r * IW + 8 * q;
    hout[k] = r * TWS + 8 * q;
  }
  const int cp = lane, run = warp;  // pass V: column pair, 8-row run
  const float* tc = T + (8 * run) * TWS + 2 * cp;

  int t = blockIdx.x;
  if (t >= ntiles) return;
  Tile cur = tile_of(t);
  if (cur.interior) load_async(cur, smem);
  else load_border(cur, smem);
  cp_async_commit();
  for (int it = 0; t < ntiles; ++it) {
    float* In = smem + (it & 1) * (IR * IW);
    float* Nx = smem + ((it & 1) ^ 1) * (IR * IW);
    cp_async_wait<0>();
    __syncthreads();  // current input visible; T and the other buffer are free
    const int tn = t + gridDim.x;
    Tile nxt = cur;
    if (tn < ntiles) {
      nxt = tile_of(tn);
      if (nxt.interior) load_async(nxt, Nx);
    }
    cp_async_commit();
    // ---------------- pass H
#pragma unroll
    for (int k = 0; k < NI; ++k) {
      if (IR * (TW / 8) % NT == 0 || k < NI - 1 || tid + k * NT < IR * (TW / 8)) {
        const float* src = In + hin[k];
        float v[8 + 2 * HP];
#pragma unroll
        for (int q = 0; q < (8 + 2 * HP) / 4; ++q) {
          const float4 w = reinterpret_cast<const float4*>(src)[q];
          v[4 * q] = w.x; v[4 * q + 1] = w.y; v[4 * q + 2] = w.z; v[4 * q + 3] = w.w;
        }
        // output columns (2m, 2m+1) share FFMA2 lanes: input element e feeds column 2m with tap
        // i = e - (HP-R) - 2m and column 2m+1 with tap i-1 -> (fx[i], fx[i-1]) x broadcast(v[e]);
        // the pair's first / last element feeds one column only (scalar FFMA).  Each lane runs
        // its own output's chain over i in order: bit-identical.
        float2 tp[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          float2 a = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int i = 0; i <= P; ++i) {
            const float ve = v[HP - R + 2 * m + i];
            if (i == 0) a.x = __fmaf_rn(p.fx[0], ve, a.x);
            else if (i == P) a.y = __fmaf_rn(p.fx[P - 1], ve, a.y);
            else a = __ffma2_rn(make_float2(ve, ve), p.fxp[i], a);
          }
          tp[m] = a;
        }
        const float tt[8] = {tp[0].x, tp[0].y, tp[1].x, tp[1].y, tp[2].x, tp[2].y, tp[3].x, tp[3].y};
        float* dst = T + hout[k];
        reinterpret_cast<float4*>(dst)[0] = make_float4(tt[0], tt[1], tt[2], tt[3]);
        reinterpret_cast<float4*>(dst)[1] = make_float4(tt[4], tt[5], tt[6], tt[7]);
      }
    }
    __syncthreads();
    // ---------------- pass V
    {
      float2 o[8];
#pragma unroll
      for (int y = 0; y < 8; ++y) o[y] = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int rr = 0; rr < 8 + 2 * R; ++rr) {
        const float2 tv = *reinterpret_cast<const float2*>(tc + rr * TWS);
#pragma unroll
        for (int y = 0; y < 8; ++y) {
          const int j = rr - y;
          if (j >= 0 && j < P) o[y] = __ffma2_rn(make_float2(p.gy[j], p.gy[j]), tv, o[y]);
        }
      }
      const int gx = cur.x0 + 2 * cp;
      const int ly = cur.ly0 + 8 * run;
      char* drow = reinterpret_cast<char*>(dst_row(p.dst, cur.b, ly) + gx);
      if (cur.x0 + TW <= W && cur.ly0 + TH <= p.dst.H) {
        // whole tile in range; a16 images => 8-byte aligned pairs
#pragma unroll
        for (int y = 0; y < 8; ++y) {
          *reinterpret_cast<float2*>(drow) = o[y];
          drow += p.dst.pitch;
        }
      } else {
#pragma unroll
        for (int y = 0; y < 8; ++y) {
          if (ly + y < p.dst.H) {
            float* d = reinterpret_cast<float*>(drow);
            if (gx + 1 < W) {
              *reinterpret_cast<float2*>(d) = o[y];
            } else if (gx < W) {
              d[0] = o[y].x;
            }
          }
          drow += p.dst.pitch;
        }
      }
    }
    // a border next tile is filled synchronously (after everyone is done with T / In)
    if (tn < ntiles && !nxt.interior) {
      __syncthreads();
      load_border(nxt, Nx);
    }
    t = tn;
    cur = nxt;
  }
  cp_async_wait<0>();
}

template <int R, int TH_ = 64>
static cudaError_t launch_tilep_R(const SepParams& p, int batch, cudaStream_t s) {
  using G = TileGeom<R, TH_>;
  constexpr size_t smem = TilePGeom<R, TH_>::smem_bytes;
  static_assert(smem <= 227 * 1024, "shared memory");
  auto kern = sep_tile_p<R, TH_>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ntx = (p.src.W + G::TW - 1) / G::TW, nty = (p.dst.H + G::TH - 1) / G::TH;
  const int ntiles = ntx * nty * batch;
  const int per_sm = TH_ == 64 ? 2 : 1;
  const int grid = ntiles < per_sm * sms ? ntiles : per_sm * sms;
  kern<<<grid, G::NT, smem, s>>>(p, ntx, nty, ntiles);
  count_launch();
  return cudaGetLastError();
}

template <int R>
static cudaError_t launch_tile_R(const SepParams& p, int batch, cudaStream_t s) {
  using G = TileGeom<R>;
  static_assert(G::smem_bytes <= 227 * 1024, "shared memory");
  auto kern = sep_tile<R>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grd((p.src.W + G::TW - 1) / G::TW, (p.dst.H + G::TH - 1) / G::TH, batch);
  kern<<<grd, G::NT, G::smem_bytes, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_sep_tile128(const SepCall& c, cudaStream_t s) {
  SepParams p = make_sep_params(c, true);
  const int R = c.rx > c.ry ? c.rx : c.ry;
  switch (R) {  // (the radii where the FP32 work, not HBM, bounds the tile kernels)
    case 7: return launch_tilep_R<7, 128>(p, c.batch, s);
    case 8: return launch_tilep_R<8, 128>(p, c.batch, s);
    case 9: return launch_tilep_R<9, 128>(p, c.batch, s);
    case 10: return launch_tilep_R<10, 128>(p, c.batch, s);
    case 11: return launch_tilep_R<11, 128>(p, c.batch, s);
    case 12: return launch_tilep_R<12, 128>(p, c.batch, s);
    case 13: return launch_tilep_R<13, 128>(p, c.batch, s);
    case 14: return launch_tilep_R<14, 128>(p, c.batch, s);
    case 15: return launch_tilep_R<15, 128>(p, c.batch, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_sep_tile(const SepCall& c, bool persistent, cudaStream_t s) {
  SepParams p = make_sep_params(c, true);
  const int R = c.rx > c.ry ? c.rx : c.ry;
  switch (R) {
#define ICL_TILE_CASE(r) \
  case r:                \
    return persistent ? launch_tilep_R<r>(p, c.batch, s) : launch_tile_R<r>(p, c.batch, s);
    ICL_TILE_CASE(0) ICL_TILE_CASE(1) ICL_TILE_CASE(2) ICL_TILE_CASE(3) ICL_TILE_CASE(4) ICL_TILE_CASE(5)
    ICL_TILE_CASE(6) ICL_TILE_CASE(7) ICL_TILE_CASE(8) ICL_TILE_CASE(9) ICL_TILE_CASE(10) ICL_TILE_CASE(11)
    ICL_TILE_CASE(12) ICL_TILE_CASE(13) ICL_TILE_CASE(14) ICL_TILE_CASE(15)
#undef ICL_TILE_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace icl
