// conv2d.cu -- non-separable 2-D convolution of an 8-bit image, the paper's
// third benchmark (§6: 8192^2 unsigned char, a 5x5 filter
// whose values are a run-time input, clamped boundary; Table 3 lines
// 631-649; output type: DESIGN.md reading R22):
//     out(x,y) = sum_{j=-r..r} sum_{i=-r..r} f[j+r][i+r] * in_B(x+i, y+j)
// Every variant evaluates, per output, one fp32 FMA chain over j then i,
// starting from +0, with the byte converted exactly to fp32 -> variants and
// band splits are bit-identical.  The taps live in the kernel parameter
// block (the constant-memory analog of Table 3), so every FFMA reads its tap
// straight from the constant bank.
//
// Variants (Table 1 axes):
//   naive_direct  one thread per output, byte loads through the read-only path;
//   tile_c4r<RPT> 64 x (16*RPT) output tile per 256-thread CTA: the 8-bit
//                 input tile (+halo) is staged with 16-byte cp.async, converted
//                 once to an fp32 smem tile, and each thread computes a
//                 4-column x RPT-row register block from LDS.128 windows
//                 (coarsening 4 x RPT, local memory on, interleaved off).
#include "common.cuh"
#include "internal.h"

namespace icl {

struct C2Params {
  SrcView src;
  DstView dst;
  float f[49];
};

// in_B(x, y) of the 8-bit image at GLOBAL row gy (Fig. 3).
__device__ __forceinline__ float read_B8(const SrcView& s, int b, int x, int gy) {
  if (x < 0 || x >= s.W || gy < 0 || gy >= s.Hg) {
    if (s.border == kBorderConstant) return s.cval;
    x = clampi(x, 0, s.W - 1);
    gy = clampi(gy, 0, s.Hg - 1);
  }
  const unsigned char* row =
      reinterpret_cast<const unsigned char*>(s.base + (int64_t)b * s.bstride + (int64_t)(gy - s.y0) * s.pitch);
  return (float)__ldg(row + x);
}

static C2Params make_c2_params(const Conv2dCall& c) {
  C2Params p;
  p.src = c.src;
  p.dst = c.dst;
  for (int k = 0; k < 49; ++k) p.f[k] = c.f[k];
  return p;
}

// ---------------------------------------------------------------- naive_direct
template <int R>
__global__ void __launch_bounds__(128) c2_naive(C2Params p) {
  constexpr int N = 2 * R + 1;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int ly = blockIdx.y, b = blockIdx.z;
  if (x >= p.src.W) return;
  const int gy = p.dst.y0 + ly;
  float acc = 0.0f;
#pragma unroll
  for (int j = -R; j <= R; ++j)
#pragma unroll
    for (int i = -R; i <= R; ++i) acc = __fmaf_rn(p.f[(j + R) * N + (i + R)], read_B8(p.src, b, x + i, gy + j), acc);
  dst_row(p.dst, b, ly)[x] = acc;
}

// ---------------------------------------------------------------- tile_c4r<RPT>
template <int R, int RPT>
struct C2Geom {
  static constexpr int TW = 64, NT = 256;       // 16 x 16 threads
  static constexpr int TH = 16 * RPT;
  static constexpr int IR = TH + 2 * R;         // input rows
  static constexpr int UW = TW + 32;            // staged bytes per row: x0-16 .. x0+TW+16
  static constexpr int FW0 = TW + 2 * R;        // fp32 columns x0-R .. x0+TW+R
  static constexpr int NWIN = (4 + 2 * R + 3) / 4;  // LDS.128 per window row
  static constexpr int FW = ((FW0 + 3) / 4) * 4 > 4 * 15 + 4 * NWIN ? ((FW0 + 3) / 4) * 4 : 4 * 15 + 4 * NWIN;
  static constexpr int U8B = ((IR * UW + 15) / 16) * 16;
  static constexpr size_t smem_bytes = (size_t)U8B + (size_t)IR * FW * sizeof(float);
};

template <int R, int RPT>
__global__ void __launch_bounds__(256) c2_tile(C2Params p) {
  using G = C2Geom<R, RPT>;
  constexpr int TW = G::TW, TH = G::TH, IR = G::IR, UW = G::UW, FW0 = G::FW0, FW = G::FW, NWIN = G::NWIN;
  constexpr int N = 2 * R + 1, NT = G::NT;
  extern __shared__ __align__(16) unsigned char sm8[];
  unsigned char* U8 = sm8;                                 // [IR][UW]
  float* F = reinterpret_cast<float*>(sm8 + G::U8B);        // [IR][FW], column c <-> x0 - R + c
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * TW, ly0 = blockIdx.y * TH;
  const int g0 = p.dst.y0 + ly0;
  const int W = p.src.W, Hg = p.src.Hg;
  const bool interior = x0 - 16 >= 0 && x0 + TW + 16 <= W && g0 - R >= 0 && g0 + TH + R <= Hg;

  if (interior) {
    // 16-byte cp.async of the byte tile (rows g0-R .., columns x0-16 ..)
    const char* rowb = p.src.base + (int64_t)b * p.src.bstride + (int64_t)(g0 - R - p.src.y0) * p.src.pitch;
    constexpr int NCH = UW / 16;
    for (int i = tid; i < IR * NCH; i += NT) {
      const int r = i / NCH, c = i - r * NCH;
      cp_async16(U8 + r * UW + 16 * c, rowb + (int64_t)r * p.src.pitch + (x0 - 16 + 16 * c), 16);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    // convert once: F[r][c] = U8[r][16 - R + c]  (4 columns per item, from two aligned words)
    constexpr int NQ = (FW0 + 3) / 4;
    for (int i = tid; i < IR * NQ; i += NT) {
      const int r = i / NQ, q = i - r * NQ;
      const int byte0 = 16 - R + 4 * q;  // first byte of this group
      const uint32_t* w = reinterpret_cast<const uint32_t*>(U8 + r * UW + (byte0 & ~3));
      const uint32_t v = __funnelshift_r(w[0], w[1], 8 * (byte0 & 3));
      *reinterpret_cast<float4*>(F + r * FW + 4 * q) =
          make_float4((float)(v & 0xffu), (float)((v >> 8) & 0xffu), (float)((v >> 16) & 0xffu), (float)(v >> 24));
    }
  } else {
    for (int i = tid; i < IR * FW0; i += NT) {
      const int r = i / FW0, c = i - r * FW0;
      F[r * FW + c] = read_B8(p.src, b, x0 - R + c, g0 - R + r);
    }
  }
  __syncthreads();

  float acc[RPT][4];
#pragma unroll
  for (int y = 0; y < RPT; ++y)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[y][c] = 0.0f;
  const float* fb = F + (RPT * ty) * FW + 4 * tx;
#pragma unroll
  for (int k = 0; k < RPT + 2 * R; ++k) {  // input row (relative), ascending -> j ascending per output
    float w[4 * NWIN];
#pragma unroll
    for (int q = 0; q < NWIN; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(fb + k * FW + 4 * q);
      w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
    }
#pragma unroll
    for (int y = 0; y < RPT; ++y) {
      const int j = k - y;  // tap row for output row y
      if (j >= 0 && j < N) {
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[y][c] = __fmaf_rn(p.f[j * N + i], w[c + i], acc[y][c]);
      }
    }
  }
  const int gx = x0 + 4 * tx;
#pragma unroll
  for (int y = 0; y < RPT; ++y) {
    const int ly = ly0 + RPT * ty + y;
    if (ly < p.dst.H) {
      float* d = dst_row(p.dst, b, ly) + gx;
      if (gx + 3 < W) {
        st_cs4(d, make_float4(acc[y][0], acc[y][1], acc[y][2], acc[y][3]));
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (gx + c < W) d[c] = acc[y][c];
      }
    }
  }
}

// ---------------------------------------------------------------- launchers
template <int R>
static cudaError_t launch_naive_R(const C2Params& p, int batch, cudaStream_t s) {
  dim3 grd((p.src.W + 127) / 128, p.dst.H, batch);
  c2_naive<R><<<grd, 128, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_conv2d_naive(const Conv2dCall& c, cudaStream_t s) {
  const C2Params p = make_c2_params(c);
  switch (c.r) {
    case 0: return launch_naive_R<0>(p, c.batch, s);
    case 1: return launch_naive_R<1>(p, c.batch, s);
    case 2: return launch_naive_R<2>(p, c.batch, s);
    case 3: return launch_naive_R<3>(p, c.batch, s);
  }
  return cudaErrorInvalidValue;
}

template <int R, int RPT>
static cudaError_t launch_tile_R(const C2Params& p, int batch, cudaStream_t s) {
  using G = C2Geom<R, RPT>;
  auto kern = c2_tile<R, RPT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::smem_bytes);
  if (e != cudaSuccess) return e;
  dim3 grd((p.src.W + G::TW - 1) / G::TW, (p.dst.H + G::TH - 1) / G::TH, batch);
  kern<<<grd, G::NT, G::smem_bytes, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

template <int RPT>
static cudaError_t launch_tile_rpt(const C2Params& p, int r, int batch, cudaStream_t s) {
  switch (r) {
    case 0: return launch_tile_R<0, RPT>(p, batch, s);
    case 1: return launch_tile_R<1, RPT>(p, batch, s);
    case 2: return launch_tile_R<2, RPT>(p, batch, s);
    case 3: return launch_tile_R<3, RPT>(p, batch, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_conv2d_tile(const Conv2dCall& c, int rows_per_thread, cudaStream_t s) {
  const C2Params p = make_c2_params(c);
  if (rows_per_thread == 4) return launch_tile_rpt<4>(p, c.r, c.batch, s);
  if (rows_per_thread == 8) return launch_tile_rpt<8>(p, c.r, c.batch, s);
  return cudaErrorInvalidValue;
}

}  // namespace icl
