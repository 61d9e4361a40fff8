// tex.cu -- Table 1's "Image mem." axis on B200 (§5.2.4:
// ImageCL maps an Image to OpenCL image memory, whose sampler gives clamped /
// constant-0 boundaries in hardware; Tables 2-5 show it winning on some
// devices).  Here: CUDA texture objects over the pitched image (point
// sampling, unnormalised coordinates, element reads), cudaAddressModeClamp for
// the clamp boundary and cudaAddressModeBorder (returns 0) for constant-0, so
// the kernels contain no boundary code at all; reads go through the texture
// path of L1.
//
//   sepconv  tex_c4s16 (R <= 8): a thread owns 4 columns and a 16-row output segment,
//            fetches each input row's 4+2R texels, keeps the row-pass results
//            in a register ring and emits a float4 per output row;
//   conv2d   tex_c4r4 : a thread owns a 4 x 4 output block, fetches the 8x8
//            byte window row by row.
// Same per-output fp32 operation order as every variant of the filter (taps
// padded with leading zeros where radii differ, which add exact +0), so the
// results are bit-identical.  Eligible for clamp or constant 0; the texture
// spans the band buffer, whose rows cover every row the stencil reads inside
// the global image, so clamping at its edges is clamping at the image's.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "internal.h"
#include "sepconv_stream.cuh"

namespace icl {

// --------------------------------------------------------------- texture cache
namespace {
using TexKey = std::tuple<int, uintptr_t, int64_t, int64_t, int64_t, int, int>;  // dev, ptr, pitch, W, H, elem, clamp
std::mutex g_tex_mu;
std::map<TexKey, cudaTextureObject_t> g_tex;

cudaError_t tex_of(const void* base, int64_t pitch, int64_t W, int64_t H, int elem, bool clamp,
                   cudaTextureObject_t* out) {
  int dev = 0;
  cudaGetDevice(&dev);
  const TexKey key{dev, reinterpret_cast<uintptr_t>(base), pitch, W, H, elem, clamp ? 1 : 0};
  std::lock_guard<std::mutex> lk(g_tex_mu);
  auto it = g_tex.find(key);
  if (it != g_tex.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  if (g_tex.size() >= 256) {  // bounded: drop everything once idle
    cudaDeviceSynchronize();
    for (auto& kv : g_tex) cudaDestroyTextureObject(kv.second);
    g_tex.clear();
  }
  cudaResourceDesc rd{};
  rd.resType = cudaResourceTypePitch2D;
  rd.res.pitch2D.devPtr = const_cast<void*>(base);
  rd.res.pitch2D.desc = elem == 1 ? cudaCreateChannelDesc<unsigned char>() : cudaCreateChannelDesc<float>();
  rd.res.pitch2D.width = (size_t)W;
  rd.res.pitch2D.height = (size_t)H;
  rd.res.pitch2D.pitchInBytes = (size_t)pitch;
  cudaTextureDesc td{};
  td.addressMode[0] = td.addressMode[1] = clamp ? cudaAddressModeClamp : cudaAddressModeBorder;
  td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType;
  td.normalizedCoords = 0;
  cudaTextureObject_t t = 0;
  cudaError_t e = cudaCreateTextureObject(&t, &rd, &td, nullptr);
  if (e != cudaSuccess) return e;
  g_tex[key] = t;
  *out = t;
  return cudaSuccess;
}
}  // namespace

// Can a pitch-2D texture describe this (band) image?  Alignment and size limits of the device.
bool tex_eligible(const SrcView& s, int64_t rows, int batch, int elem, bool clamp_or_zero) {
  if (!clamp_or_zero) return false;
  int dev = 0, talign = 512, palign = 32, maxw = 0, maxh = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&talign, cudaDevAttrTextureAlignment, dev);
  cudaDeviceGetAttribute(&palign, cudaDevAttrTexturePitchAlignment, dev);
  cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxTexture2DLinearWidth, dev);
  cudaDeviceGetAttribute(&maxh, cudaDevAttrMaxTexture2DLinearHeight, dev);
  if (s.W > maxw || rows > maxh) return false;
  if (s.pitch % palign) return false;
  for (int b = 0; b < batch; ++b)
    if ((reinterpret_cast<uintptr_t>(s.base) + (uintptr_t)((int64_t)b * s.bstride)) % talign) return false;
  (void)elem;
  return true;
}

// --------------------------------------------------------------- sepconv tex_c4s16
template <int R>
__global__ void __launch_bounds__(128) sep_tex(SepParams p, cudaTextureObject_t tex, int64_t src_rows, int b) {
  constexpr int S = 16, NW = 4 + 2 * R, NR = S + 2 * R;
  const int x0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int ly0 = blockIdx.y * S;
  if (x0 >= p.src.W) return;
  const int r0 = p.dst.y0 + ly0 - R - p.src.y0;  // first input row, relative to the texture (band buffer)
  float4 ring[2 * R + 1];
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    const float yy = (float)(r0 + k) + 0.5f;
    float w[NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) w[i] = tex2D<float>(tex, (float)(x0 - R + i) + 0.5f, yy);
    float t[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float a = 0.0f;
#pragma unroll
      for (int i = 0; i < 2 * R + 1; ++i) a = __fmaf_rn(p.fx[i], w[c + i], a);
      t[c] = a;
    }
    ring[k % (2 * R + 1)] = make_float4(t[0], t[1], t[2], t[3]);
    if (k >= 2 * R) {
      const int y = k - 2 * R;  // output row ly0 + y
      float o[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float a = 0.0f;
#pragma unroll
        for (int j = 0; j < 2 * R + 1; ++j) {
          const float4 tv = ring[(y + j) % (2 * R + 1)];
          const float v = c == 0 ? tv.x : c == 1 ? tv.y : c == 2 ? tv.z : tv.w;
          a = __fmaf_rn(p.gy[j], v, a);
        }
        o[c] = a;
      }
      const int ly = ly0 + y;
      if (ly < p.dst.H) {
        float* d = dst_row(p.dst, b, ly) + x0;
        if (x0 + 3 < p.src.W && (reinterpret_cast<uintptr_t>(d) & 15) == 0) {
          st_cs4(d, make_float4(o[0], o[1], o[2], o[3]));
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (x0 + c < p.src.W) d[c] = o[c];
        }
      }
    }
  }
  (void)src_rows;
}

cudaError_t launch_sep_tex(const SepCall& c, cudaStream_t s) {
  SepParams p = make_sep_params(c, true);
  const int R = c.rx > c.ry ? c.rx : c.ry;
  const int64_t rows = c.dst.y0 + c.dst.H + R - c.src.y0;  // texture height: the band buffer's rows in use
  const int64_t hrows = std::min<int64_t>(rows, c.src.Hg - c.src.y0);
  for (int b = 0; b < c.batch; ++b) {
    cudaTextureObject_t tex;
    cudaError_t e = tex_of(c.src.base + (int64_t)b * c.src.bstride, c.src.pitch, c.src.W, hrows, 4,
                           c.src.border == kBorderClamp, &tex);
    if (e != cudaSuccess) return e;
    dim3 grd((unsigned)((c.src.W + 4 * 128 - 1) / (4 * 128)), (unsigned)((c.dst.H + 15) / 16));
    switch (R) {
#define ICL_TEX_CASE(r) \
  case r: sep_tex<r><<<grd, 128, 0, s>>>(p, tex, hrows, b); break;
      ICL_TEX_CASE(0) ICL_TEX_CASE(1) ICL_TEX_CASE(2) ICL_TEX_CASE(3) ICL_TEX_CASE(4) ICL_TEX_CASE(5)
      ICL_TEX_CASE(6) ICL_TEX_CASE(7) ICL_TEX_CASE(8)
#undef ICL_TEX_CASE
      default: return cudaErrorInvalidValue;
    }
    count_launch();
  }
  return cudaGetLastError();
}

// --------------------------------------------------------------- conv2d tex_c4r4
struct C2TexParams {
  DstView dst;
  int W, y_off;  // y_off: texture row of output row 0 = dst.y0 - src.y0
  float f[49];
};

template <int R>
__global__ void __launch_bounds__(128) c2_tex(C2TexParams p, cudaTextureObject_t tex, int b) {
  constexpr int N = 2 * R + 1, NW = 4 + 2 * R;
  const int x0 = 4 * (blockIdx.x * 32 + (threadIdx.x & 31));
  const int ly0 = 4 * (blockIdx.y * 4 + (threadIdx.x >> 5));
  if (x0 >= p.W || ly0 >= p.dst.H) return;
  float acc[4][4];
#pragma unroll
  for (int y = 0; y < 4; ++y)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[y][c] = 0.0f;
#pragma unroll
  for (int k = 0; k < 4 + 2 * R; ++k) {
    const float yy = (float)(p.y_off + ly0 - R + k) + 0.5f;
    float w[NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) w[i] = (float)tex2D<unsigned char>(tex, (float)(x0 - R + i) + 0.5f, yy);
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int j = k - y;
      if (j >= 0 && j < N) {
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[y][c] = __fmaf_rn(p.f[j * N + i], w[c + i], acc[y][c]);
      }
    }
  }
#pragma unroll
  for (int y = 0; y < 4; ++y) {
    const int ly = ly0 + y;
    if (ly < p.dst.H) {
      float* d = dst_row(p.dst, b, ly) + x0;
      if (x0 + 3 < p.W && (reinterpret_cast<uintptr_t>(d) & 15) == 0) {
        st_cs4(d, make_float4(acc[y][0], acc[y][1], acc[y][2], acc[y][3]));
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (x0 + c < p.W) d[c] = acc[y][c];
      }
    }
  }
}

cudaError_t launch_conv2d_tex(const Conv2dCall& c, cudaStream_t s) {
  C2TexParams p;
  p.dst = c.dst;
  p.W = c.src.W;
  p.y_off = c.dst.y0 - c.src.y0;
  for (int k = 0; k < 49; ++k) p.f[k] = c.f[k];
  const int64_t hrows = std::min<int64_t>(c.dst.y0 + c.dst.H + c.r - c.src.y0, c.src.Hg - c.src.y0);
  for (int b = 0; b < c.batch; ++b) {
    cudaTextureObject_t tex;
    cudaError_t e = tex_of(c.src.base + (int64_t)b * c.src.bstride, c.src.pitch, c.src.W, hrows, 1,
                           c.src.border == kBorderClamp, &tex);
    if (e != cudaSuccess) return e;
    dim3 grd((unsigned)((c.src.W + 127) / 128), (unsigned)((c.dst.H + 15) / 16));
    switch (c.r) {
      case 0: c2_tex<0><<<grd, 128, 0, s>>>(p, tex, b); break;
      case 1: c2_tex<1><<<grd, 128, 0, s>>>(p, tex, b); break;
      case 2: c2_tex<2><<<grd, 128, 0, s>>>(p, tex, b); break;
      case 3: c2_tex<3><<<grd, 128, 0, s>>>(p, tex, b); break;
      default: return cudaErrorInvalidValue;
    }
    count_launch();
  }
  return cudaGetLastError();
}

}  // namespace icl
