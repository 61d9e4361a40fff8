// sep3d.cu -- separable convolution of 3-D volumes (ImageCL Images support
// "2D/3D indexing"; R26).
//
//     out(x,y,z) = sum_k h_k sum_j g_j sum_i f_i in_B(x+i, y+j, z+k)
//
// A volume is an icl_image whose batch axis is z (batch = depth, the batch
// stride = the slice stride); the boundary applies per axis.  Every variant
// evaluates the same fp32 chains (from 0.0f, taps in index order):
//     t = fma-chain_i f_i in_B,  s = fma-chain_j g_j t,  out = fma-chain_k h_k s
// so the variants are bit-identical (R16's rule carried to 3-D).
//
// Variants: "naive_direct" (one thread per voxel, direct loads) and
// "tile64x16" (tile<R>): a CTA owns a 64 x 16 (x, y) tile and streams a
// chunk of slices along z.  Per input slice: the (16+2R) x (64+2R) input tile
// arrives in a 4-stage cp.async ring in shared memory, the row pass goes into
// a second smem tile, the column pass into registers (4 consecutive rows per
// thread), and a register ring keeps the last 2R+1 column-pass results per
// output; once it is full each new slice emits one output slice.
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace icl {

__device__ __forceinline__ float read_B3(const Sep3Params& p, int x, int y, int z) {
  if (x < 0 || x >= p.W || y < 0 || y >= p.H || z < 0 || z >= p.D) {
    if (p.border == kBorderConstant) return p.cval;
    x = clampi(x, 0, p.W - 1);
    y = clampi(y, 0, p.H - 1);
    z = clampi(z, 0, p.D - 1);
  }
  return __ldg(reinterpret_cast<const float*>(p.src + (int64_t)z * p.sslice + (int64_t)y * p.spitch) + x);
}

__global__ void __launch_bounds__(256) sep3d_naive(Sep3Params p) {
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (x >= p.W || y >= p.H) return;
  for (int z = blockIdx.z; z < p.D; z += gridDim.z) {
    float out = 0.0f;
    for (int k = -p.rz; k <= p.rz; ++k) {
      float s = 0.0f;
      for (int j = -p.ry; j <= p.ry; ++j) {
        float t = 0.0f;
        for (int i = -p.rx; i <= p.rx; ++i) t = __fmaf_rn(p.fx[i + p.rx], read_B3(p, x + i, y + j, z + k), t);
        s = __fmaf_rn(p.gy[j + p.ry], t, s);
      }
      out = __fmaf_rn(p.hz[k + p.rz], s, out);
    }
    reinterpret_cast<float*>(p.dst + (int64_t)z * p.dslice + (int64_t)y * p.dpitch)[x] = out;
  }
}

constexpr int k3TW = 64, k3NT = 256;

// Input slices stream through an NS-stage ring of shared-memory tiles filled by
// 4-byte cp.async (per-element source address: clamped for the clamp boundary,
// zero-fill for a constant-0 boundary), so NS-1 slices of loads are in flight
// while a slice is convolved; two barriers per slice.  Constant boundaries with
// c != 0 take the synchronous loader (async = false).
// Tile height per radius: 32 rows (8 per thread) with a 3-stage slice ring for R <= 3 (halves
// the y halo and the barriers per voxel), 16 rows with 4 stages above (static smem < 48 KB).
template <int R>
struct Sep3Geom {
  static constexpr int TH = R <= 3 ? 32 : 16;
  static constexpr int NS = R <= 3 ? 3 : 4;
};

template <int R>
__global__ void __launch_bounds__(k3NT, 2) sep3d_tile(Sep3Params p, int zchunk, int async) {
  constexpr int K = 2 * R + 1;
  constexpr int TH = Sep3Geom<R>::TH, RPT = TH / 4, NS = Sep3Geom<R>::NS;  // rows per thread
  constexpr int HA = 4 * ((R + 3) / 4);           // 16-byte aligned halo >= R
  constexpr int IW = k3TW + 2 * R, IH = TH + 2 * R;
  constexpr int IWS = k3TW + 2 * HA;              // smem row: columns x0-HA .. x0+64+HA
  __shared__ __align__(16) float sin_[NS][IH][IWS];
  __shared__ __align__(16) float st[IH][k3TW];
  const int tid = threadIdx.x;
  const int x0 = blockIdx.x * k3TW, y0 = blockIdx.y * TH;
  const int z0 = blockIdx.z * zchunk, z1 = min(z0 + zchunk, p.D);
  const int tx = tid & (k3TW - 1), ty = (tid / k3TW) * RPT;  // outputs (x0+tx, y0+ty .. +RPT-1)
  const int x = x0 + tx;
  float ring[K][RPT];
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int q = 0; q < RPT; ++q) ring[k][q] = 0.0f;
  const bool clampb = p.border == kBorderClamp;
  // interior tile with 16-byte aligned rows: whole-row 16-byte copies of the aligned superset
  const bool vec16 = async && x0 - HA >= 0 && x0 + k3TW + HA <= p.W && y0 - R >= 0 && y0 + TH + R <= p.H &&
                     ((p.spitch | p.sslice | (int64_t)p.src) & 15) == 0;

  // The loader's element list is slice-invariant: precompute each element's slice-relative
  // source byte offset (clamped columns / rows for the clamp boundary) and whether it lies
  // outside the image (zero-fill for a constant-0 boundary).
  constexpr int NV = IH * (IWS / 4);                  // 16-byte chunks per slice (vec16)
  constexpr int NPRE = (IH * IW + k3NT - 1) / k3NT;   // elements per thread (4-byte path)
  constexpr int NPRE16 = (NV + k3NT - 1) / k3NT;
  int soff[NPRE > NPRE16 ? NPRE : NPRE16];
  unsigned outm = 0;  // bit e: element e outside the image in x or y
  if (vec16) {
#pragma unroll
    for (int e = 0; e < NPRE16; ++e) {
      const int idx = tid + e * k3NT;
      const int r = idx / (IWS / 4), c4 = idx - r * (IWS / 4);
      soff[e] = (int)((y0 - R + r) * p.spitch + 4 * (x0 - HA + 4 * c4));
    }
  } else {
#pragma unroll
    for (int e = 0; e < NPRE; ++e) {
      const int idx = tid + e * k3NT;
      const int r = idx / IW, c = idx - r * IW;
      const int xx = x0 - R + c, yy = y0 - R + r;
      if (xx < 0 || xx >= p.W || yy < 0 || yy >= p.H) outm |= 1u << e;
      soff[e] = (int)(clampi(yy, 0, p.H - 1) * p.spitch + 4 * clampi(xx, 0, p.W - 1));
    }
  }
  // issue the loads of input slice zz into stage s (element (r, c) of the R-halo tile lives at
  // smem column HA - R + c)
  auto issue = [&](int zz, int s) {
    const bool zout = zz < 0 || zz >= p.D;
    const int zs = clampi(zz, 0, p.D - 1);
    const char* sl = p.src + (int64_t)zs * p.sslice;
    float* dst = &sin_[s][0][0];
    if (vec16) {
#pragma unroll
      for (int e = 0; e < NPRE16; ++e) {
        const int idx = tid + e * k3NT;
        if (idx < NV) {
          const bool zero = !clampb && zout;
          cp_async16(dst + 4 * idx, sl + (zero ? 0 : soff[e]), zero ? 0 : 16);
        }
      }
      return;
    }
#pragma unroll
    for (int e = 0; e < NPRE; ++e) {
      const int idx = tid + e * k3NT;
      if (idx < IH * IW) {
        const int r = idx / IW, c = idx - r * IW;
        float* d = dst + r * IWS + (HA - R) + c;
        if (async) {
          const bool zero = !clampb && (zout || ((outm >> e) & 1u));  // constant 0: zero-fill
          cp_async4(d, sl + (zero ? 0 : soff[e]), zero ? 0 : 4);
        } else {
          *d = (zout && !clampb) ? p.cval : read_B3(p, x0 - R + c, y0 - R + r, zs);
        }
      }
    }
  };
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) {
    if (z0 - R + s < z1 + R) issue(z0 - R + s, s);
    cp_async_commit();
  }
#pragma unroll 1
  for (int zz = z0 - R; zz < z1 + R; ++zz) {
    const int s = (zz - (z0 - R)) % NS;
    cp_async_wait<NS - 2>();
    __syncthreads();  // slice zz landed; the previous slice's st reads are done
    if (zz + NS - 1 < z1 + R) issue(zz + NS - 1, (s + NS - 1) % NS);
    cp_async_commit();
    // row pass: t(x, y') for the tile's columns and its TH + 2R rows
    for (int e = tid; e < IH * (k3TW / 4); e += k3NT) {  // item = 4 consecutive columns of one row
      const int r = e / (k3TW / 4), c = 4 * (e - r * (k3TW / 4));
      // smem columns c .. c+4+2HA-1 as aligned LDS.128 (lanes 16 bytes apart: conflict-free)
      float v[4 + 2 * HA];
#pragma unroll
      for (int m4 = 0; m4 < (4 + 2 * HA) / 4; ++m4) {
        const float4 w4 = *reinterpret_cast<const float4*>(&sin_[s][r][c + 4 * m4]);
        v[4 * m4] = w4.x; v[4 * m4 + 1] = w4.y; v[4 * m4 + 2] = w4.z; v[4 * m4 + 3] = w4.w;
      }
      float tq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float acc = 0.0f;
#pragma unroll
        for (int i = 0; i < K; ++i) acc = __fmaf_rn(p.fx[i], v[(HA - R) + q + i], acc);
        tq[q] = acc;
      }
      *reinterpret_cast<float4*>(&st[r][c]) = make_float4(tq[0], tq[1], tq[2], tq[3]);
    }
    __syncthreads();
    // column pass for RPT consecutive rows; slide the z ring
    float sc[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      float a = 0.0f;
#pragma unroll
      for (int j = 0; j < K; ++j) a = __fmaf_rn(p.gy[j], st[ty + q + j][tx], a);
      sc[q] = a;
    }
#pragma unroll
    for (int k = 0; k + 1 < K; ++k)
#pragma unroll
      for (int q = 0; q < RPT; ++q) ring[k][q] = ring[k + 1][q];
#pragma unroll
    for (int q = 0; q < RPT; ++q) ring[K - 1][q] = sc[q];
    const int z = zz - R;  // output slice completed by input slice zz
    if (z >= z0 && x < p.W) {
      float* drow = reinterpret_cast<float*>(p.dst + (int64_t)z * p.dslice);
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int y = y0 + ty + q;
        if (y < p.H) {
          float o = 0.0f;
#pragma unroll
          for (int k = 0; k < K; ++k) o = __fmaf_rn(p.hz[k], ring[k][q], o);
          reinterpret_cast<float*>(reinterpret_cast<char*>(drow) + (int64_t)y * p.dpitch)[x] = o;
        }
      }
    }
  }
  cp_async_wait<0>();
}

bool sep3d_tile_supported(int R) { return R >= 0 && R <= 7; }

cudaError_t launch_sep3d(const Sep3Params& p0, int variant, cudaStream_t s) {
  Sep3Params p = p0;
  if (variant == 0) {
    dim3 grd((p.W + 31) / 32, (p.H + 7) / 8, (unsigned)min(p.D, 65535));
    sep3d_naive<<<grd, 256, 0, s>>>(p);
    count_launch();
    return cudaGetLastError();
  }
  const int R = max(p.rx, max(p.ry, p.rz));
  // zero-pad the taps to R (fma(0, v, a) == a: the same values)
  float f[15] = {0}, g[15] = {0}, h[15] = {0};
  for (int i = -p.rx; i <= p.rx; ++i) f[R + i] = p0.fx[p.rx + i];
  for (int j = -p.ry; j <= p.ry; ++j) g[R + j] = p0.gy[p.ry + j];
  for (int k = -p.rz; k <= p.rz; ++k) h[R + k] = p0.hz[p.rz + k];
  for (int i = 0; i < 15; ++i) { p.fx[i] = f[i]; p.gy[i] = g[i]; p.hz[i] = h[i]; }
  // z chunk: enough CTAs for ~4 per SM (2 resident at 256 threads x ~120 registers), but at
  // least 8R slices so the 2R recomputed halo slices stay <= 25% of a chunk
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || nsm < 1) nsm = 148;
  const int th = R <= 3 ? 32 : 16;  // Sep3Geom<R>::TH
  const int64_t tiles = (int64_t)((p.W + k3TW - 1) / k3TW) * ((p.H + th - 1) / th);
  int zchunk = (int)std::min<int64_t>(64, std::max<int64_t>(1, (int64_t)p.D * tiles / (4 * nsm)));
  zchunk = std::max(zchunk, std::max(8, 8 * R));
  const int zb = (p.D + zchunk - 1) / zchunk;
  if (zb > 65535) return cudaErrorInvalidValue;
  const int async = (p.border == kBorderClamp || p.cval == 0.0f) ? 1 : 0;
  dim3 grd((p.W + k3TW - 1) / k3TW, (p.H + th - 1) / th, zb);
  switch (R) {
#define ICL_S3(RR) \
  case RR: sep3d_tile<RR><<<grd, k3NT, 0, s>>>(p, zchunk, async); break;
    ICL_S3(0) ICL_S3(1) ICL_S3(2) ICL_S3(3) ICL_S3(4) ICL_S3(5) ICL_S3(6) ICL_S3(7)
#undef ICL_S3
    default: return cudaErrorInvalidValue;
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace icl
