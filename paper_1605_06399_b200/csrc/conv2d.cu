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
//                 once to an fp32 smem tile (exact PRMT + FADD, no I2F), and
//                 each thread computes a 4-column x RPT-row register block from
//                 LDS.128 windows, two output rows per FFMA2 (coarsening 4 x RPT,
//                 local memory on, interleaved off).
#include "common.cuh"
#include "internal.h"

namespace icl {

struct C2Params {
  SrcView src;
  DstView dst;
  float f[49];
  // tap pairs for two output rows y, y+1 fed by one input row: tp[j][i] = (f[j][i], f[j-1][i]),
  // j = 1..2r used (j = 0 / 2r+1 feed one row only and run as scalar FFMAs)
  float2 tp[8 * 7];
};

// in_B(x, y) of the 8-bit image at GLOBAL row gy (Fig. 3).
__device__ __forceinline__ float read_B8(const SrcView& s, int b, int x, int gy) {
  if (x < 0 || x >= s.W || gy < 0 || gy >= s.Hg) {
    if (s.border == kBorderConstant) return s.cval;
    x = clampi(x, 0, s.W - 1);
    gy = clampi(gy, 0, s.Hg - 1);
  }
  if ((unsigned)(gy - s.y0) >= (unsigned)s.Hl) return 0.0f;  // (see read_B)
  const unsigned char* row =
      reinterpret_cast<const unsigned char*>(s.base + (int64_t)b * s.bstride + (int64_t)(gy - s.y0) * s.pitch);
  return (float)__ldg(row + x);
}

static C2Params make_c2_params(const Conv2dCall& c) {
  C2Params p;
  p.src = c.src;
  p.dst = c.dst;
  for (int k = 0; k < 49; ++k) p.f[k] = c.f[k];
  const int n = 2 * c.r + 1;
  for (int j = 0; j <= n; ++j)
    for (int i = 0; i < n; ++i)
      p.tp[j * n + i] = make_float2(j < n ? c.f[j * n + i] : 0.0f, j >= 1 ? c.f[(j - 1) * n + i] : 0.0f);
  return p;
}

// ---------------------------------------------------------------- naive_direct
template <int R>
__global__ void __launch_bounds__(128) c2_naive(C2Params p) {
  constexpr int N = 2 * R + 1;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.z;
  if (x >= p.src.W) return;
  for (int ly = blockIdx.y; ly < p.dst.H; ly += gridDim.y) {  // grid-stride: any height
    const int gy = p.dst.y0 + ly;
    float acc = 0.0f;
#pragma unroll
    for (int j = -R; j <= R; ++j)
#pragma unroll
      for (int i = -R; i <= R; ++i) acc = __fmaf_rn(p.f[(j + R) * N + (i + R)], read_B8(p.src, b, x + i, gy + j), acc);
    dst_row(p.dst, b, ly)[x] = acc;
  }
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

// Pieces of one tile, shared by the one-tile-per-CTA and the persistent kernels.
template <int R, int RPT>
struct C2Tile {
  using G = C2Geom<R, RPT>;
  static constexpr int TW = G::TW, TH = G::TH, IR = G::IR, UW = G::UW, FW0 = G::FW0, FW = G::FW, NWIN = G::NWIN;
  static constexpr int N = 2 * R + 1, NT = G::NT;

  __device__ static bool interior(const C2Params& p, int x0, int g0) {
    return x0 - 16 >= 0 && x0 + TW + 16 <= p.src.W && g0 - R >= 0 && g0 + TH + R <= p.src.Hg &&
           g0 - R >= p.src.y0 && g0 + TH + R <= p.src.y0 + p.src.Hl;  // (rows held by a band buffer)
  }
  // 16-byte cp.async of the byte tile (rows g0-R .., columns x0-16 ..); caller commits
  __device__ static void stage(const C2Params& p, int b, int x0, int g0, unsigned char* U8) {
    const char* rowb = p.src.base + (int64_t)b * p.src.bstride + (int64_t)(g0 - R - p.src.y0) * p.src.pitch;
    constexpr int NCH = UW / 16;
    for (int i = threadIdx.x; i < IR * NCH; i += NT) {
      const int r = i / NCH, c = i - r * NCH;
      cp_async16(U8 + r * UW + 16 * c, rowb + (int64_t)r * p.src.pitch + (x0 - 16 + 16 * c), 16);
    }
  }
  // F[r][c] = U8[r][16 - R + c], 4 columns per item from two aligned words.  byte -> fp32 exactly
  // without the XU pipe: PRMT builds 0x4B0000bb (= 2^23 + b), one FADD subtracts 2^23.
  __device__ static void convert(const unsigned char* U8, float* F) {
    constexpr int NQ = (FW0 + 3) / 4;  // item i = (r, q) = (i / NQ, i % NQ)
    constexpr int DR = NT / NQ, DQ = NT % NQ;
    const int tid = threadIdx.x;
    int r = tid / NQ, q = tid - (tid / NQ) * NQ;
    const float m = 8388608.0f;
#pragma unroll 2
    for (; r < IR;) {
      const int byte0 = 16 - R + 4 * q;
      const uint32_t* w = reinterpret_cast<const uint32_t*>(U8 + r * UW + (byte0 & ~3));
      const uint32_t v = __funnelshift_r(w[0], w[1], 8 * (byte0 & 3));
      float4 o;
      o.x = __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7440)) - m;
      o.y = __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7441)) - m;
      o.z = __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7442)) - m;
      o.w = __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7443)) - m;
      *reinterpret_cast<float4*>(F + r * FW + 4 * q) = o;
      r += DR;
      q += DQ;
      if (q >= NQ) { q -= NQ; ++r; }
    }
  }
  // border tile: in_B per element straight into F
  __device__ static void border_fill(const C2Params& p, int b, int x0, int g0, float* F) {
    for (int i = threadIdx.x; i < IR * FW0; i += NT) {
      const int r = i / FW0, c = i - r * FW0;
      F[r * FW + c] = read_B8(p.src, b, x0 - R + c, g0 - R + r);
    }
  }
  // 4 columns x RPT rows per thread; output rows (2m, 2m+1) share FFMA2 lanes: one input pixel
  // (broadcast) times the tap pair (f[j][i], f[j-1][i]) for the input rows that feed both outputs;
  // the first / last input row of the pair feeds one output only and runs as scalar FFMAs on that
  // lane.  Each lane runs its own pixel's chain j = 0..2R in order: the per-output order is the
  // naive one.
  __device__ static void compute_store(const C2Params& p, const float* F, int b, int x0, int ly0) {
    static_assert(RPT % 2 == 0, "row pairs");
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    float2 acc[RPT / 2][4];
#pragma unroll
    for (int m = 0; m < RPT / 2; ++m)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[m][c] = make_float2(0.0f, 0.0f);
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
      for (int m = 0; m < RPT / 2; ++m) {
        const int j = k - 2 * m;  // tap row of output row 2m (row 2m+1 uses j-1)
        if (j == 0) {
#pragma unroll
          for (int i = 0; i < N; ++i)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[m][c].x = __fmaf_rn(p.f[i], w[c + i], acc[m][c].x);
        } else if (j == N) {
#pragma unroll
          for (int i = 0; i < N; ++i)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[m][c].y = __fmaf_rn(p.f[(N - 1) * N + i], w[c + i], acc[m][c].y);
        } else if (j > 0 && j < N) {
#pragma unroll
          for (int i = 0; i < N; ++i) {
            const float2 t = p.tp[j * N + i];
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[m][c] = __ffma2_rn(make_float2(w[c + i], w[c + i]), t, acc[m][c]);
          }
        }
      }
    }
    const int W = p.src.W;
    const int gx = x0 + 4 * tx;
#pragma unroll
    for (int y = 0; y < RPT; ++y) {
      const int ly = ly0 + RPT * ty + y;
      if (ly < p.dst.H) {
        float* d = dst_row(p.dst, b, ly) + gx;
        const int m = y >> 1;
        const float o[4] = {(y & 1) ? acc[m][0].y : acc[m][0].x, (y & 1) ? acc[m][1].y : acc[m][1].x,
                            (y & 1) ? acc[m][2].y : acc[m][2].x, (y & 1) ? acc[m][3].y : acc[m][3].x};
        if (gx + 3 < W) {
          st_cs4(d, make_float4(o[0], o[1], o[2], o[3]));
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (gx + c < W) d[c] = o[c];
        }
      }
    }
  }
};

template <int R, int RPT>
__global__ void __launch_bounds__(256) c2_tile(C2Params p) {
  using T = C2Tile<R, RPT>;
  extern __shared__ __align__(16) unsigned char sm8[];
  unsigned char* U8 = sm8;                                          // [IR][UW]
  float* F = reinterpret_cast<float*>(sm8 + C2Geom<R, RPT>::U8B);  // [IR][FW], column c <-> x0 - R + c
  const int b = blockIdx.z, x0 = blockIdx.x * T::TW, ly0 = blockIdx.y * T::TH;
  const int g0 = p.dst.y0 + ly0;
  if (T::interior(p, x0, g0)) {
    T::stage(p, b, x0, g0, U8);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    T::convert(U8, F);
  } else {
    T::border_fill(p, b, x0, g0, F);
  }
  __syncthreads();
  T::compute_store(p, F, b, x0, ly0);
}

// Persistent form: a grid of CTAs walks the tiles; while a tile converts and computes, the NEXT
// tile's bytes stream in by cp.async into the second staging buffer.  Same arithmetic.
template <int R, int RPT>
__global__ void __launch_bounds__(256) c2_tile_p(C2Params p, int ntx, int nty, int ntiles) {
  using T = C2Tile<R, RPT>;
  using G = C2Geom<R, RPT>;
  extern __shared__ __align__(16) unsigned char sm8[];
  float* F = reinterpret_cast<float*>(sm8 + 2 * G::U8B);
  const int per_img = ntx * nty;
  auto coords = [&](int t, int& b, int& x0, int& ly0) {
    b = t / per_img;
    const int r = t - b * per_img;
    const int tyy = r / ntx;
    ly0 = tyy * T::TH;
    x0 = (r - tyy * ntx) * T::TW;
  };
  int t = blockIdx.x;
  if (t >= ntiles) return;
  int b, x0, ly0;
  coords(t, b, x0, ly0);
  bool inter = T::interior(p, x0, p.dst.y0 + ly0);
  if (inter) T::stage(p, b, x0, p.dst.y0 + ly0, sm8);
  cp_async_commit();
  for (int it = 0; t < ntiles; ++it) {
    unsigned char* U8 = sm8 + (it & 1) * G::U8B;
    cp_async_wait<0>();
    __syncthreads();  // staged bytes visible; F and the other staging buffer are free
    const int tn = t + gridDim.x;
    int b2 = 0, x2 = 0, y2 = 0;
    bool inter2 = false;
    if (tn < ntiles) {
      coords(tn, b2, x2, y2);
      inter2 = T::interior(p, x2, p.dst.y0 + y2);
      if (inter2) T::stage(p, b2, x2, p.dst.y0 + y2, sm8 + ((it + 1) & 1) * G::U8B);
    }
    cp_async_commit();
    if (inter) T::convert(U8, F);
    else T::border_fill(p, b, x0, p.dst.y0 + ly0, F);
    __syncthreads();
    T::compute_store(p, F, b, x0, ly0);
    t = tn;
    b = b2; x0 = x2; ly0 = y2;
    inter = inter2;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------- launchers
template <int R>
static cudaError_t launch_naive_R(const C2Params& p, int batch, cudaStream_t s) {
  dim3 grd((p.src.W + 127) / 128, p.dst.H < 65535 ? p.dst.H : 65535, batch);
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

template <int R, int RPT>
static cudaError_t launch_tilep_R(const C2Params& p, int batch, cudaStream_t s) {
  using G = C2Geom<R, RPT>;
  const size_t smem = 2 * (size_t)G::U8B + (size_t)G::IR * G::FW * sizeof(float);
  auto kern = c2_tile_p<R, RPT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::NT, smem);
  const int ntx = (p.src.W + G::TW - 1) / G::TW, nty = (p.dst.H + G::TH - 1) / G::TH;
  const int ntiles = ntx * nty * batch;
  const int cap = sms * (per_sm > 0 ? per_sm : 1);
  kern<<<ntiles < cap ? ntiles : cap, G::NT, smem, s>>>(p, ntx, nty, ntiles);
  count_launch();
  return cudaGetLastError();
}

template <int RPT>
static cudaError_t launch_tilep_rpt(const C2Params& p, int r, int batch, cudaStream_t s) {
  switch (r) {
    case 0: return launch_tilep_R<0, RPT>(p, batch, s);
    case 1: return launch_tilep_R<1, RPT>(p, batch, s);
    case 2: return launch_tilep_R<2, RPT>(p, batch, s);
    case 3: return launch_tilep_R<3, RPT>(p, batch, s);
  }
  return cudaErrorInvalidValue;
}

// rows_per_thread 4 / 8; persistent = the prefetching grid-stride form
cudaError_t launch_conv2d_tile(const Conv2dCall& c, int rows_per_thread, bool persistent, cudaStream_t s) {
  const C2Params p = make_c2_params(c);
  if (persistent) {
    if (rows_per_thread == 4) return launch_tilep_rpt<4>(p, c.r, c.batch, s);
    if (rows_per_thread == 8) return launch_tilep_rpt<8>(p, c.r, c.batch, s);
    return cudaErrorInvalidValue;
  }
  if (rows_per_thread == 4) return launch_tile_rpt<4>(p, c.r, c.batch, s);
  if (rows_per_thread == 8) return launch_tile_rpt<8>(p, c.r, c.batch, s);
  return cudaErrorInvalidValue;
}

}  // namespace icl
