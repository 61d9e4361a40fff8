// pmap.cu -- the paper's own tuning space as real kernel axes (§5.2,
// Table 1): the one-pixel-per-
// logical-thread kernels of ImageCL (separable convolution as Listing 1's fused
// 2-D loop nest, Harris as Table 5's loops) wrapped in the transformations the
// paper's source-to-source compiler applies:
//   work-group size      -> CTA shape (wx, wy)                      (§5.2.1)
//   thread coarsening    -> cx x cy logical pixels per thread      (§5.2.2)
//   thread mapping       -> blocked / interleaved / interleaved in
//                           the work-group (Fig. 4; formulas SPEC.md:302-306)  (§5.2.3)
//   local memory         -> the CTA's pixel block + halo staged in
//                           shared memory by cooperative loads       (§5.2.4)
//   loop unrolling       -> unroll factor of the filter loops       (§5.2.5)
// "Constant memory" for the taps is the kernel parameter block (every variant).
// Interleaving with local memory is interleaving within the work-group, as the
// paper prescribes (the CTA's pixels must stay one contiguous block).
//
// Every variant evaluates each output with the naive per-output fp32 order
// (sepconv: t_j = fma-chain over i, out = fma-chain over j; Harris: harris_naive's
// loops), so the whole space is bit-identical to naive_direct and the tuner's
// equivalence check is exact.  These variants are the baseline the hand-built
// streaming kernels beat on B200; they make the tuner's search space the paper's
// (hundreds of configurations per filter), which is what the ANN-guided search
// (icl_tune_ann) exists for.
#include "common.cuh"
#include "harris_stream.cuh"
#include "internal.h"
#include "sepconv_stream.cuh"

namespace icl {

// logical pixel (x, y) of coarsening step (ix, iy) -- SPEC.md:302-306
struct PmapIndex {
  int gx, gy;    // global thread id (logical grid)
  int lx, ly;    // thread in CTA
  int bx0, by0;  // CTA pixel-block origin (blocked / in-WG)
  int Gx, Gy;    // threads of the logical grid per dimension
  __device__ __forceinline__ void at(const PmapCfg& m, int ix, int iy, int& x, int& y) const {
    if (m.map == kMapBlocked) {
      x = gx * m.cx + ix;
      y = gy * m.cy + iy;
    } else if (m.map == kMapInterleaved) {
      x = gx + ix * Gx;
      y = gy + iy * Gy;
    } else {  // interleaved within the work-group
      x = bx0 + lx + ix * m.wx;
      y = by0 + ly + iy * m.wy;
    }
  }
};

// ------------------------------------------------------------------ sepconv
template <bool LOCAL, int UNR>
__global__ void __launch_bounds__(256) sep_pmap(SepParams p, PmapCfg m, int nby) {
  extern __shared__ float tile[];
  // programmatic dependent launch (launch_sep_pmap): wait for the previous grid on the stream before
  // touching global memory (a no-op when launched without the attribute); each CTA releases the next
  // grid after its stores (end of the kernel), so the next launch overlaps this grid's tail.  A release
  // at the start let waiting CTAs of the next grid crowd the SMs that finished first: 6.15 vs 5.88 us
  // per 512^2 call; at the end 5.57 us (profiles/r02i_pdl_small_sepconv.txt)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int rx = p.rx, ry = p.ry;
  const int W = p.src.W, H = p.dst.H, b = blockIdx.z;
  const int TW = m.wx * m.cx + 2 * rx, TH = m.wy * m.cy + 2 * ry;
  PmapIndex ix_;
  ix_.lx = threadIdx.x;
  ix_.ly = threadIdx.y;
  ix_.gx = blockIdx.x * m.wx + threadIdx.x;
  ix_.Gx = gridDim.x * m.wx;
  ix_.Gy = nby * m.wy;
  ix_.bx0 = blockIdx.x * m.wx * m.cx;
  for (int byi = blockIdx.y; byi < nby; byi += gridDim.y) {  // gridDim.y <= 65535
    ix_.gy = byi * m.wy + threadIdx.y;
    ix_.by0 = byi * m.wy * m.cy;
    if (LOCAL) {
      __syncthreads();  // (previous block's readers done)
      const int nt = m.wx * m.wy, t0 = threadIdx.y * m.wx + threadIdx.x;
      // rows past the last output row's stencil are never read (and may lie outside a band buffer)
      const int rlim = H - 1 + ry - (ix_.by0 - ry);
      for (int i = t0; i < TW * TH; i += nt) {
        const int r = i / TW, c = i - r * TW;
        tile[i] = r <= rlim ? read_B(p.src, b, ix_.bx0 - rx + c, p.dst.y0 + ix_.by0 - ry + r) : 0.0f;
      }
      __syncthreads();
    }
    for (int iy = 0; iy < m.cy; ++iy)
      for (int ix = 0; ix < m.cx; ++ix) {
        int x, y;
        ix_.at(m, ix, iy, x, y);
        if (x >= W || y >= H) continue;
        const int gyy = p.dst.y0 + y;
        float acc = 0.0f;
#pragma unroll UNR
        for (int j = -ry; j <= ry; ++j) {
          float t = 0.0f;
          if (LOCAL) {
            const float* row = tile + (y - ix_.by0 + ry + j) * TW + (x - ix_.bx0 + rx);
#pragma unroll UNR
            for (int i = -rx; i <= rx; ++i) t = __fmaf_rn(p.fx[i + rx], row[i], t);
          } else {
#pragma unroll UNR
            for (int i = -rx; i <= rx; ++i) t = __fmaf_rn(p.fx[i + rx], read_B(p.src, b, x + i, gyy + j), t);
          }
          acc = __fmaf_rn(p.gy[j + ry], t, acc);
        }
        dst_row(p.dst, b, y)[x] = acc;
      }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------------------------------------------ Harris
// dx_B, dy_B at global (qx, qy) from a shared tile holding in_B over
// [ox, ox+TW) x [oy, oy+TH) (per-stage boundary as sobel_B in harris.cu)
__device__ __forceinline__ void sobel_T(const SrcView& s, const float* tile, int TW, int ox, int oy, int qx, int qy,
                                        float& dx, float& dy) {
  if (qx < 0 || qx >= s.W || qy < 0 || qy >= s.Hg) {
    if (s.border == kBorderConstant) { dx = 0.0f; dy = 0.0f; return; }
    qx = clampi(qx, 0, s.W - 1);
    qy = clampi(qy, 0, s.Hg - 1);
  }
  const float* c = tile + (qy - oy) * TW + (qx - ox);
  float hd[3], vd[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    hd[i] = __fsub_rn(c[(i - 1) * TW + 1], c[(i - 1) * TW - 1]);
    vd[i] = __fsub_rn(c[TW + i - 1], c[-TW + i - 1]);
  }
  dx = __fmaf_rn(2.0f, hd[1], __fadd_rn(hd[0], hd[2]));
  dy = __fmaf_rn(2.0f, vd[1], __fadd_rn(vd[0], vd[2]));
}

__device__ __forceinline__ void sobel_G(const SrcView& s, int b, int qx, int qy, float& dx, float& dy) {
  if (qx < 0 || qx >= s.W || qy < 0 || qy >= s.Hg) {
    if (s.border == kBorderConstant) { dx = 0.0f; dy = 0.0f; return; }
    qx = clampi(qx, 0, s.W - 1);
    qy = clampi(qy, 0, s.Hg - 1);
  }
  float hd[3], vd[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    hd[i] = __fsub_rn(read_B(s, b, qx + 1, qy - 1 + i), read_B(s, b, qx - 1, qy - 1 + i));
    vd[i] = __fsub_rn(read_B(s, b, qx - 1 + i, qy + 1), read_B(s, b, qx - 1 + i, qy - 1));
  }
  dx = __fmaf_rn(2.0f, hd[1], __fadd_rn(hd[0], hd[2]));
  dy = __fmaf_rn(2.0f, vd[1], __fadd_rn(vd[0], vd[2]));
}

template <bool LOCAL, int UNR>
__global__ void __launch_bounds__(256) harris_pmap(HarrisParams p, PmapCfg m, int nby) {
  extern __shared__ float tile[];
  const int a = p.block / 2, bb = p.block - 1 - a;
  const int W = p.src.W, H = p.dst.H, b = blockIdx.z;
  // input tile: pixel block + (a + 1) / (bb + 1) halo (window then Sobel)
  const int TW = m.wx * m.cx + a + bb + 2, TH = m.wy * m.cy + a + bb + 2;
  PmapIndex ix_;
  ix_.lx = threadIdx.x;
  ix_.ly = threadIdx.y;
  ix_.gx = blockIdx.x * m.wx + threadIdx.x;
  ix_.Gx = gridDim.x * m.wx;
  ix_.Gy = nby * m.wy;
  ix_.bx0 = blockIdx.x * m.wx * m.cx;
  for (int byi = blockIdx.y; byi < nby; byi += gridDim.y) {
    ix_.gy = byi * m.wy + threadIdx.y;
    ix_.by0 = byi * m.wy * m.cy;
    const int ox = ix_.bx0 - a - 1, oy = p.dst.y0 + ix_.by0 - a - 1;  // tile origin (global)
    if (LOCAL) {
      __syncthreads();
      const int nt = m.wx * m.wy, t0 = threadIdx.y * m.wx + threadIdx.x;
      const int rlim = (p.dst.y0 + H - 1 + bb + 1) - oy;  // (see sep_pmap)
      for (int i = t0; i < TW * TH; i += nt) {
        const int r = i / TW, c = i - r * TW;
        tile[i] = r <= rlim ? read_B(p.src, b, ox + c, oy + r) : 0.0f;
      }
      __syncthreads();
    }
    for (int iy = 0; iy < m.cy; ++iy)
      for (int ix = 0; ix < m.cx; ++ix) {
        int x, y;
        ix_.at(m, ix, iy, x, y);
        if (x >= W || y >= H) continue;
        const int gyy = p.dst.y0 + y;
        float sxx = 0.0f, sxy = 0.0f, syy = 0.0f;
#pragma unroll UNR
        for (int ty = -a; ty <= bb; ++ty) {
          float hxx = 0.0f, hxy = 0.0f, hyy = 0.0f;
#pragma unroll UNR
          for (int tx = -a; tx <= bb; ++tx) {
            float dx, dy;
            if (LOCAL) sobel_T(p.src, tile, TW, ox, oy, x + tx, gyy + ty, dx, dy);
            else sobel_G(p.src, b, x + tx, gyy + ty, dx, dy);
            hxx = __fmaf_rn(dx, dx, hxx);
            hxy = __fmaf_rn(dx, dy, hxy);
            hyy = __fmaf_rn(dy, dy, hyy);
          }
          if (ty == -a) { sxx = hxx; sxy = hxy; syy = hyy; }
          else { sxx = __fadd_rn(sxx, hxx); sxy = __fadd_rn(sxy, hxy); syy = __fadd_rn(syy, hyy); }
        }
        const float R = harris_R(sxx, sxy, syy, p.k);
        dst_row(p.dst, b, y)[x] = R;
        if (p.mask) p.mask[(int64_t)b * p.mbstride + (int64_t)y * p.mpitch + x] = R > p.threshold ? 1 : 0;
      }
  }
}

// ------------------------------------------------------------------ launchers
static inline dim3 pm_grid(const PmapCfg& m, int W, int H, int batch, int* nby) {
  *nby = (H + m.wy * m.cy - 1) / (m.wy * m.cy);
  return dim3((unsigned)((W + m.wx * m.cx - 1) / (m.wx * m.cx)), (unsigned)(*nby < 65535 ? *nby : 65535),
              (unsigned)batch);
}

cudaError_t launch_sep_pmap(const SepCall& c, const PmapCfg& m, cudaStream_t s) {
  SepParams p = make_sep_params(c, false);
  int nby;
  const dim3 grd = pm_grid(m, c.src.W, c.dst.H, c.batch, &nby);
  const dim3 blk(m.wx, m.wy);
  const size_t smem = m.local ? (size_t)(m.wx * m.cx + 2 * c.rx) * (m.wy * m.cy + 2 * c.ry) * sizeof(float) : 0;
#define ICL_PM_SEP(L, U)                                                                                    \
  if (m.local == L && m.unr == U) {                                                                        \
    if (smem > 48 * 1024) {                                                                                \
      cudaError_t e = cudaFuncSetAttribute(sep_pmap<L, U>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                           (int)smem);                                                     \
      if (e != cudaSuccess) return e;                                                                      \
    }                                                                                                      \
    cudaLaunchConfig_t cfg = {};                                                                           \
    cudaLaunchAttribute at[1];                                                                             \
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                                         \
    at[0].val.programmaticStreamSerializationAllowed = 1;                                                  \
    cfg.gridDim = grd; cfg.blockDim = blk; cfg.dynamicSmemBytes = smem; cfg.stream = s;                    \
    cfg.attrs = at; cfg.numAttrs = 1;                                                                      \
    cudaError_t e = cudaLaunchKernelEx(&cfg, sep_pmap<L, U>, p, m, nby);                                   \
    count_launch();                                                                                        \
    return e != cudaSuccess ? e : cudaGetLastError();                                                      \
  }
  ICL_PM_SEP(false, 1) ICL_PM_SEP(false, 4) ICL_PM_SEP(true, 1) ICL_PM_SEP(true, 4)
#undef ICL_PM_SEP
  return cudaErrorInvalidValue;
}

cudaError_t launch_harris_pmap(const HarrisCall& c, const PmapCfg& m, cudaStream_t s) {
  HarrisParams p;
  p.src = c.src;
  p.dst = c.dst;
  p.mask = c.mask;
  p.mpitch = c.mpitch;
  p.mbstride = c.mbstride;
  p.block = c.block;
  p.k = c.k;
  p.threshold = c.threshold;
  int nby;
  const dim3 grd = pm_grid(m, c.src.W, c.dst.H, c.batch, &nby);
  const dim3 blk(m.wx, m.wy);
  const int hal = c.block + 1;  // a + bb + 2
  const size_t smem = m.local ? (size_t)(m.wx * m.cx + hal) * (m.wy * m.cy + hal) * sizeof(float) : 0;
#define ICL_PM_HAR(L, U)                                                                                    \
  if (m.local == L && m.unr == U) {                                                                        \
    if (smem > 48 * 1024) {                                                                                \
      cudaError_t e = cudaFuncSetAttribute(harris_pmap<L, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                           (int)smem);                                                     \
      if (e != cudaSuccess) return e;                                                                      \
    }                                                                                                      \
    harris_pmap<L, U><<<grd, blk, smem, s>>>(p, m, nby);                                                   \
    count_launch();                                                                                        \
    return cudaGetLastError();                                                                             \
  }
  ICL_PM_HAR(false, 1) ICL_PM_HAR(false, 4) ICL_PM_HAR(true, 1) ICL_PM_HAR(true, 4)
#undef ICL_PM_HAR
  return cudaErrorInvalidValue;
}

}  // namespace icl
