// harris.cu -- Harris corner response variants (§6;
// Table 4 "Sobel" kernel and Table 5 "Harris" kernel, lines 651-687).
//
// Per-stage semantics (R6-R10): dx/dy are images with their own
// boundary (clamp: dx(clamp(q)); constant: 0 outside), the input is read
// with in_B.  All variants use the SAME fp32 operation order per output, so
// they are bit-identical (and so are row-band splits):
//   hd(r) = in(c+1,r) - in(c-1,r)  (r = y-1, y, y+1);  vd(c) = in(c,y+1) - in(c,y-1)
//   dx = fma(2, hd(y), hd(y-1) + hd(y+1));            dy = fma(2, vd(x), vd(x-1) + vd(x+1))
// (differences first: the rounding error of dx/dy is then relative to the
// gradient terms, not to the pixel level -- DESIGN.md "Harris numerics")
//   H*(r) = fma-chain over tx = -a..b of the products (from 0.0f)
//   S*    = H*(y-a) + H*(y-a+1) + ... + H*(y+b)       (left to right)
//   R     = fma(-k, tr*tr, fma(Sxx, Syy, -(Sxy*Sxy))),  tr = Sxx + Syy
//   mask  = R > threshold
#include "common.cuh"
#include "internal.h"
#include "harris_stream.cuh"

namespace icl {

// dx_B, dy_B at (qx, qy) global (per-stage boundary).
__device__ __forceinline__ void sobel_B(const SrcView& s, int b, int qx, int qy, float& dx, float& dy) {
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

// --------------------------------------------------------------------------
// Variant "naive_direct": one logical thread per pixel; the window loops of
// Table 5 ("Loop 1/2") with dx/dy recomputed from global memory (no
// intermediate images, no local memory).
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) harris_naive(HarrisParams p) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int ly = blockIdx.y * blockDim.y + threadIdx.y;
  const int b = blockIdx.z;
  if (x >= p.src.W || ly >= p.dst.H) return;
  const int y = p.dst.y0 + ly;
  const int a = p.block / 2, bb = p.block - 1 - a;
  float sxx = 0.0f, sxy = 0.0f, syy = 0.0f;
  for (int ty = -a; ty <= bb; ++ty) {
    float hxx = 0.0f, hxy = 0.0f, hyy = 0.0f;
    for (int tx = -a; tx <= bb; ++tx) {
      float dx, dy;
      sobel_B(p.src, b, x + tx, y + ty, dx, dy);
      hxx = __fmaf_rn(dx, dx, hxx);
      hxy = __fmaf_rn(dx, dy, hxy);
      hyy = __fmaf_rn(dy, dy, hyy);
    }
    if (ty == -a) { sxx = hxx; sxy = hxy; syy = hyy; }
    else { sxx = __fadd_rn(sxx, hxx); sxy = __fadd_rn(sxy, hxy); syy = __fadd_rn(syy, hyy); }
  }
  const float R = harris_R(sxx, sxy, syy, p.k);
  dst_row(p.dst, b, ly)[x] = R;
  if (p.mask) p.mask[(int64_t)b * p.mbstride + (int64_t)ly * p.mpitch + x] = R > p.threshold ? 1 : 0;
}

// ----------------------------------------------------------------- launchers
static HarrisParams make_params(const HarrisCall& c) {
  HarrisParams p;
  p.src = c.src;
  p.dst = c.dst;
  p.mask = c.mask;
  p.mpitch = c.mpitch;
  p.mbstride = c.mbstride;
  p.block = c.block;
  p.k = c.k;
  p.threshold = c.threshold;
  return p;
}

cudaError_t launch_harris_naive(const HarrisCall& c, cudaStream_t s) {
  HarrisParams p = make_params(c);
  dim3 blk(32, 8), grd((c.src.W + 31) / 32, (c.dst.H + 7) / 8, c.batch);
  harris_naive<<<grd, blk, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

template <int NT, int VEC>
cudaError_t dispatch_hs(const HarrisParams& p, int batch, int S, cudaStream_t s);
extern template cudaError_t dispatch_hs<32, 4>(const HarrisParams&, int, int, cudaStream_t);
extern template cudaError_t dispatch_hs<64, 4>(const HarrisParams&, int, int, cudaStream_t);
extern template cudaError_t dispatch_hs<128, 4>(const HarrisParams&, int, int, cudaStream_t);
extern template cudaError_t dispatch_hs<64, 1>(const HarrisParams&, int, int, cudaStream_t);
template <int NW>
cudaError_t dispatch_hshfl(const HarrisParams& p, int batch, int S, cudaStream_t s);
extern template cudaError_t dispatch_hshfl<1>(const HarrisParams&, int, int, cudaStream_t);
extern template cudaError_t dispatch_hshfl<2>(const HarrisParams&, int, int, cudaStream_t);
extern template cudaError_t dispatch_hshfl<4>(const HarrisParams&, int, int, cudaStream_t);

template <int NW>
cudaError_t dispatch_hshfl_tma(const HarrisParams& p, int batch, int S, cudaStream_t s);
extern template cudaError_t dispatch_hshfl_tma<2>(const HarrisParams&, int, int, cudaStream_t);

cudaError_t launch_harris_shfl(const HarrisCall& c, int nw, int S, cudaStream_t s, bool tma) {
  HarrisParams p = make_params(c);
  if (tma) return nw == 2 ? dispatch_hshfl_tma<2>(p, c.batch, S, s) : cudaErrorInvalidValue;
  if (nw == 1) return dispatch_hshfl<1>(p, c.batch, S, s);
  if (nw == 2) return dispatch_hshfl<2>(p, c.batch, S, s);
  if (nw == 4) return dispatch_hshfl<4>(p, c.batch, S, s);
  return cudaErrorInvalidValue;
}

template <int NW, int UNR, bool HF = false>
cudaError_t dispatch_hslide(const HarrisParams& p, int batch, int S, cudaStream_t s);
extern template cudaError_t dispatch_hslide<2, 1, true>(const HarrisParams&, int, int, cudaStream_t);
extern template cudaError_t dispatch_hslide<4, 1, true>(const HarrisParams&, int, int, cudaStream_t);
extern template cudaError_t dispatch_hslide<2, 1>(const HarrisParams&, int, int, cudaStream_t);
extern template cudaError_t dispatch_hslide<4, 1>(const HarrisParams&, int, int, cudaStream_t);
extern template cudaError_t dispatch_hslide<2, 2>(const HarrisParams&, int, int, cudaStream_t);
extern template cudaError_t dispatch_hslide<4, 2>(const HarrisParams&, int, int, cudaStream_t);

// unr: the step loop of interior CTAs unrolled by 1 or 2 (two independent Sobel rows in flight)
cudaError_t launch_harris_slide(const HarrisCall& c, int nw, int unr, int S, cudaStream_t s) {
  HarrisParams p = make_params(c);
  if (unr == 3) {  // "slide2": products' horizontal pair sums first (harris_slide.cuh HFIRST)
    if (nw == 2) return dispatch_hslide<2, 1, true>(p, c.batch, S, s);
    if (nw == 4) return dispatch_hslide<4, 1, true>(p, c.batch, S, s);
    return cudaErrorInvalidValue;
  }
  if (nw == 2) return unr == 2 ? dispatch_hslide<2, 2>(p, c.batch, S, s) : dispatch_hslide<2, 1>(p, c.batch, S, s);
  if (nw == 4) return unr == 2 ? dispatch_hslide<4, 2>(p, c.batch, S, s) : dispatch_hslide<4, 1>(p, c.batch, S, s);
  return cudaErrorInvalidValue;
}

// The tuner's per-pixel scale for Harris variants that re-associate the window sums
// (SURVEY.md §8(c) tolerance): D(p) = |Sxx Syy| + Sxy^2 + k (Sxx + Syy)^2, the magnitude of
// the terms that cancel in R, from the naive per-output order, into a compact W x H x batch
// buffer.
__global__ void __launch_bounds__(256) harris_dhat(HarrisParams p, float* out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int ly = blockIdx.y * blockDim.y + threadIdx.y;
  const int b = blockIdx.z;
  if (x >= p.src.W || ly >= p.dst.H) return;
  const int y = p.dst.y0 + ly;
  const int a = p.block / 2, bb = p.block - 1 - a;
  float sxx = 0.0f, sxy = 0.0f, syy = 0.0f;
  for (int ty = -a; ty <= bb; ++ty)
    for (int tx = -a; tx <= bb; ++tx) {
      float dx, dy;
      sobel_B(p.src, b, x + tx, y + ty, dx, dy);
      sxx = __fmaf_rn(dx, dx, sxx);
      sxy = __fmaf_rn(dx, dy, sxy);
      syy = __fmaf_rn(dy, dy, syy);
    }
  const float tr = sxx + syy;
  out[((int64_t)b * p.dst.H + ly) * p.src.W + x] = fabsf(sxx * syy) + sxy * sxy + fabsf(p.k) * tr * tr;
}

cudaError_t launch_harris_dhat(const HarrisCall& c, float* out, cudaStream_t s) {
  HarrisParams p = make_params(c);
  dim3 blk(32, 8), grd((c.src.W + 31) / 32, (c.dst.H + 7) / 8, c.batch);
  harris_dhat<<<grd, blk, 0, s>>>(p, out);
  return cudaGetLastError();
}

cudaError_t launch_harris_stream(const HarrisCall& c, int nt, int vec, int S, cudaStream_t s) {
  HarrisParams p = make_params(c);
  if (vec == 4) {
    if (nt == 32) return dispatch_hs<32, 4>(p, c.batch, S, s);
    if (nt == 64) return dispatch_hs<64, 4>(p, c.batch, S, s);
    if (nt == 128) return dispatch_hs<128, 4>(p, c.batch, S, s);
  } else if (vec == 1 && nt == 64) {
    return dispatch_hs<64, 1>(p, c.batch, S, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace icl
