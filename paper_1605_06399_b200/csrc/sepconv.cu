// sepconv.cu -- separable convolution variants (§6,
// Table 2; Halide-style fusion PAPER.md:701-704).
//
// Every variant evaluates, for each output pixel, the SAME fp32 operation
// sequence (R16):
//     t_j  = fma-chain over i = -R..R of  fx[i] * in_B(x+i, y+j)   (from 0.0f)
//     out  = fma-chain over j = -R..R of  gy[j] * t_j               (from 0.0f)
// so the naive, two-pass and fused variants are bit-identical, and so are
// row-band splits.  Fused variants use taps zero-padded to R = max(rx, ry);
// fma(0, v, acc) == acc for finite v, so padding does not change values.
#include "common.cuh"
#include "internal.h"
#include "sepconv_stream.cuh"

namespace icl {

// --------------------------------------------------------------------------
// Variant "naive_direct": one logical thread per output pixel (ImageCL's flat
// thread grid), direct global loads with a boundary check
// per read -- the A6 "naive OpenCL" baseline of SURVEY.md §2a.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) sep_naive_direct(SepParams p) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int ly = blockIdx.y * blockDim.y + threadIdx.y;
  const int b = blockIdx.z;
  if (x >= p.src.W || ly >= p.dst.H) return;
  const int gy = p.dst.y0 + ly;
  float acc = 0.0f;
  for (int j = -p.ry; j <= p.ry; ++j) {
    float t = 0.0f;
    for (int i = -p.rx; i <= p.rx; ++i) t = __fmaf_rn(p.fx[i + p.rx], read_B(p.src, b, x + i, gy + j), t);
    acc = __fmaf_rn(p.gy[j + p.ry], t, acc);
  }
  dst_row(p.dst, b, ly)[x] = acc;
}

// --------------------------------------------------------------------------
// Variant "naive_2pass": the paper's R kernel then C kernel (Table 2), with
// the fp32 intermediate in global memory (workspace).  Intermediate row lt
// holds global row dst.y0 - ry + lt, so its boundary semantics are those of
// the extended input (reading a constant row gives the fma chain over c:
// DESIGN.md R5).
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) sep_row_pass(SepParams p, float* tmp, int64_t tpitch, int64_t tbstride,
                                                    int trows) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int lt = blockIdx.y * blockDim.y + threadIdx.y;
  const int b = blockIdx.z;
  if (x >= p.src.W || lt >= trows) return;
  const int gy = p.dst.y0 - p.ry + lt;
  float t = 0.0f;
  for (int i = -p.rx; i <= p.rx; ++i) t = __fmaf_rn(p.fx[i + p.rx], read_B(p.src, b, x + i, gy), t);
  tmp[(int64_t)b * tbstride + (int64_t)lt * tpitch + x] = t;
}

__global__ void __launch_bounds__(256) sep_col_pass(SepParams p, const float* __restrict__ tmp, int64_t tpitch,
                                                    int64_t tbstride) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int ly = blockIdx.y * blockDim.y + threadIdx.y;
  const int b = blockIdx.z;
  if (x >= p.src.W || ly >= p.dst.H) return;
  const float* tb = tmp + (int64_t)b * tbstride + x;
  float acc = 0.0f;
  for (int j = 0; j <= 2 * p.ry; ++j) acc = __fmaf_rn(p.gy[j], __ldg(tb + (int64_t)(ly + j) * tpitch), acc);
  dst_row(p.dst, b, ly)[x] = acc;
}

// ----------------------------------------------------------------- launchers
cudaError_t launch_sep_naive_direct(const SepCall& c, cudaStream_t s) {
  SepParams p = make_sep_params(c, false);
  dim3 blk(32, 8), grd((c.src.W + 31) / 32, (c.dst.H + 7) / 8, c.batch);
  sep_naive_direct<<<grd, blk, 0, s>>>(p);
  count_launch();
  return cudaGetLastError();
}

size_t sep_2pass_workspace(int64_t W, int64_t H, int64_t batch, int ry) {
  const int64_t tpitch = (W + 31) / 32 * 32;
  return (size_t)(tpitch * (H + 2 * ry) * batch * sizeof(float));
}

cudaError_t launch_sep_naive_2pass(const SepCall& c, cudaStream_t s) {
  SepParams p = make_sep_params(c, false);
  const int64_t tpitch = ((int64_t)c.src.W + 31) / 32 * 32;
  const int trows = c.dst.H + 2 * c.ry;
  const int64_t tbstride = tpitch * trows;
  float* tmp = static_cast<float*>(c.workspace);
  dim3 blk(32, 8);
  dim3 g1((c.src.W + 31) / 32, (trows + 7) / 8, c.batch);
  sep_row_pass<<<g1, blk, 0, s>>>(p, tmp, tpitch, tbstride, trows);
  count_launch();
  dim3 g2((c.src.W + 31) / 32, (c.dst.H + 7) / 8, c.batch);
  sep_col_pass<<<g2, blk, 0, s>>>(p, tmp, tpitch, tbstride);
  count_launch();
  return cudaGetLastError();
}

template <int NT, int VEC>
cudaError_t dispatch_stream(const SepParams& p, int R, int batch, int S, cudaStream_t s);
extern template cudaError_t dispatch_stream<32, 4>(const SepParams&, int, int, int, cudaStream_t);
extern template cudaError_t dispatch_stream<64, 4>(const SepParams&, int, int, int, cudaStream_t);
extern template cudaError_t dispatch_stream<128, 4>(const SepParams&, int, int, int, cudaStream_t);
extern template cudaError_t dispatch_stream<64, 1>(const SepParams&, int, int, int, cudaStream_t);
extern template cudaError_t dispatch_stream<256, 4>(const SepParams&, int, int, int, cudaStream_t);
template <int NT>
cudaError_t dispatch_bulk(const SepParams& p, int R, int batch, int S, cudaStream_t s);
extern template cudaError_t dispatch_bulk<32>(const SepParams&, int, int, int, cudaStream_t);
extern template cudaError_t dispatch_bulk<64>(const SepParams&, int, int, int, cudaStream_t);
extern template cudaError_t dispatch_bulk<128>(const SepParams&, int, int, int, cudaStream_t);

cudaError_t launch_sep_bulk(const SepCall& c, int nt, int S, cudaStream_t s) {
  SepParams p = make_sep_params(c, true);
  const int R = c.rx > c.ry ? c.rx : c.ry;
  if (nt == 32) return dispatch_bulk<32>(p, R, c.batch, S, s);
  if (nt == 64) return dispatch_bulk<64>(p, R, c.batch, S, s);
  if (nt == 128) return dispatch_bulk<128>(p, R, c.batch, S, s);
  return cudaErrorInvalidValue;
}

size_t sep_stream_smem_bytes(int nt, int R) {
  const int P = 2 * R + 1;
  const int RB = P * ((4 + P - 1) / P);
  const int NSR = RB * (RB <= 8 ? 3 : 2);
  const int HP = ((R + 3) / 4) * 4;
  const size_t blk = ((size_t)RB * (4 * nt + 2 * HP) * 4 + 127) / 128 * 128;  // 128-byte block slots
  return (size_t)(NSR / RB) * blk + 64;
}

bool make_view_tmap(const SrcView& src, int batch, int box_w, int box_h, CUtensorMap* map);

// The source of a sepconv call as a 3-D tensor map for the TMA variants (sepconv_stream.cuh).
bool make_src_tmap(const SepParams& p, int batch, int box_w, int box_h, CUtensorMap* map) {
  return make_view_tmap(p.src, batch, box_w, box_h, map);
}

// Any source view as a 3-D tensor map (x = W columns, y = the rows held locally, z = images),
// box box_w x box_h x 1, zero fill out of bounds (also the NLM sym_tmem tiles, nlm_sym.cuh).
bool make_view_tmap(const SrcView& src, int batch, int box_w, int box_h, CUtensorMap* map) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess) fn = nullptr;
    return reinterpret_cast<EncodeFn>(fn);
  }();
  if (!enc) return false;
  const cuuint64_t rows = (cuuint64_t)src.Hl;
  const cuuint64_t dims[3] = {(cuuint64_t)src.W, rows, (cuuint64_t)batch};
  const cuuint64_t bstride = batch > 1 ? (cuuint64_t)src.bstride : (cuuint64_t)src.pitch * rows;
  const cuuint64_t strides[2] = {(cuuint64_t)src.pitch, bstride};
  const cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<char*>(src.base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NT>
cudaError_t dispatch_stream_tma(const SepParams& p, int R, int batch, int S, cudaStream_t s);
extern template cudaError_t dispatch_stream_tma<32>(const SepParams&, int, int, int, cudaStream_t);

cudaError_t launch_sep_stream(const SepCall& c, int nt, int vec, int S, cudaStream_t s) {
  SepParams p = make_sep_params(c, true);
  const int R = c.rx > c.ry ? c.rx : c.ry;
  if (vec == 7) return nt == 32 ? dispatch_stream_tma<32>(p, R, c.batch, S, s) : cudaErrorInvalidValue;  // TMA
  if (vec == 4) {
    if (nt == 32) return dispatch_stream<32, 4>(p, R, c.batch, S, s);
    if (nt == 64) return dispatch_stream<64, 4>(p, R, c.batch, S, s);
    if (nt == 128) return dispatch_stream<128, 4>(p, R, c.batch, S, s);
    if (nt == 256) return dispatch_stream<256, 4>(p, R, c.batch, S, s);
  } else if (vec == 1 && nt == 64) {
    return dispatch_stream<64, 1>(p, R, c.batch, S, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace icl
