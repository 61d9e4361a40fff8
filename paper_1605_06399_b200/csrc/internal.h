// internal.h -- host-side declarations shared by the C-ABI layer (api.cu) and
// the kernel translation units.  Product code only.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <vector>

#include "../../include/icl.h"
#include "common.cuh"

namespace icl {

void count_launch();

struct SepCall {
  SrcView src;
  DstView dst;
  int batch;
  int rx, ry;
  const float* fx;  // host, 2rx+1
  const float* gy;  // host, 2ry+1
  void* workspace;
  size_t workspace_bytes;
  // the src rows cover R = max(rx, ry) rows around the dst rows (always true without a band):
  // the fused variants pad the taps to R and READ those rows (times a zero tap), so in a band
  // holding only ry halo rows they are ineligible (they would read outside the band buffer)
  bool pad_rows_ok;
};

struct HarrisCall {
  SrcView src;
  DstView dst;      // response
  char* mask;       // nullable
  int64_t mpitch, mbstride;
  int batch;
  int block;
  float k;
  float threshold;
  // restrict dispatch to the variants sharing the naive per-output fp32 order (the fused chain's
  // two-pass schedule and the peer bands, whose edge kernels use that order): bit-identical
  bool naive_order;
};

struct NlmCall {
  SrcView src;
  DstView dst;
  int batch;
  int P;      // patch radius
  int S;      // search radius
  float h;    // +inf allowed
  float coef; // log2(e) / ((2P+1)^2 h^2), 0 when h = +inf
};

// non-separable convolution of an 8-bit image (src views bytes)
struct Conv2dCall {
  SrcView src;  // uint8 pixels: base / pitch / bstride in bytes
  DstView dst;  // fp32
  int batch;
  int r;        // radius, 0..3
  float f[49];  // (2r+1)^2 taps, row j major
};

// error reporting shared by the library's translation units (api.cu)
icl_status report_error(icl_status st, const char* msg);

// texture ("image memory") variants, tex.cu
bool tex_eligible(const SrcView& s, int64_t rows, int batch, int elem, bool clamp_or_zero);
cudaError_t launch_sep_tex(const SepCall& c, cudaStream_t s);
cudaError_t launch_conv2d_tex(const Conv2dCall& c, cudaStream_t s);

// sepconv
cudaError_t launch_sep_naive_direct(const SepCall& c, cudaStream_t s);
cudaError_t launch_sep_naive_2pass(const SepCall& c, cudaStream_t s);
size_t sep_2pass_workspace(int64_t W, int64_t H, int64_t batch, int ry);
cudaError_t launch_sep_stream(const SepCall& c, int nt, int vec, int S, cudaStream_t s);
size_t sep_stream_smem_bytes(int nt, int R);
cudaError_t launch_sep_bulk(const SepCall& c, int nt, int S, cudaStream_t s);
cudaError_t launch_sep_tile128(const SepCall& c, cudaStream_t s);
cudaError_t launch_sep_tile(const SepCall& c, bool persistent, cudaStream_t s);

// harris
cudaError_t launch_harris_naive(const HarrisCall& c, cudaStream_t s);
cudaError_t launch_harris_stream(const HarrisCall& c, int nt, int vec, int S, cudaStream_t s);
cudaError_t launch_harris_shfl(const HarrisCall& c, int nw, int S, cudaStream_t s, bool tma = false);
cudaError_t launch_harris_slide(const HarrisCall& c, int nw, int unr, int S, cudaStream_t s);
cudaError_t launch_harris_dhat(const HarrisCall& c, float* out, cudaStream_t s);
// two-filter chain (blur_harris.cu): separable blur (radius <= 3) then Harris (block <= 5) in one pass
cudaError_t launch_blur_harris(const HarrisCall& h, const SrcView& raw, const float* fx, int rx, const float* gy,
                               int ry, int S, cudaStream_t s);

// nlm
cudaError_t launch_nlm_naive(const NlmCall& c, cudaStream_t s);
cudaError_t launch_nlm_tiled(const NlmCall& c, int tw, int th, cudaStream_t s);
cudaError_t launch_nlm_boxsum(const NlmCall& c, int variant, cudaStream_t s);
cudaError_t launch_nlm_r8(const NlmCall& c, cudaStream_t s);
cudaError_t launch_nlm_r16(const NlmCall& c, cudaStream_t s);
cudaError_t launch_nlm_x2(const NlmCall& c, cudaStream_t s);
cudaError_t launch_nlm_w(const NlmCall& c, int unroll, cudaStream_t s);
cudaError_t launch_nlm_sym(const NlmCall& c, cudaStream_t s);
cudaError_t launch_nlm_sym_ring(const NlmCall& c, cudaStream_t s);
cudaError_t launch_nlm_sym8(const NlmCall& c, cudaStream_t s);
// conv2d (u8)
cudaError_t launch_conv2d_naive(const Conv2dCall& c, cudaStream_t s);
cudaError_t launch_conv2d_tile(const Conv2dCall& c, int rows_per_thread, bool persistent, cudaStream_t s);

// auto-tuner performance model (ann.cu): phase 1 runs n1 random configurations,
// phase 2 trains the surrogate on the ok ones and runs the topk best-predicted
// unmeasured ones; returns the number of ok measurements.
constexpr int kAnnMinSamples = 10;
int ann_search(int ncfg, int nf, const double* feats, const std::function<bool(int, double*)>& evaluate, int n1,
               int topk, uint64_t seed, std::vector<int>* evaluated, int* best, double* best_val);

// 3-D separable convolution (sep3d.cu); variant 0 naive, 1 tile<R>.  A volume's z axis is the
// icl_image batch axis (slice stride = batch stride).
struct Sep3Params {
  const char* src;
  int64_t spitch, sslice;  // bytes
  char* dst;
  int64_t dpitch, dslice;
  int W, H, D;
  int border;
  float cval;
  int rx, ry, rz;
  float fx[2 * 7 + 1], gy[2 * 7 + 1], hz[2 * 7 + 1];  // padded to R in tile<R>
};
bool sep3d_tile_supported(int R);
cudaError_t launch_sep3d(const Sep3Params& p, int variant, cudaStream_t s);

// synthetic inputs
cudaError_t launch_fill_uniform(float* base, int64_t W, int64_t H, int64_t pitch, int64_t batch,
                                int64_t bstride, uint64_t seed, int64_t row0, cudaStream_t s);

// icl_harris restricted to the naive-order variants (HarrisCall::naive_order)
icl_status harris_naive_order(const icl_image* src, const icl_image* response, int block, float k, icl_border border,
                              float border_value, const icl_image* mask, float threshold, const icl_band* band,
                              void* stream);

// The paper's Table-1 axes as a run-time configuration of one-pixel-per-logical-thread kernels
// (pmap.cu): CTA (wx, wy), coarsening (cx, cy), mapping (Fig. 4), local memory, unroll factor.
enum { kMapBlocked = 0, kMapInterleaved = 1, kMapInWG = 2 };
struct PmapCfg {
  int wx, wy, cx, cy, map, local, unr;
};
cudaError_t launch_sep_pmap(const SepCall& c, const PmapCfg& m, cudaStream_t s);
cudaError_t launch_harris_pmap(const HarrisCall& c, const PmapCfg& m, cudaStream_t s);

}  // namespace icl

// An NCCL symmetric window (icl_comm_window_register): `win` is the ncclWindow_t (a device-
// readable descriptor; kernels resolve a peer's address with ncclGetPeerPointer)
struct icl_window {
  void* win;
  void* buf;
  size_t bytes;
  int rank, nranks;
};
