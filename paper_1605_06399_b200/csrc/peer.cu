// peer.cu -- row-band sharding with the halo read IN the filter kernel from the
// neighbouring ranks' memory ("in-kernel NVLink halo
// reads instead of send/recv ... the edge CTAs load neighbor rows directly,
// which fuses the 'collective' into the filter kernel").
//
// Ranks of one node map each other's band buffers with CUDA IPC
// (icl_ipc_get_handle / icl_ipc_open; the 64-byte handles travel over any
// host channel, e.g. the torch process group).  A rank's buffer then holds
// ONLY its own rows -- no halo rows, no staging, no send/recv, no pack /
// unpack: the rows that need no halo run through the ordinary icl_sepconv
// kernels on the own band, and the edge rows run through sep_edge_peer, whose
// loads resolve every input row to the own band or to the up / down
// neighbour's band (peer loads over NVLink on a multi-GPU node).  The global
// boundary is applied before the resolution, in global coordinates, so the
// stitched result equals the unsharded call bit for bit (same fp32 chains as
// every sepconv variant, R16).
//
// Ordering contract: the neighbours' rows must be written before this call's
// kernels run and must not be overwritten until they finish -- the caller
// brackets the call with a barrier across the ranks (the pattern of a
// static, pre-sharded input such as BASELINE configs[3]).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>

#include <algorithm>
#include <cstring>

#include "../../include/icl.h"
#include "common.cuh"
#include "internal.h"
#ifdef ICL_HAVE_NCCL_DEVICE
#include <nccl.h>
#include <nccl_device.h>
#endif

namespace icl {
namespace {

// NCCL symmetric-window neighbours (icl_*_window): the host fills a segment's base with
// kWinFake + (byte offset in the peer's window) and the kernel replaces it by the peer's address
// from ncclGetPeerPointer -- resolved on the device, as the window API defines it.
constexpr uintptr_t kWinFake = (uintptr_t)1 << 46;

__device__ __forceinline__ const char* win_resolve(void* win, int peer, const char* fake) {
#ifdef ICL_HAVE_NCCL_DEVICE
  if (win && peer >= 0)
    return static_cast<const char*>(
        ncclGetPeerPointer(static_cast<ncclWindow_t>(win), (size_t)((uintptr_t)fake - kWinFake), peer));
#endif
  return fake;
}

struct RowSeg {     // rows [y0, y1) of one band buffer
  const char* base; // row y0 of image 0
  int64_t pitch, bstride;
  int y0, y1;
};

struct EdgeParams {
  RowSeg seg[3];  // up, own, down (empty: y0 == y1)
  void* win;      // ncclWindow_t of icl_sepconv_window (nullptr: plain pointers)
  int wpeer[3];   // per segment: the window peer (< 0: plain pointer)
  int W, Hg;
  int border;
  float cval;
  int rx, ry;
  float fx[2 * kMaxRadius + 1], gy[2 * kMaxRadius + 1];
  char* dst;      // output row `out_y0` of image 0
  int64_t dpitch, dbstride;
  int out_y0, out_y1;  // global output rows of this launch
};

constexpr int kEdgeTW = 128;  // output columns per CTA (one per thread)
constexpr int kEdgeCH = 16;   // output rows per CTA

// in_B(x, gy) row pointer after the global boundary; nullptr -> the constant row
__device__ __forceinline__ const float* edge_row(const EdgeParams& p, const char* const* base, int b, int gy) {
  if (gy < 0 || gy >= p.Hg) {
    if (p.border == kBorderConstant) return nullptr;
    gy = clampi(gy, 0, p.Hg - 1);
  }
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const RowSeg& g = p.seg[s];
    if (gy >= g.y0 && gy < g.y1)
      return reinterpret_cast<const float*>(base[s] + (int64_t)b * g.bstride + (int64_t)(gy - g.y0) * g.pitch);
  }
  return nullptr;  // unreachable for a validated call
}

// One CTA: kEdgeTW columns x kEdgeCH output rows.  Row pass of every input row
// the chunk needs into shared memory (the fp32 chain over i), then the column
// pass (the chain over j) -- the per-output operation order of every sepconv
// variant.  Input rows come from the own band or straight from a peer's band.
__global__ void __launch_bounds__(kEdgeTW) sep_edge_peer(EdgeParams p) {
  extern __shared__ float sm[];
  const int tid = threadIdx.x;
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * kEdgeTW;
  const int y0 = p.out_y0 + blockIdx.y * kEdgeCH;
  const int y1 = min(y0 + kEdgeCH, p.out_y1);
  const int NR = (y1 - y0) + 2 * p.ry;  // input rows
  const int RL = kEdgeTW + 2 * p.rx;
  float* raw = sm;                      // one input row (+ rx columns each side)
  float* t = sm + RL + 2 * kMaxRadius;  // NR row-pass rows
  const int x = x0 + tid;
  const char* base[3];
#pragma unroll
  for (int s = 0; s < 3; ++s) base[s] = win_resolve(p.win, p.wpeer[s], p.seg[s].base);
  for (int k = 0; k < NR; ++k) {
    const float* row = edge_row(p, base, b, y0 - p.ry + k);
    __syncthreads();
    for (int c = tid; c < RL; c += kEdgeTW) {
      int xx = x0 - p.rx + c;
      float v;
      if (!row) v = p.cval;
      else if (xx < 0 || xx >= p.W) v = p.border == kBorderConstant ? p.cval : row[clampi(xx, 0, p.W - 1)];
      else v = row[xx];
      raw[c] = v;
    }
    __syncthreads();
    float a = 0.0f;
    for (int i = 0; i <= 2 * p.rx; ++i) a = __fmaf_rn(p.fx[i], raw[tid + i], a);
    t[k * kEdgeTW + tid] = a;
  }
  __syncthreads();
  if (x >= p.W) return;
  for (int y = y0; y < y1; ++y) {
    const int k0 = y - y0;
    float acc = 0.0f;
    for (int j = 0; j <= 2 * p.ry; ++j) acc = __fmaf_rn(p.gy[j], t[(k0 + j) * kEdgeTW + tid], acc);
    reinterpret_cast<float*>(p.dst + (int64_t)b * p.dbstride + (int64_t)(y - p.out_y0) * p.dpitch)[x] = acc;
  }
}

// Harris edge rows of a band whose input rows come from the own band or a
// neighbour's band: the naive Harris kernel's per-output operations (the one
// fp32 order of every Harris variant, harris.cu) with the row resolver above.
struct HarrisEdgeParams {
  RowSeg seg[3];
  void* win;     // (see EdgeParams)
  int wpeer[3];
  int W, Hg;
  int border;
  float cval;
  int block;
  float k, threshold;
  char* dst;  // response row out_y0, image 0
  int64_t dpitch, dbstride;
  char* mask;  // nullable, row out_y0, image 0
  int64_t mpitch, mbstride;
  int out_y0, out_y1;
};

__device__ __forceinline__ float hread(const HarrisEdgeParams& p, const char* const* base, int b, int x, int y) {
  if (x < 0 || x >= p.W || y < 0 || y >= p.Hg) {
    if (p.border == kBorderConstant) return p.cval;
    x = clampi(x, 0, p.W - 1);
    y = clampi(y, 0, p.Hg - 1);
  }
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const RowSeg& g = p.seg[s];
    if (y >= g.y0 && y < g.y1)
      return reinterpret_cast<const float*>(base[s] + (int64_t)b * g.bstride + (int64_t)(y - g.y0) * g.pitch)[x];
  }
  return 0.0f;  // unreachable for a validated call
}

__device__ __forceinline__ void hsobel(const HarrisEdgeParams& p, const char* const* base, int b, int qx, int qy,
                                       float& dx, float& dy) {
  if (qx < 0 || qx >= p.W || qy < 0 || qy >= p.Hg) {  // per-stage boundary of dx / dy
    if (p.border == kBorderConstant) { dx = 0.0f; dy = 0.0f; return; }
    qx = clampi(qx, 0, p.W - 1);
    qy = clampi(qy, 0, p.Hg - 1);
  }
  float hd[3], vd[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    hd[i] = __fsub_rn(hread(p, base, b, qx + 1, qy - 1 + i), hread(p, base, b, qx - 1, qy - 1 + i));
    vd[i] = __fsub_rn(hread(p, base, b, qx - 1 + i, qy + 1), hread(p, base, b, qx - 1 + i, qy - 1));
  }
  dx = __fmaf_rn(2.0f, hd[1], __fadd_rn(hd[0], hd[2]));
  dy = __fmaf_rn(2.0f, vd[1], __fadd_rn(vd[0], vd[2]));
}

__global__ void __launch_bounds__(256) harris_edge_peer(HarrisEdgeParams p) {
  const int x = blockIdx.x * 32 + (threadIdx.x & 31);
  const int y = p.out_y0 + blockIdx.y * 8 + (threadIdx.x >> 5);
  const int b = blockIdx.z;
  if (x >= p.W || y >= p.out_y1) return;
  const char* base[3];
#pragma unroll
  for (int s = 0; s < 3; ++s) base[s] = win_resolve(p.win, p.wpeer[s], p.seg[s].base);
  const int a = p.block / 2, bb = p.block - 1 - a;
  float sxx = 0.0f, sxy = 0.0f, syy = 0.0f;
  for (int ty = -a; ty <= bb; ++ty) {
    float hxx = 0.0f, hxy = 0.0f, hyy = 0.0f;
    for (int tx = -a; tx <= bb; ++tx) {
      float dx, dy;
      hsobel(p, base, b, x + tx, y + ty, dx, dy);
      hxx = __fmaf_rn(dx, dx, hxx);
      hxy = __fmaf_rn(dx, dy, hxy);
      hyy = __fmaf_rn(dy, dy, hyy);
    }
    if (ty == -a) { sxx = hxx; sxy = hxy; syy = hyy; }
    else { sxx = __fadd_rn(sxx, hxx); sxy = __fadd_rn(sxy, hxy); syy = __fadd_rn(syy, hyy); }
  }
  const float det = __fmaf_rn(sxx, syy, -__fmul_rn(sxy, sxy));
  const float tr = __fadd_rn(sxx, syy);
  const float R = __fmaf_rn(-p.k, __fmul_rn(tr, tr), det);
  reinterpret_cast<float*>(p.dst + (int64_t)b * p.dbstride + (int64_t)(y - p.out_y0) * p.dpitch)[x] = R;
  if (p.mask) p.mask[(int64_t)b * p.mbstride + (int64_t)(y - p.out_y0) * p.mpitch + x] = R > p.threshold ? 1 : 0;
}

// Copy rows of a neighbour's band (peer memory) into this rank's halo rows:
// one thread per 16-byte (or 4-byte) chunk, rows x chunks x images.
struct PullParams {
  const char* src;  // first source row, image 0
  int64_t spitch, sbstride;
  char* dst;        // first destination row, image 0
  int64_t dpitch, dbstride;
  int rows, chunks;  // chunks per row
  int vec16;
  void* win;  // (see EdgeParams): src resolved from the peer's window when wpeer >= 0
  int wpeer;
};

__global__ void __launch_bounds__(256) halo_pull(PullParams p) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y, b = blockIdx.z;
  if (c >= p.chunks || r >= p.rows) return;
  const char* s = win_resolve(p.win, p.wpeer, p.src) + (int64_t)b * p.sbstride + (int64_t)r * p.spitch;
  char* d = p.dst + (int64_t)b * p.dbstride + (int64_t)r * p.dpitch;
  if (p.vec16) reinterpret_cast<float4*>(d)[c] = __ldcv(reinterpret_cast<const float4*>(s) + c);
  else reinterpret_cast<float*>(d)[c] = __ldcv(reinterpret_cast<const float*>(s) + c);
}

// The window entry points run the pointer entry points' validation and launches with the
// neighbour bands described by placeholder images (base kWinFake + window offset); this context
// tells them which window / peers resolve those bases on the device.
struct WinCtx {
  void* win;
  int peer[2];  // up, down
};
thread_local const WinCtx* t_win = nullptr;

}  // namespace
}  // namespace icl

using namespace icl;

extern "C" {

icl_status icl_ipc_get_handle(const void* dev_ptr, void* handle, uint64_t* offset) {
  if (!dev_ptr || !handle || !offset) return report_error(ICL_ERR_INVALID_ARG, "null argument");
  // the handle names the whole allocation; the pointer's offset inside it travels beside it
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
    return report_error(ICL_ERR_CUDA, "cuMemGetAddressRange not available");
  CUdeviceptr base = 0;
  size_t size = 0;
  auto range = reinterpret_cast<CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr)>(fn);
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return report_error(ICL_ERR_INVALID_ARG, "not a device allocation");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return report_error(ICL_ERR_CUDA, cudaGetErrorString(e));
  memcpy(handle, &h, sizeof h);
  *offset = reinterpret_cast<uintptr_t>(dev_ptr) - (uintptr_t)base;
  return ICL_OK;
}

icl_status icl_ipc_open(const void* handle, uint64_t offset, void** dev_ptr) {
  if (!handle || !dev_ptr) return report_error(ICL_ERR_INVALID_ARG, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  void* p = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return report_error(ICL_ERR_CUDA, cudaGetErrorString(e));
  *dev_ptr = static_cast<char*>(p) + offset;
  return ICL_OK;
}

icl_status icl_ipc_close(void* dev_ptr, uint64_t offset) {
  if (!dev_ptr) return ICL_OK;
  cudaError_t e = cudaIpcCloseMemHandle(static_cast<char*>(dev_ptr) - offset);
  return e == cudaSuccess ? ICL_OK : report_error(ICL_ERR_CUDA, cudaGetErrorString(e));
}

// Descriptor checks every peer entry point runs up front (own / dst / neighbour bands), so a
// thin band whose interior call is skipped never launches an edge kernel on unchecked
// descriptors.
static icl_status check_peer_image(const icl_image* im, int64_t elem, const char* name) {
  char m[160];
  if (!im || !im->data) {
    snprintf(m, sizeof m, "%s: null image", name);
    return report_error(ICL_ERR_INVALID_ARG, m);
  }
  if (im->width < 1 || im->height < 1 || im->batch < 1 || im->pitch_bytes < im->width * elem ||
      im->pitch_bytes % elem != 0 ||
      (im->batch > 1 && im->batch_stride_bytes < im->pitch_bytes * im->height)) {
    snprintf(m, sizeof m, "%s: bad width / height / pitch / batch stride", name);
    return report_error(ICL_ERR_INVALID_ARG, m);
  }
  return ICL_OK;
}

icl_status icl_sepconv_peer(const icl_image* own, const icl_image* dst, int64_t global_height, int64_t own_y0,
                            const icl_image* up, const icl_image* down, const float* taps_x, int rx,
                            const float* taps_y, int ry, icl_border border, float border_value, void* stream) {
  if (!own || !dst || !taps_x || !taps_y) return report_error(ICL_ERR_INVALID_ARG, "null argument");
  if (rx < 0 || ry < 0 || rx > kMaxRadius || ry > kMaxRadius)
    return report_error(ICL_ERR_INVALID_ARG, "radius outside [0, 15]");
  if (border != ICL_BORDER_CONSTANT && border != ICL_BORDER_CLAMP)
    return report_error(ICL_ERR_INVALID_ARG, "border must be ICL_BORDER_CONSTANT or ICL_BORDER_CLAMP");
  if (std::isnan(border_value)) return report_error(ICL_ERR_INVALID_ARG, "border_value is NaN");
  {
    icl_status st0;
    if ((st0 = check_peer_image(own, 4, "own")) || (st0 = check_peer_image(dst, 4, "dst"))) return st0;
  }
  const int64_t H = global_height, y0 = own_y0, y1 = own_y0 + own->height;
  if (H < 1 || H >= (1ll << 31) || y0 < 0 || y1 > H || dst->height != own->height || dst->width != own->width ||
      dst->batch != own->batch || own->width < 1 || own->height < 1 || own->batch < 1 || own->batch > 65535)
    return report_error(ICL_ERR_INVALID_ARG, "bad band geometry");
  // the neighbours must provide the rows the edges need (ry rows, or up to the image edge)
  const int64_t need_up = std::min<int64_t>(ry, y0), need_dn = std::min<int64_t>(ry, H - y1);
  auto check_nb = [&](const icl_image* nb, int64_t need, const char* which) -> icl_status {
    if (need == 0) return ICL_OK;
    if (!nb || !nb->data || nb->height < need || nb->width != own->width || nb->batch != own->batch ||
        check_peer_image(nb, 4, which) != ICL_OK)
      return report_error(ICL_ERR_INVALID_ARG, which);
    return ICL_OK;
  };
  icl_status st;
  if ((st = check_nb(up, need_up, "up neighbour band missing or thinner than the halo"))) return st;
  if ((st = check_nb(down, need_dn, "down neighbour band missing or thinner than the halo"))) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // rows needing no halo: the ordinary kernels on the own band
  const int64_t i0 = y0 + (y0 > 0 ? ry : 0), i1 = y1 - (y1 < H ? ry : 0);
  if (i1 > i0) {
    icl_image dv = *dst;
    dv.data = static_cast<char*>(dst->data) + (i0 - y0) * dst->pitch_bytes;
    dv.height = i1 - i0;
    const icl_band bi{H, y0, i0};
    if ((st = icl_sepconv(own, &dv, taps_x, rx, taps_y, ry, border, border_value, &bi, nullptr, 0, s))) return st;
  }
  // edge rows: input rows from the own band and the neighbours' bands (peer loads)
  EdgeParams p;
  memset(&p, 0, sizeof p);
  auto seg = [](const icl_image* im, int64_t gy0) {
    RowSeg g;
    g.base = static_cast<const char*>(im->data);
    g.pitch = im->pitch_bytes;
    g.bstride = im->batch > 1 ? im->batch_stride_bytes : 0;
    g.y0 = (int)gy0;
    g.y1 = (int)(gy0 + im->height);
    return g;
  };
  p.seg[1] = seg(own, y0);
  if (need_up) {  // the up neighbour's LAST rows end at y0
    p.seg[0] = seg(up, y0 - up->height);
  }
  if (need_dn) p.seg[2] = seg(down, y1);
  p.wpeer[0] = p.wpeer[1] = p.wpeer[2] = -1;
  if (t_win) {
    p.win = t_win->win;
    p.wpeer[0] = need_up ? t_win->peer[0] : -1;
    p.wpeer[2] = need_dn ? t_win->peer[1] : -1;
  }
  p.W = (int)own->width;
  p.Hg = (int)H;
  p.border = border == ICL_BORDER_CLAMP ? kBorderClamp : kBorderConstant;
  p.cval = border_value;
  p.rx = rx;
  p.ry = ry;
  for (int i = 0; i <= 2 * rx; ++i) p.fx[i] = taps_x[i];
  for (int j = 0; j <= 2 * ry; ++j) p.gy[j] = taps_y[j];
  p.dpitch = dst->pitch_bytes;
  p.dbstride = dst->batch > 1 ? dst->batch_stride_bytes : 0;
  const size_t smem = (size_t)(kEdgeTW + 4 * kMaxRadius + (kEdgeCH + 2 * ry) * kEdgeTW) * sizeof(float);
  auto edge = [&](int64_t a0, int64_t a1) -> icl_status {
    if (a1 <= a0) return ICL_OK;
    p.dst = static_cast<char*>(dst->data) + (a0 - y0) * dst->pitch_bytes;
    p.out_y0 = (int)a0;
    p.out_y1 = (int)a1;
    dim3 grd((unsigned)((own->width + kEdgeTW - 1) / kEdgeTW), (unsigned)((a1 - a0 + kEdgeCH - 1) / kEdgeCH),
             (unsigned)own->batch);
    cudaError_t e0 = cudaFuncSetAttribute(sep_edge_peer, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e0 != cudaSuccess) return report_error(ICL_ERR_CUDA, cudaGetErrorString(e0));
    sep_edge_peer<<<grd, kEdgeTW, smem, s>>>(p);
    count_launch();
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? ICL_OK : report_error(ICL_ERR_CUDA, cudaGetErrorString(e));
  };
  if (i1 <= i0) return edge(y0, y1);  // thin band: every row is an edge row
  if ((st = edge(y0, i0))) return st;
  return edge(i1, y1);
}

icl_status icl_harris_peer(const icl_image* own, const icl_image* response, int64_t global_height, int64_t own_y0,
                          const icl_image* up, const icl_image* down, int block, float k, icl_border border,
                          float border_value, const icl_image* mask, float threshold, void* stream) {
  if (!own || !response) return report_error(ICL_ERR_INVALID_ARG, "null argument");
  if (block < 1 || block > 7) return report_error(ICL_ERR_INVALID_ARG, "block must be in [1, 7]");
  if (border != ICL_BORDER_CONSTANT && border != ICL_BORDER_CLAMP)
    return report_error(ICL_ERR_INVALID_ARG, "border must be ICL_BORDER_CONSTANT or ICL_BORDER_CLAMP");
  if (std::isnan(border_value) || std::isnan(k)) return report_error(ICL_ERR_INVALID_ARG, "border_value or k is NaN");
  {
    icl_status st0;
    if ((st0 = check_peer_image(own, 4, "own")) || (st0 = check_peer_image(response, 4, "response"))) return st0;
  }
  const int64_t H = global_height, y0 = own_y0, y1 = own_y0 + own->height;
  if (H < 1 || H >= (1ll << 31) || y0 < 0 || y1 > H || response->height != own->height ||
      response->width != own->width || response->batch != own->batch || own->width < 1 || own->height < 1 ||
      own->batch < 1 || own->batch > 65535 || !own->data || !response->data)
    return report_error(ICL_ERR_INVALID_ARG, "bad band geometry");
  if (mask && mask->data && (mask->width != own->width || mask->height != own->height || mask->batch != own->batch))
    return report_error(ICL_ERR_INVALID_ARG, "mask shape differs from the response");
  const int a = block / 2, bb = block - 1 - a;
  const int64_t hu = a + 1, hdn = bb + 1;  // input rows a response row needs above / below
  const int64_t need_up = std::min<int64_t>(hu, y0), need_dn = std::min<int64_t>(hdn, H - y1);
  auto check_nb = [&](const icl_image* nb, int64_t need, const char* which) -> icl_status {
    if (need == 0) return ICL_OK;
    if (!nb || !nb->data || nb->height < need || nb->width != own->width || nb->batch != own->batch ||
        check_peer_image(nb, 4, which) != ICL_OK)
      return report_error(ICL_ERR_INVALID_ARG, which);
    return ICL_OK;
  };
  icl_status st;
  if ((st = check_nb(up, need_up, "up neighbour band missing or thinner than the halo"))) return st;
  if ((st = check_nb(down, need_dn, "down neighbour band missing or thinner than the halo"))) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // rows needing no halo: the ordinary Harris kernels on the own band
  const int64_t i0 = y0 + (y0 > 0 ? hu : 0), i1 = y1 - (y1 < H ? hdn : 0);
  if (i1 > i0) {
    icl_image dv = *response;
    dv.data = static_cast<char*>(response->data) + (i0 - y0) * response->pitch_bytes;
    dv.height = i1 - i0;
    icl_image mv;
    if (mask && mask->data) {
      mv = *mask;
      mv.data = static_cast<char*>(mask->data) + (i0 - y0) * mask->pitch_bytes;
      mv.height = i1 - i0;
    }
    const icl_band bi{H, y0, i0};
    if ((st = harris_naive_order(own, &dv, block, k, border, border_value, mask && mask->data ? &mv : nullptr, threshold, &bi,
                         s)))
      return st;
  }
  // edge rows: input rows from the own band or straight from the neighbours' bands
  HarrisEdgeParams p;
  memset(&p, 0, sizeof p);
  auto seg = [](const icl_image* im, int64_t gy0) {
    RowSeg g;
    g.base = static_cast<const char*>(im->data);
    g.pitch = im->pitch_bytes;
    g.bstride = im->batch > 1 ? im->batch_stride_bytes : 0;
    g.y0 = (int)gy0;
    g.y1 = (int)(gy0 + im->height);
    return g;
  };
  p.seg[1] = seg(own, y0);
  if (need_up) p.seg[0] = seg(up, y0 - up->height);
  if (need_dn) p.seg[2] = seg(down, y1);
  p.wpeer[0] = p.wpeer[1] = p.wpeer[2] = -1;
  if (t_win) {
    p.win = t_win->win;
    p.wpeer[0] = need_up ? t_win->peer[0] : -1;
    p.wpeer[2] = need_dn ? t_win->peer[1] : -1;
  }
  p.W = (int)own->width;
  p.Hg = (int)H;
  p.border = border == ICL_BORDER_CLAMP ? kBorderClamp : kBorderConstant;
  p.cval = border_value;
  p.block = block;
  p.k = k;
  p.threshold = threshold;
  p.dpitch = response->pitch_bytes;
  p.dbstride = response->batch > 1 ? response->batch_stride_bytes : 0;
  auto edge = [&](int64_t a0, int64_t a1) -> icl_status {
    if (a1 <= a0) return ICL_OK;
    p.dst = static_cast<char*>(response->data) + (a0 - y0) * response->pitch_bytes;
    p.mask = nullptr;
    if (mask && mask->data) {
      p.mask = static_cast<char*>(mask->data) + (a0 - y0) * mask->pitch_bytes;
      p.mpitch = mask->pitch_bytes;
      p.mbstride = mask->batch > 1 ? mask->batch_stride_bytes : 0;
    }
    p.out_y0 = (int)a0;
    p.out_y1 = (int)a1;
    dim3 grd((unsigned)((own->width + 31) / 32), (unsigned)((a1 - a0 + 7) / 8), (unsigned)own->batch);
    harris_edge_peer<<<grd, 256, 0, s>>>(p);
    count_launch();
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? ICL_OK : report_error(ICL_ERR_CUDA, cudaGetErrorString(e));
  };
  if (i1 <= i0) return edge(y0, y1);
  if ((st = edge(y0, i0))) return st;
  return edge(i1, y1);
}

icl_status icl_halo_pull(const icl_image* buf, int64_t global_height, int64_t buf_y0, int64_t own_y0,
                         int64_t own_y1, const icl_image* up, const icl_image* down, int elem_bytes, void* stream) {
  if (!buf || !buf->data || (elem_bytes != 1 && elem_bytes != 4) || check_peer_image(buf, elem_bytes, "buf") != ICL_OK)
    return report_error(ICL_ERR_INVALID_ARG, "bad buffer");
  const int64_t H = global_height, s0 = buf_y0, s1 = buf_y0 + buf->height;
  if (H < 1 || s0 < 0 || s1 > H || own_y0 < s0 || own_y1 > s1 || own_y0 > own_y1 || buf->batch < 1 ||
      buf->batch > 65535)
    return report_error(ICL_ERR_INVALID_ARG, "bad band geometry");
  const int64_t rowb = buf->width * elem_bytes;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto pull = [&](const icl_image* nb, int64_t nb_y0, int64_t g0, int64_t g1, int side) -> icl_status {
    if (g1 <= g0) return ICL_OK;
    if (!nb || !nb->data || nb->width != buf->width || nb->batch != buf->batch || g0 < nb_y0 ||
        g1 > nb_y0 + nb->height || check_peer_image(nb, elem_bytes, "neighbour") != ICL_OK)
      return report_error(ICL_ERR_INVALID_ARG, "neighbour band does not hold the halo rows (rows, pitch or stride)");
    PullParams p;
    p.win = t_win ? t_win->win : nullptr;
    p.wpeer = t_win ? t_win->peer[side] : -1;
    p.src = static_cast<const char*>(nb->data) + (g0 - nb_y0) * nb->pitch_bytes;
    p.spitch = nb->pitch_bytes;
    p.sbstride = nb->batch > 1 ? nb->batch_stride_bytes : 0;
    p.dst = static_cast<char*>(buf->data) + (g0 - s0) * buf->pitch_bytes;
    p.dpitch = buf->pitch_bytes;
    p.dbstride = buf->batch > 1 ? buf->batch_stride_bytes : 0;
    p.rows = (int)(g1 - g0);
    const uintptr_t al = reinterpret_cast<uintptr_t>(p.src) | reinterpret_cast<uintptr_t>(p.dst) |
                         (uintptr_t)p.spitch | (uintptr_t)p.dpitch | (uintptr_t)p.sbstride | (uintptr_t)p.dbstride;
    p.vec16 = (al % 16 == 0) && rowb % 16 == 0;
    if (!p.vec16 && (al % 4 != 0 || rowb % 4 != 0)) return report_error(ICL_ERR_UNSUPPORTED, "rows not 4-byte aligned");
    p.chunks = (int)(rowb / (p.vec16 ? 16 : 4));
    dim3 grd((unsigned)((p.chunks + 255) / 256), (unsigned)p.rows, (unsigned)buf->batch);
    halo_pull<<<grd, 256, 0, s>>>(p);
    count_launch();
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? ICL_OK : report_error(ICL_ERR_CUDA, cudaGetErrorString(e));
  };
  icl_status st = pull(up, own_y0 - (up ? up->height : 0), s0, own_y0, 0);
  if (st != ICL_OK) return st;
  return pull(down, own_y1, own_y1, s1, 1);
}

// ---------------------------------------------------------------- NCCL symmetric windows
static icl_status window_call(const icl_window* win, const icl_image* like, const icl_window_band* up,
                              const icl_window_band* down, int elem_bytes, icl_image* ui, icl_image* di,
                              WinCtx* ctx, const icl_image** upp, const icl_image** dnp) {
#ifndef ICL_HAVE_NCCL_DEVICE
  (void)win; (void)like; (void)up; (void)down; (void)elem_bytes; (void)ui; (void)di; (void)ctx; (void)upp; (void)dnp;
  return report_error(ICL_ERR_UNSUPPORTED, "built without the NCCL >= 2.28 device headers");
#else
  if (!win || !win->win || !like) return report_error(ICL_ERR_INVALID_ARG, "null window or image");
  ctx->win = win->win;
  ctx->peer[0] = ctx->peer[1] = -1;
  *upp = *dnp = nullptr;
  auto mk = [&](const icl_window_band* wb, icl_image* im) -> const icl_image* {
    if (!wb || wb->peer < 0) return nullptr;
    *im = *like;
    im->data = reinterpret_cast<void*>(kWinFake + (uintptr_t)wb->offset);
    im->height = wb->height;
    im->pitch_bytes = wb->pitch_bytes;
    im->batch_stride_bytes = wb->batch_stride_bytes;
    return im;
  };
  for (const icl_window_band* wb : {up, down})
    if (wb && wb->peer >= 0 && (wb->peer >= win->nranks || wb->offset >= win->bytes || wb->height < 1 ||
                                wb->pitch_bytes < like->width * elem_bytes))
      return report_error(ICL_ERR_INVALID_ARG, "neighbour window band outside the window / communicator");
  *upp = mk(up, ui);
  *dnp = mk(down, di);
  ctx->peer[0] = up ? up->peer : -1;
  ctx->peer[1] = down ? down->peer : -1;
  return ICL_OK;
#endif
}

icl_status icl_sepconv_window(const icl_window* win, const icl_image* own, const icl_image* dst,
                              int64_t global_height, int64_t own_y0, const icl_window_band* up,
                              const icl_window_band* down, const float* taps_x, int rx, const float* taps_y, int ry,
                              icl_border border, float border_value, void* stream) {
  icl_image ui, di;
  WinCtx ctx;
  const icl_image *upp, *dnp;
  icl_status st = window_call(win, own, up, down, 4, &ui, &di, &ctx, &upp, &dnp);
  if (st != ICL_OK) return st;
  t_win = &ctx;
  st = icl_sepconv_peer(own, dst, global_height, own_y0, upp, dnp, taps_x, rx, taps_y, ry, border, border_value,
                        stream);
  t_win = nullptr;
  return st;
}

icl_status icl_harris_window(const icl_window* win, const icl_image* own, const icl_image* response,
                             int64_t global_height, int64_t own_y0, const icl_window_band* up,
                             const icl_window_band* down, int block, float k, icl_border border, float border_value,
                             const icl_image* mask, float threshold, void* stream) {
  icl_image ui, di;
  WinCtx ctx;
  const icl_image *upp, *dnp;
  icl_status st = window_call(win, own, up, down, 4, &ui, &di, &ctx, &upp, &dnp);
  if (st != ICL_OK) return st;
  t_win = &ctx;
  st = icl_harris_peer(own, response, global_height, own_y0, upp, dnp, block, k, border, border_value, mask, threshold,
                       stream);
  t_win = nullptr;
  return st;
}

icl_status icl_halo_pull_window(const icl_window* win, const icl_image* buf, int64_t global_height, int64_t buf_y0,
                                int64_t own_y0, int64_t own_y1, const icl_window_band* up,
                                const icl_window_band* down, int elem_bytes, void* stream) {
  icl_image ui, di;
  WinCtx ctx;
  const icl_image *upp, *dnp;
  icl_status st = window_call(win, buf, up, down, elem_bytes, &ui, &di, &ctx, &upp, &dnp);
  if (st != ICL_OK) return st;
  t_win = &ctx;
  st = icl_halo_pull(buf, global_height, buf_y0, own_y0, own_y1, upp, dnp, elem_bytes, stream);
  t_win = nullptr;
  return st;
}

}  // extern "C"
