// api.cu -- the C ABI of include/icl.h: argument validation, row-band views,
// the variant registry (Table 1 -> B200 axes),
// dispatch, the auto-tuner and its winner cache (§4;
// SURVEY.md §8(a) a11).  No compute happens here: every step of the filters
// runs in the kernels of sepconv.cu / harris.cu / nlm.cu.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <deque>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/icl.h"
#include "internal.h"

#define ICL_VERSION_STRING "icl-b200 0.1 (sm_100a)"

namespace icl {

bool nlm_tiled_supported(int P, int S);
bool nlm_boxsum_supported(int P, int S);
bool nlm_r8_supported(int P, int S);
bool nlm_r16_supported(int P, int S);
bool nlm_x2_supported(int P, int S);
bool nlm_w_supported(int P, int S);
bool nlm_sym_supported(int P, int S);
bool nlm_sym_ring_supported(int P, int S);
bool nlm_sym8_supported(int P, int S);

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// ------------------------------------------------------------------ errors
static thread_local std::string t_err;
static icl_status fail(icl_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
  return st;
}
// for the other translation units of the library (comm.cu): report an error status + message
icl_status report_error(icl_status st, const char* msg) { return fail(st, "%s", msg); }

static icl_status cuda_fail(cudaError_t e, const char* what) {
  return fail(ICL_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// ------------------------------------------------------------------ images
static icl_status check_image(const icl_image* im, int64_t elem, const char* name) {
  if (!im) return fail(ICL_ERR_INVALID_ARG, "%s: null image descriptor", name);
  if (!im->data) return fail(ICL_ERR_INVALID_ARG, "%s: null data pointer", name);
  if (im->width < 1 || im->height < 1 || im->batch < 1)
    return fail(ICL_ERR_INVALID_ARG, "%s: width/height/batch must be >= 1", name);
  if (im->width >= (1ll << 31) || im->height >= (1ll << 31) || im->batch >= (1ll << 31))
    return fail(ICL_ERR_INVALID_ARG, "%s: size out of range", name);
  if (im->pitch_bytes < im->width * elem || im->pitch_bytes % elem)
    return fail(ICL_ERR_INVALID_ARG, "%s: pitch_bytes must be >= width*%lld and a multiple of %lld", name,
                (long long)elem, (long long)elem);
  if (im->batch > 1 && (im->batch_stride_bytes < im->height * im->pitch_bytes || im->batch_stride_bytes % elem))
    return fail(ICL_ERR_INVALID_ARG, "%s: batch_stride_bytes must be >= height*pitch_bytes", name);
  if (reinterpret_cast<uintptr_t>(im->data) % elem)
    return fail(ICL_ERR_INVALID_ARG, "%s: data pointer not aligned to the element size", name);
  return ICL_OK;
}

struct Range {
  uintptr_t lo, hi;
};
static Range byte_range(const icl_image* im, int64_t elem) {
  const uintptr_t lo = reinterpret_cast<uintptr_t>(im->data);
  const int64_t last = (im->batch - 1) * (im->batch > 1 ? im->batch_stride_bytes : 0) +
                       (im->height - 1) * im->pitch_bytes + im->width * elem;
  return {lo, lo + (uintptr_t)last};
}
static bool overlap(Range a, Range b) { return a.lo < b.hi && b.lo < a.hi; }

static bool aligned16(const icl_image* im) {
  const uint64_t bits = reinterpret_cast<uintptr_t>(im->data) | (uint64_t)im->pitch_bytes |
                        (im->batch > 1 ? (uint64_t)im->batch_stride_bytes : 0);
  return bits % 16 == 0;
}
static bool aligned4(const icl_image* im) {
  const uint64_t bits = reinterpret_cast<uintptr_t>(im->data) | (uint64_t)im->pitch_bytes |
                        (im->batch > 1 ? (uint64_t)im->batch_stride_bytes : 0);
  return bits % 4 == 0;
}

// Resolve band + views; `up`/`down` = rows of stencil above/below an output.
static icl_status make_views(const icl_image* src, const icl_image* dst, const icl_band* band, icl_border border,
                             float cval, int up, int down, SrcView* sv, DstView* dv) {
  if (border != ICL_BORDER_CONSTANT && border != ICL_BORDER_CLAMP)
    return fail(ICL_ERR_INVALID_ARG, "border must be ICL_BORDER_CONSTANT or ICL_BORDER_CLAMP");
  if (std::isnan(cval)) return fail(ICL_ERR_INVALID_ARG, "border_value is NaN");
  if (src->width != dst->width) return fail(ICL_ERR_INVALID_ARG, "src and dst widths differ");
  if (src->batch != dst->batch) return fail(ICL_ERR_INVALID_ARG, "src and dst batch differ");
  int64_t Hg, sy0, dy0;
  if (band) {
    Hg = band->global_height;
    sy0 = band->src_y0;
    dy0 = band->dst_y0;
    if (Hg < 1 || Hg >= (1ll << 31)) return fail(ICL_ERR_INVALID_ARG, "band: bad global_height");
    if (sy0 < 0 || sy0 + src->height > Hg) return fail(ICL_ERR_INVALID_ARG, "band: src rows outside the image");
    if (dy0 < 0 || dy0 + dst->height > Hg) return fail(ICL_ERR_INVALID_ARG, "band: dst rows outside the image");
    const int64_t need_lo = std::max<int64_t>(0, dy0 - up);
    const int64_t need_hi = std::min<int64_t>(Hg - 1, dy0 + dst->height - 1 + down);
    if (need_lo < sy0 || need_hi > sy0 + src->height - 1)
      return fail(ICL_ERR_INVALID_ARG, "band: src rows [%lld,%lld) do not cover the stencil rows [%lld,%lld]",
                  (long long)sy0, (long long)(sy0 + src->height), (long long)need_lo, (long long)need_hi);
  } else {
    Hg = src->height;
    sy0 = dy0 = 0;
    if (dst->height != src->height) return fail(ICL_ERR_INVALID_ARG, "src and dst heights differ");
  }
  sv->base = static_cast<const char*>(src->data);
  sv->pitch = src->pitch_bytes;
  sv->bstride = src->batch > 1 ? src->batch_stride_bytes : 0;
  sv->W = (int)src->width;
  sv->Hg = (int)Hg;
  sv->y0 = (int)sy0;
  sv->Hl = (int)std::min<int64_t>(src->height, Hg - sy0);
  sv->border = border == ICL_BORDER_CLAMP ? kBorderClamp : kBorderConstant;
  sv->cval = cval;
  dv->base = static_cast<char*>(dst->data);
  dv->pitch = dst->pitch_bytes;
  dv->bstride = dst->batch > 1 ? dst->batch_stride_bytes : 0;
  dv->H = (int)dst->height;
  dv->y0 = (int)dy0;
  return ICL_OK;
}

// ------------------------------------------------------------------ variants
enum Kind { K_NAIVE, K_TWOPASS, K_STREAM, K_TILED, K_BOXSUM, K_BOXR8, K_BULK, K_BOXR16, K_SHFL, K_TILE2, K_BOXX2, K_C2TILE, K_TEX, K_SLIDE, K_BOXW, K_PMAP, K_BOXSYM, K_BOXRING, K_BOXSYM8, K_COUNT };
struct Variant {
  const char* name;
  Kind kind;
  int nt, vec, S;
  PmapCfg pm;  // K_PMAP: the paper's Table-1 configuration (pmap.cu)
};

static const Variant kSepVariants[] = {
    {"naive_direct", K_NAIVE, 0, 0, 0},
    {"naive_2pass", K_TWOPASS, 0, 0, 0},
    {"stream_nt64_s16_v4", K_STREAM, 64, 4, 16},
    {"stream_nt32_s16_v4", K_STREAM, 32, 4, 16},
    {"stream_nt128_s16_v4", K_STREAM, 128, 4, 16},
    {"stream_nt32_s8_v4", K_STREAM, 32, 4, 8},
    {"stream_nt32_s32_v4", K_STREAM, 32, 4, 32},
    {"stream_nt64_s32_v4", K_STREAM, 64, 4, 32},
    {"stream_nt64_s64_v4", K_STREAM, 64, 4, 64},
    {"stream_nt128_s64_v4", K_STREAM, 128, 4, 64},
    {"stream_nt64_s128_v4", K_STREAM, 64, 4, 128},
    {"stream_nt32_s128_v4", K_STREAM, 32, 4, 128},
    {"stream_nt128_s128_v4", K_STREAM, 128, 4, 128},
    {"stream_nt256_s16_v4", K_STREAM, 256, 4, 16},
    {"stream_nt64_s64_v1", K_STREAM, 64, 1, 64},
    {"stream_nt64_s16_v1", K_STREAM, 64, 1, 16},
    // interior row blocks staged by one cp.async.bulk.tensor (TMA) each (vec 7)
    {"tma_nt32_s16_v4", K_STREAM, 32, 7, 16},
    {"tma_nt32_s32_v4", K_STREAM, 32, 7, 32},
    {"tma_nt32_s64_v4", K_STREAM, 32, 7, 64},
    {"tma_nt32_s128_v4", K_STREAM, 32, 7, 128},
    {"bulk_nt128_s64", K_BULK, 128, 4, 64},
    {"bulk_nt64_s64", K_BULK, 64, 4, 64},
    {"tile64_v4", K_TILE2, 256, 4, 64},
    {"tile64p_v4", K_TILE2, 256, 4, 1},
    {"tile128p_v4", K_TILE2, 512, 4, 2},
    {"tex_c4s16", K_TEX, 128, 4, 16},
};
static const Variant kHarVariants[] = {
    {"naive_direct", K_NAIVE, 0, 0, 0},           {"stream_nt64_s64_v4", K_STREAM, 64, 4, 64},
    {"stream_nt32_s32_v4", K_STREAM, 32, 4, 32},  {"stream_nt128_s64_v4", K_STREAM, 128, 4, 64},
    {"stream_nt64_s128_v4", K_STREAM, 64, 4, 128}, {"stream_nt32_s16_v4", K_STREAM, 32, 4, 16},
    {"stream_nt64_s64_v1", K_STREAM, 64, 1, 64},
    {"shfl_nw2_s64", K_SHFL, 2, 4, 64},           {"shfl_nw4_s64", K_SHFL, 4, 4, 64},
    {"shfl_nw2_s32", K_SHFL, 2, 4, 32},           {"shfl_nw4_s32", K_SHFL, 4, 4, 32},
    {"shfl_nw2_s128", K_SHFL, 2, 4, 128},         {"shfl_nw2_s16", K_SHFL, 2, 4, 16},
    {"shfl_nw2_s8", K_SHFL, 2, 4, 8},             {"shfl_nw4_s16", K_SHFL, 4, 4, 16},
    {"shfl_nw4_s8", K_SHFL, 4, 4, 8},
    // one-warp CTAs (120-column strips): more CTAs for images that do not fill the GPU
    {"shfl_nw1_s16", K_SHFL, 1, 4, 16},           {"shfl_nw1_s32", K_SHFL, 1, 4, 32},
    {"shfl_nw1_s8", K_SHFL, 1, 4, 8},
    // interior ring blocks staged by one TMA box each (vec 7; 16-byte aligned images)
    {"shfl_tma_nw2_s32", K_SHFL, 2, 7, 32},       {"shfl_tma_nw2_s16", K_SHFL, 2, 7, 16},
    {"shfl_tma_nw2_s8", K_SHFL, 2, 7, 8},
    // separable window sums on the products (re-associated: tolerance vs naive, R16)
    {"slide_nw2_s32", K_SLIDE, 2, 4, 32},         {"slide_nw2_s16", K_SLIDE, 2, 4, 16},
    {"slide_nw2_s64", K_SLIDE, 2, 4, 64},         {"slide_nw2_s8", K_SLIDE, 2, 4, 8},
    {"slide_nw4_s32", K_SLIDE, 4, 4, 32},         {"slide_nw4_s16", K_SLIDE, 4, 4, 16},
    {"slide_nw2_s32_u2", K_SLIDE, 2, 8, 32},      {"slide_nw2_s16_u2", K_SLIDE, 2, 8, 16},
    // products' horizontal pair sums first, then vertical chains (vec 6 selects HFIRST)
    {"slide2_nw2_s32", K_SLIDE, 2, 6, 32},        {"slide2_nw2_s16", K_SLIDE, 2, 6, 16},
    {"slide2_nw2_s64", K_SLIDE, 2, 6, 64},        {"slide2_nw4_s32", K_SLIDE, 4, 6, 32},
};
static const Variant kNlmVariants[] = {
    {"naive_direct", K_NAIVE, 0, 0, 0},
    {"tiled_direct_32x8", K_TILED, 32, 0, 8},
    {"boxsum_32x32", K_BOXSUM, 32, 0, 32},
    {"boxsum_r8", K_BOXR8, 0, 0, 0},
    {"boxsum_r16", K_BOXR16, 0, 0, 0},
    {"boxsum_x2", K_BOXX2, 0, 0, 0},
    {"boxsum_w", K_BOXW, 0, 0, 1},
    {"sym_tmem", K_BOXSYM, 0, 0, 0},
    {"sym_ring", K_BOXRING, 0, 0, 0},
    {"sym_tmem8", K_BOXSYM8, 0, 0, 0},
};

static const Variant kConvVariants[] = {
    {"naive_direct", K_NAIVE, 0, 0, 0},
    {"tile_c4r4", K_C2TILE, 256, 4, 4},
    {"tile_c4r8", K_C2TILE, 256, 4, 8},
    {"tile_c4r4p", K_C2TILE, 1, 4, 4},
    {"tile_c4r8p", K_C2TILE, 1, 4, 8},
    {"tex_c4r4", K_TEX, 128, 4, 4},
};

// 3-D volumes (icl_sepconv3d; sep3d.cu): dispatched by icl_sepconv3d itself
static const Variant kSep3Variants[] = {
    {"naive_direct", K_NAIVE, 0, 0, 0},
    {"tile64x16", K_TILE2, 256, 1, 64},
};

// The paper's Table-1 space for the one-pixel-per-logical-thread kernels (pmap.cu), appended to
// the sepconv and Harris tables: CTA shape x coarsening x (mapping, local memory) x unroll =
// 6 x 6 x 4 x 2 = 288 configurations per filter.  Name: pm_w<wx>x<wy>_c<cx>x<cy>_<map>_l<0|1>_u<1|4>
// with map = blk (blocked) / int (interleaved) / iwg (interleaved in the work-group; with local
// memory the interleaving is within the work-group).
static void append_pmap(std::vector<Variant>* out) {
  static std::deque<std::string> names;  // storage for the generated names (built once)
  const int wg[][2] = {{32, 4}, {64, 2}, {128, 1}, {16, 8}, {32, 8}, {64, 4}};
  const int co[][2] = {{1, 1}, {2, 1}, {4, 1}, {1, 2}, {2, 2}, {1, 4}};
  const int ml[][2] = {{kMapBlocked, 0}, {kMapInterleaved, 0}, {kMapBlocked, 1}, {kMapInWG, 1}};
  const char* mname[] = {"blk", "int", "iwg"};
  for (auto& w : wg)
    for (auto& c : co)
      for (auto& m : ml)
        for (int u : {1, 4}) {
          char buf[64];
          snprintf(buf, sizeof buf, "pm_w%dx%d_c%dx%d_%s_l%d_u%d", w[0], w[1], c[0], c[1], mname[m[0]], m[1], u);
          names.emplace_back(buf);
          Variant v{};
          v.name = names.back().c_str();
          v.kind = K_PMAP;
          v.nt = w[0] * w[1];
          v.vec = c[0];
          v.S = c[1];
          v.pm = PmapCfg{w[0], w[1], c[0], c[1], m[0], m[1], u};
          out->push_back(v);
        }
}

template <size_t N>
static std::vector<Variant> with_pmap(const Variant (&base)[N]) {
  std::vector<Variant> t(base, base + N);
  append_pmap(&t);
  return t;
}

static const Variant* table(icl_filter f, int* n) {
  switch (f) {
    case ICL_FILTER_SEPCONV: {
      static const std::vector<Variant> v = with_pmap(kSepVariants);
      *n = (int)v.size();
      return v.data();
    }
    case ICL_FILTER_HARRIS: {
      static const std::vector<Variant> v = with_pmap(kHarVariants);
      *n = (int)v.size();
      return v.data();
    }
    case ICL_FILTER_NLM: *n = (int)(sizeof kNlmVariants / sizeof *kNlmVariants); return kNlmVariants;
    case ICL_FILTER_CONV2D: *n = (int)(sizeof kConvVariants / sizeof *kConvVariants); return kConvVariants;
    case ICL_FILTER_SEPCONV3D: *n = (int)(sizeof kSep3Variants / sizeof *kSep3Variants); return kSep3Variants;
  }
  *n = 0;
  return nullptr;
}

constexpr int kNFilters = 5;
static thread_local int t_force[kNFilters] = {-1, -1, -1, -1, -1};
static thread_local int t_last[kNFilters] = {-1, -1, -1, -1, -1};

// Prepared call of any filter (what a variant launcher needs).
struct Prepared {
  icl_filter f;
  SepCall sep;
  HarrisCall har;
  NlmCall nlm;
  Conv2dCall c2d;
  bool a16;       // src/dst (and mask) 16B-aligned
  int64_t pixels; // W * H * batch
  size_t dst_bytes_compact;
  std::string key;
};

static bool eligible(const Prepared& pc, const Variant& v, icl_status* why) {
  *why = ICL_ERR_UNSUPPORTED;
  if ((v.kind == K_STREAM || v.kind == K_BULK || v.kind == K_SHFL || v.kind == K_TILE2 || v.kind == K_C2TILE ||
       v.kind == K_SLIDE) &&
      v.vec >= 4 && !pc.a16)
    return false;
  if ((v.kind == K_SHFL || v.kind == K_SLIDE) && pc.har.block > 5) return false;
  if (v.kind == K_SLIDE && pc.har.naive_order) return false;
  if (v.kind == K_TEX) {  // hardware boundary: clamp, or constant 0 (border addressing)
    const SrcView& sv = pc.f == ICL_FILTER_SEPCONV ? pc.sep.src : pc.c2d.src;
    const int bt = pc.f == ICL_FILTER_SEPCONV ? pc.sep.batch : pc.c2d.batch;
    if (pc.f == ICL_FILTER_SEPCONV && (pc.sep.rx > 8 || pc.sep.ry > 8)) return false;
    const bool ok_border = sv.border == kBorderClamp || sv.cval == 0.0f;
    if (!tex_eligible(sv, sv.Hg - sv.y0, bt, pc.f == ICL_FILTER_CONV2D ? 1 : 4, ok_border)) return false;
  }
  if (v.kind == K_PMAP && v.pm.local) {  // the staged block + halo must fit in shared memory
    const size_t t = pc.f == ICL_FILTER_SEPCONV
                         ? (size_t)(v.pm.wx * v.pm.cx + 2 * pc.sep.rx) * (v.pm.wy * v.pm.cy + 2 * pc.sep.ry)
                         : (size_t)(v.pm.wx * v.pm.cx + pc.har.block + 1) * (v.pm.wy * v.pm.cy + pc.har.block + 1);
    if (t * sizeof(float) > 227 * 1024) return false;
  }
  if (pc.f == ICL_FILTER_SEPCONV && v.kind == K_TILE2 && v.S == 2 &&
      std::max(pc.sep.rx, pc.sep.ry) < 7)
    return false;  // tile128p: instantiated for R = 7..15
  if (pc.f == ICL_FILTER_SEPCONV && !pc.sep.pad_rows_ok &&
      (v.kind == K_STREAM || v.kind == K_BULK || v.kind == K_TILE2 || v.kind == K_TEX))
    return false;  // padded-radius variant in a band without max(rx, ry) halo rows
  if (pc.f == ICL_FILTER_SEPCONV && v.kind == K_STREAM &&
      sep_stream_smem_bytes(v.nt, pc.sep.rx > pc.sep.ry ? pc.sep.rx : pc.sep.ry) > 227 * 1024)
    return false;
  if (pc.f == ICL_FILTER_SEPCONV && v.kind == K_TWOPASS) {
    const size_t need = sep_2pass_workspace(pc.sep.src.W, pc.sep.dst.H, pc.sep.batch, pc.sep.ry);
    if (!pc.sep.workspace || pc.sep.workspace_bytes < need) {
      *why = ICL_ERR_WORKSPACE;
      return false;
    }
  }
  if (pc.f == ICL_FILTER_NLM && v.kind == K_TILED && !nlm_tiled_supported(pc.nlm.P, pc.nlm.S)) return false;
  if (pc.f == ICL_FILTER_NLM && v.kind == K_BOXSUM && !nlm_boxsum_supported(pc.nlm.P, pc.nlm.S)) return false;
  if (pc.f == ICL_FILTER_NLM && v.kind == K_BOXR8 && !nlm_r8_supported(pc.nlm.P, pc.nlm.S)) return false;
  if (pc.f == ICL_FILTER_NLM && v.kind == K_BOXR16 && !nlm_r16_supported(pc.nlm.P, pc.nlm.S)) return false;
  if (pc.f == ICL_FILTER_NLM && v.kind == K_BOXX2 && !nlm_x2_supported(pc.nlm.P, pc.nlm.S)) return false;
  if (pc.f == ICL_FILTER_NLM && v.kind == K_BOXW && !nlm_w_supported(pc.nlm.P, pc.nlm.S)) return false;
  if (pc.f == ICL_FILTER_NLM && v.kind == K_BOXSYM && !nlm_sym_supported(pc.nlm.P, pc.nlm.S)) return false;
  if (pc.f == ICL_FILTER_NLM && v.kind == K_BOXRING && !nlm_sym_ring_supported(pc.nlm.P, pc.nlm.S)) return false;
  if (pc.f == ICL_FILTER_NLM && v.kind == K_BOXSYM8 && !nlm_sym8_supported(pc.nlm.P, pc.nlm.S)) return false;
  return true;
}

static cudaError_t run_variant_1(const Prepared& pc, const Variant& v, cudaStream_t s);

// gridDim.z (the batch axis of most launchers) is capped at 65535: larger batches run as chunks
// of images, each a view offset by whole images (per-pixel results do not depend on the split).
static cudaError_t run_variant_rows(const Prepared& pc, const Variant& v, cudaStream_t s);

// Row-segment launchers put H / S (S >= 8) on gridDim.y (<= 65535): images taller than 2^19
// rows run as row chunks -- the destination view starts at a later global row (dst.y0), exactly
// an icl_band split, so results equal the one-piece call (bit for bit where the per-output
// order is shared).
static cudaError_t run_variant(const Prepared& pc, const Variant& v, cudaStream_t s) {
  constexpr int kMaxRows = 1 << 19;
  DstView d = pc.f == ICL_FILTER_SEPCONV ? pc.sep.dst
              : pc.f == ICL_FILTER_HARRIS ? pc.har.dst
              : pc.f == ICL_FILTER_NLM    ? pc.nlm.dst
                                          : pc.c2d.dst;
  if (d.H <= kMaxRows) return run_variant_rows(pc, v, s);
  for (int r0 = 0; r0 < d.H; r0 += kMaxRows) {
    Prepared c = pc;
    DstView* dv = c.f == ICL_FILTER_SEPCONV ? &c.sep.dst
                  : c.f == ICL_FILTER_HARRIS ? &c.har.dst
                  : c.f == ICL_FILTER_NLM    ? &c.nlm.dst
                                             : &c.c2d.dst;
    dv->base += (int64_t)r0 * dv->pitch;
    dv->H = std::min(kMaxRows, d.H - r0);
    dv->y0 = d.y0 + r0;
    if (c.f == ICL_FILTER_HARRIS && c.har.mask) c.har.mask += (int64_t)r0 * c.har.mpitch;
    cudaError_t e = run_variant_rows(c, v, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

static cudaError_t run_variant_rows(const Prepared& pc, const Variant& v, cudaStream_t s) {
  constexpr int kMaxZ = 65535;
  const int batch = pc.f == ICL_FILTER_SEPCONV ? pc.sep.batch
                    : pc.f == ICL_FILTER_HARRIS ? pc.har.batch
                    : pc.f == ICL_FILTER_NLM    ? pc.nlm.batch
                                                : pc.c2d.batch;
  if (batch <= kMaxZ) return run_variant_1(pc, v, s);
  for (int b0 = 0; b0 < batch; b0 += kMaxZ) {
    Prepared c = pc;
    const int nb = std::min(kMaxZ, batch - b0);
    auto shift = [&](SrcView& sv, DstView& dv, int& bt) {
      sv.base += (int64_t)b0 * sv.bstride;
      dv.base += (int64_t)b0 * dv.bstride;
      bt = nb;
    };
    switch (c.f) {
      case ICL_FILTER_SEPCONV: shift(c.sep.src, c.sep.dst, c.sep.batch); break;
      case ICL_FILTER_HARRIS:
        shift(c.har.src, c.har.dst, c.har.batch);
        if (c.har.mask) c.har.mask += (int64_t)b0 * c.har.mbstride;
        break;
      case ICL_FILTER_NLM: shift(c.nlm.src, c.nlm.dst, c.nlm.batch); break;
      case ICL_FILTER_CONV2D: shift(c.c2d.src, c.c2d.dst, c.c2d.batch); break;
    }
    cudaError_t e = run_variant_1(c, v, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

static cudaError_t run_variant_1(const Prepared& pc, const Variant& v, cudaStream_t s) {
  switch (pc.f) {
    case ICL_FILTER_SEPCONV:
      if (v.kind == K_NAIVE) return launch_sep_naive_direct(pc.sep, s);
      if (v.kind == K_TWOPASS) return launch_sep_naive_2pass(pc.sep, s);
      if (v.kind == K_BULK) return launch_sep_bulk(pc.sep, v.nt, v.S, s);
      if (v.kind == K_TILE2) return v.S == 2 ? launch_sep_tile128(pc.sep, s) : launch_sep_tile(pc.sep, v.S == 1, s);
      if (v.kind == K_TEX) return launch_sep_tex(pc.sep, s);
      if (v.kind == K_PMAP) return launch_sep_pmap(pc.sep, v.pm, s);
      return launch_sep_stream(pc.sep, v.nt, v.vec, v.S, s);
    case ICL_FILTER_HARRIS:
      if (v.kind == K_NAIVE) return launch_harris_naive(pc.har, s);
      if (v.kind == K_SHFL) return launch_harris_shfl(pc.har, v.nt, v.S, s, v.vec == 7);
      if (v.kind == K_SLIDE) return launch_harris_slide(pc.har, v.nt, v.vec == 8 ? 2 : v.vec == 6 ? 3 : 1, v.S, s);
      if (v.kind == K_PMAP) return launch_harris_pmap(pc.har, v.pm, s);
      return launch_harris_stream(pc.har, v.nt, v.vec, v.S, s);
    case ICL_FILTER_NLM:
      if (v.kind == K_NAIVE) return launch_nlm_naive(pc.nlm, s);
      if (v.kind == K_TILED) return launch_nlm_tiled(pc.nlm, v.nt, v.S, s);
      if (v.kind == K_BOXR8) return launch_nlm_r8(pc.nlm, s);
      if (v.kind == K_BOXR16) return launch_nlm_r16(pc.nlm, s);
      if (v.kind == K_BOXX2) return launch_nlm_x2(pc.nlm, s);
      if (v.kind == K_BOXW) return launch_nlm_w(pc.nlm, v.S, s);
      if (v.kind == K_BOXSYM) return launch_nlm_sym(pc.nlm, s);
      if (v.kind == K_BOXRING) return launch_nlm_sym_ring(pc.nlm, s);
      if (v.kind == K_BOXSYM8) return launch_nlm_sym8(pc.nlm, s);
      return launch_nlm_boxsum(pc.nlm, 0, s);
    case ICL_FILTER_CONV2D:
      if (v.kind == K_NAIVE) return launch_conv2d_naive(pc.c2d, s);
      if (v.kind == K_TEX) return launch_conv2d_tex(pc.c2d, s);
      return launch_conv2d_tile(pc.c2d, v.S, v.nt == 1, s);
  }
  return cudaErrorInvalidValue;
}

static int variant_id(icl_filter f, const char* name) {
  int n;
  const Variant* vt = table(f, &n);
  for (int i = 0; i < n; ++i)
    if (!strcmp(vt[i].name, name)) return i;
  return 0;
}

// Default (untuned) choice: a heuristic per filter (the measured winners of
// tools/variant_sweep.py on B200 for large images; small images take the
// narrowest CTA for more parallelism).
static int default_variant(const Prepared& pc) {
  switch (pc.f) {
    case ICL_FILTER_SEPCONV:
      if (!pc.a16) return variant_id(pc.f, pc.pixels < (1 << 20) ? "stream_nt64_s16_v1" : "stream_nt64_s64_v1");
      // latency-bound small images (BASELINE configs[0], 512^2, r <= 3): one of the paper's Table-1
      // configurations -- 32x8 work-groups, one pixel per thread, the block + halo in local memory --
      // has the shortest critical path (5.8 vs 8.7 us per call for tile64p, graph-replayed;
      // tools/small_sweep.py, round 2c); up to 2^19 pixels the persistent tile kernel's single pass
      if (pc.pixels <= (1 << 18) && (pc.sep.rx > pc.sep.ry ? pc.sep.rx : pc.sep.ry) <= 3)
        return variant_id(pc.f, "pm_w32x8_c1x1_blk_l1_u4");
      if (pc.pixels <= (1 << 19)) return variant_id(pc.f, "tile64p_v4");
      if (pc.pixels < (1 << 20)) return variant_id(pc.f, "stream_nt32_s8_v4");
      {
        // the vertical halo 2R is re-read per S output rows: S grows with R;
        // from R = 7 the register ring of stream<R> limits occupancy and the
        // shared-memory tile kernel wins (16384^2 sweep)
        // (round 2: FFMA2 in both passes of stream<> moved its crossover with tile64p to R = 9;
        // 16384^2: R = 5 / 6 / 7 / 8 in 0.426 / 0.468 / 0.579 / 0.673 ms)
        // (round 2b: the TMA-fed one-warp stream CTAs beat the cp.async ones at every R <= 10:
        // 16384^2 R = 1 / 2 / 3 / 5 / 8 / 10 in 0.361 / 0.364 / 0.385 / 0.410 / 0.591 / 0.781 ms
        // vs 0.378 / 0.383 / 0.403 / 0.453 / 0.664 / 0.841; 8 x 4096^2 R = 2 0.205 vs 0.218 ms)
        const int R = pc.sep.rx > pc.sep.ry ? pc.sep.rx : pc.sep.ry;
        // (round 2f: branch-free full blocks for R <= 4: 16384^2 R = 3 / 4 in 0.354 / 0.364 ms)
        if (R <= 4) return variant_id(pc.f, "tma_nt32_s16_v4");
        // (round 2f: predicated single-block bodies for R >= 5: 16384^2 R = 5..10 in 0.394 / 0.426 /
        // 0.476 / 0.508 / 0.618 / 0.720 ms, profiles/r02f_sweep16k.txt)
        if (R <= 5) return variant_id(pc.f, "tma_nt32_s32_v4");
        if (R == 6 || R == 8 || R == 10) return variant_id(pc.f, "tma_nt32_s64_v4");
        if (R == 7 || R == 9) return variant_id(pc.f, "tma_nt32_s128_v4");
        return variant_id(pc.f, "tile64p_v4");
      }
    case ICL_FILTER_HARRIS:
      if (!pc.a16) return variant_id(pc.f, "stream_nt64_s64_v1");
      if (pc.har.block > 5) return variant_id(pc.f, pc.pixels < (1 << 20) ? "stream_nt32_s16_v4" : "stream_nt64_s64_v4");
      // (the slide<> family -- separable window sums on the products -- is a tuner candidate only:
      // 0.417-0.42 vs 0.398 ms on 8 x 4096^2; the default keeps the naive order)
      if (pc.pixels < (1 << 16)) return variant_id(pc.f, "stream_nt32_s16_v4");
      // 240-column strips: short row segments keep enough CTAs in flight up to one 4096^2 image
      // (1024^2 24.5 vs 34.8 us, 2048^2 30.7 vs 66 us, 4096^2 76 vs 90 us; 8 x 4096^2 prefers s64)
      // (round 2f: the same kernels with TMA-fed ring blocks, bit-identical: 8 x 4096^2 0.385 vs
      // 0.396 ms, 2048^2 25.4 vs 26.6 us)
      return variant_id(pc.f, pc.pixels <= (1 << 21) ? "shfl_tma_nw2_s8"
                              : pc.pixels <= (1 << 25) ? "shfl_tma_nw2_s16" : "shfl_tma_nw2_s32");
    case ICL_FILTER_NLM:
      // the offset-symmetric TMEM kernel once the launch fills most of one wave of 118 x 128 tiles
      // (2 CTAs/SM; 2048^2: 0.265 vs 0.319 ms for boxsum_x2, 1792^2 a tie, 1536^2 0.266 vs 0.191 ms --
      // profiles/r02e_nlm_sizes.txt)
      if (nlm_sym_supported(pc.nlm.P, pc.nlm.S) && pc.pixels >= (1 << 22)) return variant_id(pc.f, "sym_tmem");
      if (nlm_x2_supported(pc.nlm.P, pc.nlm.S)) return variant_id(pc.f, "boxsum_x2");
      if (nlm_r8_supported(pc.nlm.P, pc.nlm.S)) return variant_id(pc.f, "boxsum_r8");
      return nlm_tiled_supported(pc.nlm.P, pc.nlm.S) ? variant_id(pc.f, "tiled_direct_32x8") : 0;
    case ICL_FILTER_CONV2D:
      if (!pc.a16) return 0;
      return variant_id(pc.f, pc.pixels < (1 << 22) ? "tile_c4r4" : "tile_c4r8");
  }
  return 0;
}

// ------------------------------------------------------------------ tune cache
static std::mutex g_cache_mu;
static std::map<std::string, int> g_cache;

static std::string device_tag() {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return "unknown";
  std::ostringstream os;
  os << prop.name << "|sm" << prop.major << prop.minor << "|" << prop.multiProcessorCount << "SMs|"
     << ICL_VERSION_STRING;
  return os.str();
}

static int cache_lookup(const std::string& key) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_cache.find(key);
  return it == g_cache.end() ? -1 : it->second;
}

static const char* policy() {
  const char* p = getenv("ICL_TUNE_POLICY");
  return p ? p : "off";
}

static icl_status tune_prepared(Prepared& pc, unsigned flags, cudaStream_t s, icl_variant_info* info, int ann_n1 = 0,
                                 int ann_topk = 0, uint64_t ann_seed = 0);

// ---- environment (include/icl.h "Environment"): ICL_LOG, ICL_FORCE_VARIANT, ICL_TUNE_CACHE
static bool env_log() {
  static const bool on = [] {
    const char* e = getenv("ICL_LOG");
    return e && *e && strcmp(e, "0") != 0;
  }();
  return on;
}

static int variant_id(icl_filter f, const char* name);
static const char* filter_name(icl_filter f) {
  switch (f) {
    case ICL_FILTER_SEPCONV: return "sepconv";
    case ICL_FILTER_HARRIS: return "harris";
    case ICL_FILTER_NLM: return "nlm";
    case ICL_FILTER_CONV2D: return "conv2d";
    case ICL_FILTER_SEPCONV3D: return "sepconv3d";
  }
  return "?";
}

// ICL_FORCE_VARIANT="harris=shfl_nw2_s32,nlm=boxsum_x2": process-wide forced variants (the
// thread-local icl_force_variant wins over it); unknown names are reported once and ignored
static int env_force(icl_filter f) {
  static int ids[kNFilters] = {-1, -1, -1, -1, -1};
  static std::once_flag once;
  std::call_once(once, [] {
    const char* e = getenv("ICL_FORCE_VARIANT");
    if (!e) return;
    std::string spec(e);
    size_t pos = 0;
    while (pos < spec.size()) {
      size_t end = spec.find(',', pos);
      if (end == std::string::npos) end = spec.size();
      const std::string item = spec.substr(pos, end - pos);
      pos = end + 1;
      const size_t eq = item.find('=');
      if (eq == std::string::npos) continue;
      const std::string fn = item.substr(0, eq), vn = item.substr(eq + 1);
      for (int k = 0; k < kNFilters; ++k) {
        if (fn != filter_name((icl_filter)k)) continue;
        int n;
        const Variant* vt = table((icl_filter)k, &n);
        int id = -1;
        for (int i = 0; i < n; ++i)
          if (vn == vt[i].name) id = i;
        if (id < 0) fprintf(stderr, "[icl] ICL_FORCE_VARIANT: no variant %s of %s (ignored)\n", vn.c_str(), fn.c_str());
        ids[k] = id;
      }
    }
  });
  return (f >= 0 && f < kNFilters) ? ids[f] : -1;
}

static void env_cache_load();
static void env_cache_save();

static icl_status dispatch(Prepared& pc, cudaStream_t s) {
  if (pc.f < 0 || pc.f >= kNFilters) return fail(ICL_ERR_INVALID_ARG, "unknown filter");
  env_cache_load();
  int n;
  const Variant* vt = table(pc.f, &n);
  int vid = t_force[pc.f] >= 0 ? t_force[pc.f] : env_force(pc.f);
  const char* why_s = "forced";
  icl_status why;
  if (vid >= 0) {
    if (vid >= n) return fail(ICL_ERR_INVALID_ARG, "forced variant %d out of range", vid);
    if (!eligible(pc, vt[vid], &why)) return fail(why, "forced variant %s is not eligible for this call", vt[vid].name);
  } else {
    vid = cache_lookup(pc.key);
    why_s = "tune cache";
    if (vid >= n || (vid >= 0 && !eligible(pc, vt[vid], &why))) vid = -1;
    if (vid < 0) {
      const char* pol = policy();
      if (!strcmp(pol, "require")) return fail(ICL_ERR_NOT_TUNED, "no tune-cache entry for %s", pc.key.c_str());
      if (!strcmp(pol, "on_miss")) {
        icl_variant_info info;
        icl_status st = tune_prepared(pc, 0, s, &info);
        if (st != ICL_OK) return st;
        t_last[pc.f] = info.variant_id;
        if (env_log()) fprintf(stderr, "[icl] %s -> %s (tuned on miss)\n", pc.key.c_str(), info.name);
        return ICL_OK;  // the tuner leaves the winner's output in dst
      }
      vid = default_variant(pc);
      why_s = "default";
      if (!eligible(pc, vt[vid], &why)) {
        vid = 0;
        why_s = "default ineligible -> naive";
      }
    }
  }
  if (env_log()) fprintf(stderr, "[icl] %s -> %s (%s)\n", pc.key.c_str(), vt[vid].name, why_s);
  // NVTX range around the enqueue (free without a profiler attached): Nsight / ncu timelines show
  // which variant each filter call ran
  char rng[96];
  snprintf(rng, sizeof rng, "icl %s %s", filter_name(pc.f), vt[vid].name);
  nvtxRangePushA(rng);
  cudaError_t e = run_variant(pc, vt[vid], s);
  nvtxRangePop();
  if (e != cudaSuccess) return cuda_fail(e, vt[vid].name);
  t_last[pc.f] = vid;
  return ICL_OK;
}

// ------------------------------------------------------------------ preparation
static std::string fmt_key(const char* f, const icl_image* dst, bool a16, const std::string& params) {
  std::ostringstream os;
  os << f << ":W" << dst->width << ":H" << dst->height << ":B" << dst->batch << ":a" << (a16 ? 16 : 4) << ":"
     << params;
  return os.str();
}

static icl_status prep_sepconv(const icl_image* src, const icl_image* dst, const float* tx, int rx, const float* ty,
                               int ry, icl_border border, float cval, const icl_band* band, void* ws, size_t wsb,
                               Prepared* pc) {
  icl_status st;
  if ((st = check_image(src, 4, "src")) || (st = check_image(dst, 4, "dst"))) return st;
  if (!tx || !ty) return fail(ICL_ERR_INVALID_ARG, "null taps");
  if (rx < 0 || ry < 0) return fail(ICL_ERR_INVALID_ARG, "negative radius");
  if (rx > kMaxRadius || ry > kMaxRadius) return fail(ICL_ERR_UNSUPPORTED, "radius > %d", kMaxRadius);
  for (int i = 0; i < 2 * rx + 1; ++i)
    if (!std::isfinite(tx[i])) return fail(ICL_ERR_INVALID_ARG, "non-finite tap");
  for (int i = 0; i < 2 * ry + 1; ++i)
    if (!std::isfinite(ty[i])) return fail(ICL_ERR_INVALID_ARG, "non-finite tap");
  if (overlap(byte_range(src, 4), byte_range(dst, 4))) return fail(ICL_ERR_ALIASING, "src and dst overlap");
  pc->f = ICL_FILTER_SEPCONV;
  if ((st = make_views(src, dst, band, border, cval, ry, ry, &pc->sep.src, &pc->sep.dst))) return st;
  pc->sep.batch = (int)src->batch;
  pc->sep.rx = rx;
  pc->sep.ry = ry;
  pc->sep.fx = tx;
  pc->sep.gy = ty;
  pc->sep.workspace = ws;
  pc->sep.workspace_bytes = wsb;
  {
    const int64_t R = std::max(rx, ry), Hg = pc->sep.src.Hg, sy0 = pc->sep.src.y0, dy0 = pc->sep.dst.y0;
    const int64_t lo = std::max<int64_t>(0, dy0 - R), hi = std::min<int64_t>(Hg - 1, dy0 + dst->height - 1 + R);
    pc->sep.pad_rows_ok = lo >= sy0 && hi <= sy0 + src->height - 1;
  }
  if (ws && wsb) {
    Range w{reinterpret_cast<uintptr_t>(ws), reinterpret_cast<uintptr_t>(ws) + wsb};
    if (overlap(w, byte_range(src, 4)) || overlap(w, byte_range(dst, 4)))
      return fail(ICL_ERR_ALIASING, "workspace overlaps an image");
  }
  pc->a16 = aligned16(src) && aligned16(dst);
  pc->pixels = src->width * dst->height * src->batch;
  pc->dst_bytes_compact = (size_t)pc->pixels * 4;
  std::ostringstream ps;
  ps << "rx" << rx << ":ry" << ry << ":bd" << (int)border;
  pc->key = fmt_key("sepconv", dst, pc->a16, ps.str());
  return ICL_OK;
}

static icl_status prep_harris(const icl_image* src, const icl_image* resp, int block, float k, icl_border border,
                              float cval, const icl_image* mask, float thr, const icl_band* band, Prepared* pc) {
  icl_status st;
  if ((st = check_image(src, 4, "src")) || (st = check_image(resp, 4, "response"))) return st;
  if (block < 1 || block > 7) return fail(ICL_ERR_INVALID_ARG, "block must be in [1, 7]");
  if (!std::isfinite(k)) return fail(ICL_ERR_INVALID_ARG, "k must be finite");
  if (std::isnan(thr)) return fail(ICL_ERR_INVALID_ARG, "threshold is NaN");
  if (overlap(byte_range(src, 4), byte_range(resp, 4))) return fail(ICL_ERR_ALIASING, "src and response overlap");
  pc->f = ICL_FILTER_HARRIS;
  const int a = block / 2, bb = block - 1 - a;
  if ((st = make_views(src, resp, band, border, cval, a + 1, bb + 1, &pc->har.src, &pc->har.dst))) return st;
  pc->har.mask = nullptr;
  pc->har.mpitch = pc->har.mbstride = 0;
  bool mask_a4 = true;
  if (mask && mask->data) {
    if ((st = check_image(mask, 1, "mask"))) return st;
    if (mask->width != resp->width || mask->height != resp->height || mask->batch != resp->batch)
      return fail(ICL_ERR_INVALID_ARG, "mask shape differs from the response");
    if (overlap(byte_range(mask, 1), byte_range(src, 4)) || overlap(byte_range(mask, 1), byte_range(resp, 4)))
      return fail(ICL_ERR_ALIASING, "mask overlaps an image");
    pc->har.mask = static_cast<char*>(mask->data);
    pc->har.mpitch = mask->pitch_bytes;
    pc->har.mbstride = mask->batch > 1 ? mask->batch_stride_bytes : 0;
    mask_a4 = aligned4(mask);
  }
  pc->har.batch = (int)src->batch;
  pc->har.block = block;
  pc->har.k = k;
  pc->har.threshold = thr;
  pc->har.naive_order = false;
  pc->a16 = aligned16(src) && aligned16(resp) && mask_a4;
  pc->pixels = src->width * resp->height * src->batch;
  pc->dst_bytes_compact = (size_t)pc->pixels * 4;
  std::ostringstream ps;
  ps << "B" << block << ":bd" << (int)border << ":m" << (pc->har.mask ? 1 : 0);
  pc->key = fmt_key("harris", resp, pc->a16, ps.str());
  return ICL_OK;
}

static icl_status prep_nlm(const icl_image* src, const icl_image* dst, int P, int S, float h, icl_border border,
                           float cval, const icl_band* band, Prepared* pc) {
  icl_status st;
  if ((st = check_image(src, 4, "src")) || (st = check_image(dst, 4, "dst"))) return st;
  if (P < 0 || P > 3) return fail(ICL_ERR_INVALID_ARG, "patch_radius must be in [0, 3]");
  if (S < 0 || S > 10) return fail(ICL_ERR_INVALID_ARG, "search_radius must be in [0, 10]");
  if (std::isnan(h) || !(h > 0.0f)) return fail(ICL_ERR_INVALID_ARG, "h must be > 0 (or +INF)");
  if (overlap(byte_range(src, 4), byte_range(dst, 4))) return fail(ICL_ERR_ALIASING, "src and dst overlap");
  pc->f = ICL_FILTER_NLM;
  if ((st = make_views(src, dst, band, border, cval, P + S, P + S, &pc->nlm.src, &pc->nlm.dst))) return st;
  pc->nlm.batch = (int)src->batch;
  pc->nlm.P = P;
  pc->nlm.S = S;
  pc->nlm.h = h;
  if (std::isinf(h)) {
    pc->nlm.coef = 0.0f;
  } else {
    const double pw = 2.0 * P + 1.0;
    const double coef = 1.4426950408889634 / (pw * pw * (double)h * (double)h);
    pc->nlm.coef = coef > 3.0e38 ? 3.0e38f : (float)coef;
  }
  pc->a16 = aligned16(src) && aligned16(dst);
  pc->pixels = src->width * dst->height * src->batch;
  pc->dst_bytes_compact = (size_t)pc->pixels * 4;
  std::ostringstream ps;
  ps << "P" << P << ":S" << S << ":bd" << (int)border;
  pc->key = fmt_key("nlm", dst, pc->a16, ps.str());
  return ICL_OK;
}

static icl_status prep_conv2d(const icl_image* src, const icl_image* dst, const float* filt, int r,
                              icl_border border, float cval, const icl_band* band, Prepared* pc) {
  icl_status st;
  if ((st = check_image(src, 1, "src")) || (st = check_image(dst, 4, "dst"))) return st;
  if (r < 0) return fail(ICL_ERR_INVALID_ARG, "radius must be >= 0");
  if (r > 3) return fail(ICL_ERR_UNSUPPORTED, "radius %d > 3", r);
  if (!filt) return fail(ICL_ERR_INVALID_ARG, "null filter");
  if (!std::isfinite(cval)) return fail(ICL_ERR_INVALID_ARG, "border_value must be finite");
  const int nf = (2 * r + 1) * (2 * r + 1);
  for (int k = 0; k < nf; ++k)
    if (!std::isfinite(filt[k])) return fail(ICL_ERR_INVALID_ARG, "filter tap %d is not finite", k);
  if (overlap(byte_range(src, 1), byte_range(dst, 4))) return fail(ICL_ERR_ALIASING, "src and dst overlap");
  pc->f = ICL_FILTER_CONV2D;
  if ((st = make_views(src, dst, band, border, cval, r, r, &pc->c2d.src, &pc->c2d.dst))) return st;
  pc->c2d.batch = (int)src->batch;
  pc->c2d.r = r;
  for (int k = 0; k < 49; ++k) pc->c2d.f[k] = k < nf ? filt[k] : 0.0f;
  pc->a16 = aligned16(src) && aligned16(dst);
  pc->pixels = src->width * dst->height * src->batch;
  pc->dst_bytes_compact = (size_t)pc->pixels * 4;
  std::ostringstream ps;
  ps << "r" << r << ":bd" << (int)border;
  pc->key = fmt_key("conv2d_u8", dst, pc->a16, ps.str());
  return ICL_OK;
}

// ------------------------------------------------------------------ tuner
__global__ void compare_kernel(const char* a, int64_t apitch, int64_t abstride, const float* ref, int W, int H,
                               int64_t nb, unsigned long long* out) {
  // out[0] = #unequal, out[1] = max|a-ref| (float bits), out[2] = max|ref| (float bits)
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= W) return;
  for (int64_t b = blockIdx.z; b < nb; b += gridDim.z)  // grid-stride: any height / batch
    for (int y = blockIdx.y; y < H; y += gridDim.y) {
      const float va = reinterpret_cast<const float*>(a + b * abstride + (int64_t)y * apitch)[x];
      const float vr = ref[(b * H + y) * W + x];
      const bool eq = (va == vr) || (va != va && vr != vr);
      if (!eq) atomicAdd(out, 1ull);
      const float d = fabsf(va - vr);
      atomicMax(reinterpret_cast<unsigned int*>(out + 1), __float_as_uint(d != d ? 3.0e38f : d));
      atomicMax(reinterpret_cast<unsigned int*>(out + 2), __float_as_uint(fabsf(vr)));
    }
}

// Harris acceptance (SURVEY.md §8(c) tolerance): a variant's R must satisfy
// |R - R_naive| <= tol * D(p) per pixel (D from harris_dhat; exact 0 where D = 0), and its mask
// must equal R_naive > t except where |R_naive - t| <= tol * D(p).  out[0] = #bad R, out[1] = #bad mask.
__global__ void compare_harris_kernel(const char* a, int64_t apitch, int64_t abstride, const char* m, int64_t mpitch,
                                      int64_t mbstride, const float* ref, const float* dh, int W, int H, int64_t nb,
                                      float thr, float tol, unsigned long long* out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= W) return;
  for (int64_t b = blockIdx.z; b < nb; b += gridDim.z)
    for (int y = blockIdx.y; y < H; y += gridDim.y) {
      const float va = reinterpret_cast<const float*>(a + b * abstride + (int64_t)y * apitch)[x];
      const int64_t i = (b * H + y) * W + x;
      const float vr = ref[i], d = dh[i];
      const bool okr = d > 0.0f ? fabsf(va - vr) <= tol * d : va == vr;
      if (!okr) atomicAdd(out, 1ull);
      if (m) {
        const unsigned char mv = (unsigned char)m[b * mbstride + (int64_t)y * mpitch + x];
        const bool want = vr > thr;
        if ((mv != 0) != want && !(fabsf(vr - thr) <= tol * d)) atomicAdd(out + 1, 1ull);
      }
    }
}

static std::mutex g_tune_mu;
static void* g_flush = nullptr;
static size_t g_flush_bytes = 0;

static icl_status tune_prepared(Prepared& pc, unsigned flags, cudaStream_t s, icl_variant_info* info, int ann_n1,
                                 int ann_topk, uint64_t ann_seed) {
  std::lock_guard<std::mutex> lk(g_tune_mu);
  int n;
  const Variant* vt = table(pc.f, &n);
  if (!(flags & ICL_TUNE_FORCE)) {
    const int hit = cache_lookup(pc.key);
    icl_status why;
    if (hit >= 0 && hit < n && eligible(pc, vt[hit], &why)) {
      cudaError_t e = run_variant(pc, vt[hit], s);
      if (e != cudaSuccess) return cuda_fail(e, "tune (cached winner)");
      if (info) {
        memset(info, 0, sizeof *info);
        info->variant_id = hit;
        snprintf(info->name, sizeof info->name, "%s", vt[hit].name);
        info->median_us = -1.0f;
        info->from_cache = 1;
      }
      return ICL_OK;
    }
  }
  // Views of the real destination (the problem's dst).
  const DstView real_dst = pc.f == ICL_FILTER_SEPCONV ? pc.sep.dst
                           : pc.f == ICL_FILTER_HARRIS ? pc.har.dst
                           : pc.f == ICL_FILTER_NLM    ? pc.nlm.dst
                                                       : pc.c2d.dst;
  const int W = pc.f == ICL_FILTER_SEPCONV ? pc.sep.src.W
                : pc.f == ICL_FILTER_HARRIS ? pc.har.src.W
                : pc.f == ICL_FILTER_NLM    ? pc.nlm.src.W
                                            : pc.c2d.src.W;
  const int H = real_dst.H;
  const int batch = (int)(pc.pixels / ((int64_t)W * H));
  float* ref = nullptr;
  unsigned long long* cmp = nullptr;
  cudaError_t e;
  if ((e = cudaMalloc(&ref, pc.dst_bytes_compact)) != cudaSuccess) return cuda_fail(e, "tune: cudaMalloc");
  if ((e = cudaMalloc(&cmp, 3 * sizeof(unsigned long long))) != cudaSuccess) {
    cudaFree(ref);
    return cuda_fail(e, "tune: cudaMalloc");
  }
  // L2 flush buffer (timing hygiene): 2x L2, allocated once.
  int dev = 0;
  cudaGetDevice(&dev);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  const size_t ws_bytes = 2 * pc.dst_bytes_compact;
  const bool flush = ws_bytes < (size_t)l2 * 2;
  if (flush && g_flush_bytes < (size_t)l2 * 2) {
    if (g_flush) cudaFree(g_flush);
    g_flush = nullptr;
    g_flush_bytes = 0;
    if (cudaMalloc(&g_flush, (size_t)l2 * 2) == cudaSuccess) g_flush_bytes = (size_t)l2 * 2;
  }
  // Reference: the naive variant (id 0) into the compact scratch buffer.
  Prepared pref = pc;
  DstView cdst{reinterpret_cast<char*>(ref), (int64_t)W * 4, (int64_t)W * H * 4, H, real_dst.y0};
  if (pc.f == ICL_FILTER_SEPCONV) pref.sep.dst = cdst;
  else if (pc.f == ICL_FILTER_HARRIS) { pref.har.dst = cdst; pref.har.mask = nullptr; }
  else if (pc.f == ICL_FILTER_NLM) pref.nlm.dst = cdst;
  else pref.c2d.dst = cdst;
  if ((e = run_variant(pref, vt[0], s)) != cudaSuccess) {
    cudaFree(ref);
    cudaFree(cmp);
    return cuda_fail(e, "tune: reference");
  }
  // Harris: the per-pixel scale D of the tolerance (one extra naive-order pass)
  float* dhat = nullptr;
  if (pc.f == ICL_FILTER_HARRIS && cudaMalloc(&dhat, pc.dst_bytes_compact) == cudaSuccess &&
      launch_harris_dhat(pref.har, dhat, s) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(dhat);
    dhat = nullptr;  // (shapes beyond one launch: the global criterion below)
  }
  cudaEvent_t ev0, ev1;
  cudaEventCreate(&ev0);
  cudaEventCreate(&ev1);
  int best = -1, ncand = 0, nrej = 0;
  float best_us = 0.0f;
  float seen_best_us = 1e38f;
  // Time one variant: verify against the naive output, then the median of >= 10 launches.
  auto evaluate = [&](int v, float* med_out) -> bool {
    ++ncand;
    if ((e = run_variant(pc, vt[v], s)) != cudaSuccess) { ++nrej; cudaGetLastError(); return false; }
    if (!(flags & ICL_TUNE_NO_VERIFY) && v != 0) {
      cudaMemsetAsync(cmp, 0, 3 * sizeof(unsigned long long), s);
      dim3 g((W + 255) / 256, H < 65535 ? H : 65535, batch < 65535 ? batch : 65535);
      if (dhat) {
        compare_harris_kernel<<<g, 256, 0, s>>>(real_dst.base, real_dst.pitch, real_dst.bstride, pc.har.mask,
                                                pc.har.mpitch, pc.har.mbstride, ref, dhat, W, H, batch,
                                                pc.har.threshold, 1e-4f, cmp);
        unsigned long long hc[3];
        cudaMemcpyAsync(hc, cmp, sizeof hc, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (hc[0] != 0 || hc[1] != 0) { ++nrej; return false; }
      } else {
      compare_kernel<<<g, 256, 0, s>>>(real_dst.base, real_dst.pitch, real_dst.bstride, ref, W, H, batch, cmp);
      unsigned long long hc[3];
      cudaMemcpyAsync(hc, cmp, sizeof hc, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      float md, mr;
      unsigned int b1 = (unsigned int)hc[1], b2 = (unsigned int)hc[2];
      memcpy(&md, &b1, 4);
      memcpy(&mr, &b2, 4);
      // sepconv / conv2d variants share one fp32 order per output: bit-identical or rejected
      const bool exact = pc.f == ICL_FILTER_SEPCONV || pc.f == ICL_FILTER_CONV2D;
      const bool ok = exact ? hc[0] == 0 : md <= 1e-4f * std::max(mr, 1e-30f);
      if (!ok) { ++nrej; return false; }
      }
    }
    // warm-up then timed reps (median).  A candidate whose first timed launches already take more
    // than 2x the best median seen so far cannot win the 0.5% tie-break: it keeps the median of
    // those (>= 3) launches and the remaining reps are skipped (the pm_* Table-1 space holds
    // hundreds of such configurations; every candidate is still verified and timed)
    for (int w = 0; w < 2; ++w) run_variant(pc, vt[v], s);
    std::vector<float> ts;
    float total = 0.0f;
    for (int r = 0; r < 50 && (r < 10 || total < 50000.0f); ++r) {
      if (r == 3 && seen_best_us < 1e30f) {
        std::vector<float> t3(ts);
        std::sort(t3.begin(), t3.end());
        if (t3[1] > 2.0f * seen_best_us) break;
      }
      if (flush && g_flush) cudaMemsetAsync(g_flush, r & 0xff, g_flush_bytes, s);
      cudaEventRecord(ev0, s);
      run_variant(pc, vt[v], s);
      cudaEventRecord(ev1, s);
      cudaEventSynchronize(ev1);
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, ev0, ev1);
      ts.push_back(ms * 1000.0f);
      total += ms * 1000.0f;
      if (r >= 10 && total > 200000.0f) break;
    }
    std::sort(ts.begin(), ts.end());
    *med_out = ts[ts.size() / 2];
    seen_best_us = std::min(seen_best_us, *med_out);
    return true;
  };
  if (ann_n1 <= 0) {  // exhaustive
    for (int v = 0; v < n; ++v) {
      icl_status why;
      if (!eligible(pc, vt[v], &why)) continue;
      float med;
      if (!evaluate(v, &med)) continue;
      if (best < 0 || med < best_us * 0.995f) { best = v; best_us = med; }
    }
  } else {  // model-guided (ann.cu): features = kind one-hot, log2 CTA threads, vector width, log2 segment rows
    std::vector<int> ids;
    for (int v = 0; v < n; ++v) {
      icl_status why;
      if (eligible(pc, vt[v], &why)) ids.push_back(v);
    }
    // features: kind one-hot, log2 CTA threads, vector width / coarsening x, log2 segment rows /
    // coarsening y, and the Table-1 axes of the pmap configurations (log2 wx, log2 wy, mapping
    // one-hot, local memory, log2 unroll; 0 for the hand-built kinds)
    constexpr int NK = K_COUNT, NF = NK + 3 + 7;
    std::vector<double> feats(ids.size() * NF, 0.0);
    for (size_t i = 0; i < ids.size(); ++i) {
      const Variant& vv = vt[ids[i]];
      double* x = &feats[i * NF];
      x[vv.kind] = 1.0;
      x[NK] = std::log2(1.0 + vv.nt);
      x[NK + 1] = vv.vec;
      x[NK + 2] = std::log2(1.0 + vv.S);
      if (vv.kind == K_PMAP) {
        x[NK + 3] = std::log2((double)vv.pm.wx);
        x[NK + 4] = std::log2((double)vv.pm.wy);
        x[NK + 5 + vv.pm.map] = 1.0;
        x[NK + 8] = vv.pm.local;
        x[NK + 9] = std::log2((double)vv.pm.unr);
      }
    }
    double bv = 0.0;
    int bi = -1;
    ann_search((int)ids.size(), NF, feats.data(),
               [&](int i, double* val) {
                 float med;
                 if (!evaluate(ids[i], &med)) return false;
                 *val = med;
                 return true;
               },
               ann_n1, ann_topk, ann_seed, nullptr, &bi, &bv);
    if (bi >= 0) { best = ids[bi]; best_us = (float)bv; }
  }
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  icl_status st = ICL_OK;
  if (best < 0) st = fail(ICL_ERR_CUDA, "tune: no variant succeeded");
  else {
    if ((e = run_variant(pc, vt[best], s)) != cudaSuccess) st = cuda_fail(e, "tune: winner");
    {
      std::lock_guard<std::mutex> lk2(g_cache_mu);
      g_cache[pc.key] = best;
    }
    if (info) {
      memset(info, 0, sizeof *info);
      info->variant_id = best;
      snprintf(info->name, sizeof info->name, "%s", vt[best].name);
      info->median_us = best_us;
      info->n_candidates = ncand;
      info->n_rejected = nrej;
      info->from_cache = 0;
    }
  }
  cudaStreamSynchronize(s);
  cudaFree(ref);
  cudaFree(cmp);
  if (dhat) cudaFree(dhat);
  if (st == ICL_OK && (e = cudaGetLastError()) != cudaSuccess) st = cuda_fail(e, "tune");
  return st;
}

// ------------------------------------------------------------------ host images
// A call whose src / dst / mask data pointer is HOST memory (pinned or
// pageable) streams the images through the GPU in row bands: band k's input
// rows (plus the stencil halo) are copied H2D into one of NSET device staging
// sets, the filter runs on that band through the icl_band path (so sepconv /
// Harris results equal the device-resident call bit for bit), and the band's
// output is copied D2H -- H2D of band k+1, compute of band k and D2H of band
// k-1 overlap on three library streams.  The work forks from and joins back
// into the caller's stream, so stream order and events on it bracket the
// whole transfer + compute.  Device-resident operands are used in place.
static std::atomic<uint64_t> g_h2d_bytes{0}, g_d2h_bytes{0};

static bool is_host_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;  // unknown to CUDA: plain host memory
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeUnregistered;
}

namespace {
constexpr int kNSet = 3;
struct Stager {
  std::mutex mu;
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  cudaEvent_t in_ready[kNSet], comp_done[kNSet], out_done[kNSet], fork, join_c, join_d;
  char* buf = nullptr;
  size_t cap = 0;
  uint64_t seq = 0;  // bands issued so far (all calls): staging set = seq % kNSet
  bool init = false;
};
std::mutex g_stagers_mu;
std::map<int, Stager*> g_stagers;
}  // namespace

static Stager* stager_for_current_device(icl_status* st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    *st = cuda_fail(e, "host path: cudaGetDevice");
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(g_stagers_mu);
  Stager*& sg = g_stagers[dev];
  if (!sg) sg = new Stager();
  return sg;
}

static int64_t round16(int64_t b) { return (b + 15) / 16 * 16; }

using ChunkCall = std::function<icl_status(const icl_image*, const icl_image*, const icl_image*, const icl_band*,
                                           cudaStream_t)>;

// src/dst/mask validated by the caller's prep_*; up/down = stencil rows.
static icl_status run_host(const icl_image* src, const icl_image* dst, const icl_image* mask, const icl_band* band,
                           int up, int down, const ChunkCall& call, cudaStream_t user, int src_elem = 4) {
  icl_status st = ICL_OK;
  Stager* sg = stager_for_current_device(&st);
  if (!sg) return st;
  std::lock_guard<std::mutex> lk(sg->mu);
  cudaError_t e = cudaSuccess;
  if (!sg->init) {
    const unsigned fl = cudaEventDisableTiming;
    if ((e = cudaStreamCreateWithFlags(&sg->h2d, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&sg->comp, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&sg->d2h, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "host path: stream create");
    for (int i = 0; i < kNSet; ++i) {
      if ((e = cudaEventCreateWithFlags(&sg->in_ready[i], fl)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&sg->comp_done[i], fl)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&sg->out_done[i], fl)) != cudaSuccess)
        return cuda_fail(e, "host path: event create");
    }
    if ((e = cudaEventCreateWithFlags(&sg->fork, fl)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&sg->join_c, fl)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&sg->join_d, fl)) != cudaSuccess)
      return cuda_fail(e, "host path: event create");
    sg->init = true;
  }
  const bool src_h = is_host_ptr(src->data), dst_h = is_host_ptr(dst->data);
  const bool msk_h = mask && mask->data && is_host_ptr(mask->data);
  const int64_t W = src->width, B = src->batch;
  const int64_t Hg = band ? band->global_height : src->height;
  const int64_t sy0 = band ? band->src_y0 : 0, dy0 = band ? band->dst_y0 : 0;
  const int64_t rows_out = dst->height;
  // rows per band: ~16 MiB of output (ICL_HOST_CHUNK_ROWS overrides, for tests)
  int64_t CH = std::max<int64_t>(1, (16ll << 20) / (W * 4));
  if (const char* env = std::getenv("ICL_HOST_CHUNK_ROWS")) CH = std::max<int64_t>(1, std::atoll(env));
  CH = std::min(CH, rows_out);
  const int64_t spitch = round16(W * src_elem), dpitch = round16(W * 4), mpitch = round16(W);
  const size_t in_bytes = src_h ? (size_t)(CH + up + down) * spitch : 0;
  const size_t out_bytes = dst_h ? (size_t)CH * dpitch : 0;
  const size_t m_bytes = msk_h ? (size_t)CH * mpitch : 0;
  const size_t set_bytes = round16(in_bytes) + round16(out_bytes) + round16(m_bytes);
  if (set_bytes * kNSet > sg->cap) {
    // previous calls' copies may still read the old staging buffer
    cudaStreamSynchronize(sg->h2d);
    cudaStreamSynchronize(sg->comp);
    cudaStreamSynchronize(sg->d2h);
    if (sg->buf) cudaFree(sg->buf);
    sg->buf = nullptr;
    sg->cap = 0;
    if ((e = cudaMalloc(&sg->buf, set_bytes * kNSet)) != cudaSuccess) return cuda_fail(e, "host path: staging");
    sg->cap = set_bytes * kNSet;
  }
  // fixed set stride: a set's region never moves between calls, whatever
  // their in/out/mask sizes, so the per-set events protect all of it
  const size_t stride = sg->cap / kNSet;
  auto set_in = [&](int k) { return sg->buf + k * stride; };
  auto set_out = [&](int k) { return sg->buf + k * stride + round16(in_bytes); };
  auto set_msk = [&](int k) { return sg->buf + k * stride + round16(in_bytes) + round16(out_bytes); };
  if ((e = cudaEventRecord(sg->fork, user)) != cudaSuccess) return cuda_fail(e, "host path: fork");
  cudaStreamWaitEvent(sg->h2d, sg->fork, 0);
  cudaStreamWaitEvent(sg->comp, sg->fork, 0);
  cudaStreamWaitEvent(sg->d2h, sg->fork, 0);
  const int64_t sb = src->batch > 1 ? src->batch_stride_bytes : 0;
  const int64_t db = dst->batch > 1 ? dst->batch_stride_bytes : 0;
  const int64_t mb = (mask && mask->batch > 1) ? mask->batch_stride_bytes : 0;
  uint64_t h2d = 0, d2h = 0;
  for (int64_t b = 0; b < B && st == ICL_OK; ++b) {
    for (int64_t a = dy0; a < dy0 + rows_out && st == ICL_OK; a += CH) {
      const int64_t ee = std::min(a + CH, dy0 + rows_out);
      const int64_t lo = std::max(std::max<int64_t>(0, a - up), sy0);
      const int64_t hi = std::min(std::min(Hg, ee + down), sy0 + src->height);
      // staging sets rotate across calls too (a call issued from another user
      // stream may still be using them): always wait for the set's last users
      const int set = (int)(sg->seq++ % kNSet);
      const char* sptr = static_cast<const char*>(src->data) + b * sb + (lo - sy0) * src->pitch_bytes;
      char* dptr = static_cast<char*>(dst->data) + b * db + (a - dy0) * dst->pitch_bytes;
      char* mptr = mask && mask->data ? static_cast<char*>(mask->data) + b * mb + (a - dy0) * mask->pitch_bytes
                                      : nullptr;
      icl_image iv{const_cast<char*>(sptr), W, hi - lo, src->pitch_bytes, 1, 0};
      icl_image ov{dptr, W, ee - a, dst->pitch_bytes, 1, 0};
      icl_image mv{mptr, W, ee - a, mask ? mask->pitch_bytes : 0, 1, 0};
      if (src_h) {
        // the whole set must be free: its previous band's kernel and D2H
        cudaStreamWaitEvent(sg->h2d, sg->comp_done[set], 0);
        cudaStreamWaitEvent(sg->h2d, sg->out_done[set], 0);
        e = cudaMemcpy2DAsync(set_in(set), spitch, sptr, src->pitch_bytes, W * src_elem, hi - lo,
                              cudaMemcpyHostToDevice, sg->h2d);
        if (e != cudaSuccess) { st = cuda_fail(e, "host path: H2D"); break; }
        cudaEventRecord(sg->in_ready[set], sg->h2d);
        cudaStreamWaitEvent(sg->comp, sg->in_ready[set], 0);
        iv.data = set_in(set);
        iv.pitch_bytes = spitch;
        h2d += (uint64_t)(W * src_elem) * (hi - lo);
      }
      cudaStreamWaitEvent(sg->comp, sg->out_done[set], 0);  // set outputs drained by the previous D2H
      if (dst_h) { ov.data = set_out(set); ov.pitch_bytes = dpitch; }
      if (msk_h) { mv.data = set_msk(set); mv.pitch_bytes = mpitch; }
      const icl_band bc{Hg, lo, a};
      st = call(&iv, &ov, mask && mask->data ? &mv : nullptr, &bc, sg->comp);
      if (st != ICL_OK) break;
      cudaEventRecord(sg->comp_done[set], sg->comp);
      if (dst_h || msk_h) {
        cudaStreamWaitEvent(sg->d2h, sg->comp_done[set], 0);
        if (dst_h) {
          e = cudaMemcpy2DAsync(dptr, dst->pitch_bytes, set_out(set), dpitch, W * 4, ee - a, cudaMemcpyDeviceToHost,
                                sg->d2h);
          if (e != cudaSuccess) { st = cuda_fail(e, "host path: D2H"); break; }
          d2h += (uint64_t)(W * 4) * (ee - a);
        }
        if (msk_h) {
          e = cudaMemcpy2DAsync(mptr, mask->pitch_bytes, set_msk(set), mpitch, W, ee - a, cudaMemcpyDeviceToHost,
                                sg->d2h);
          if (e != cudaSuccess) { st = cuda_fail(e, "host path: D2H mask"); break; }
          d2h += (uint64_t)W * (ee - a);
        }
        cudaEventRecord(sg->out_done[set], sg->d2h);
      }
    }
  }
  // join (also on error: nothing of this call may outlive the caller's stream order)
  cudaEventRecord(sg->join_c, sg->comp);
  cudaEventRecord(sg->join_d, sg->d2h);
  cudaStreamWaitEvent(sg->h2d, sg->join_c, 0);  // the h2d stream is drained by the compute it feeds
  cudaStreamWaitEvent(user, sg->join_c, 0);
  cudaStreamWaitEvent(user, sg->join_d, 0);
  g_h2d_bytes.fetch_add(h2d);
  g_d2h_bytes.fetch_add(d2h);
  if (st == ICL_OK && (e = cudaGetLastError()) != cudaSuccess) st = cuda_fail(e, "host path");
  return st;
}

static bool any_host(const icl_image* a, const icl_image* b, const icl_image* c) {
  return (a && a->data && is_host_ptr(a->data)) || (b && b->data && is_host_ptr(b->data)) ||
         (c && c->data && is_host_ptr(c->data));
}

}  // namespace icl

using namespace icl;

// ======================================================================== C ABI
extern "C" {

icl_status icl_sepconv(const icl_image* src, const icl_image* dst, const float* taps_x, int rx, const float* taps_y,
                       int ry, icl_border border, float border_value, const icl_band* band, void* workspace,
                       size_t workspace_bytes, void* stream) {
  Prepared pc;
  icl_status st = prep_sepconv(src, dst, taps_x, rx, taps_y, ry, border, border_value, band, workspace,
                               workspace_bytes, &pc);
  if (st != ICL_OK) return st;
  if (any_host(src, dst, nullptr)) {
    return run_host(src, dst, nullptr, band, ry, ry,
                    [&](const icl_image* s, const icl_image* d, const icl_image*, const icl_band* b, cudaStream_t cs) {
                      return icl_sepconv(s, d, taps_x, rx, taps_y, ry, border, border_value, b, nullptr, 0, cs);
                    },
                    static_cast<cudaStream_t>(stream));
  }
  return dispatch(pc, static_cast<cudaStream_t>(stream));
}

size_t icl_sepconv_workspace_bytes(int64_t width, int64_t height, int64_t batch, int ry) {
  if (width < 1 || height < 1 || batch < 1 || ry < 0) return 0;
  return sep_2pass_workspace(width, height, batch, ry);
}

static icl_status harris_impl(const icl_image* src, const icl_image* response, int block, float k,
                              icl_border border, float border_value, const icl_image* mask, float threshold,
                              const icl_band* band, void* stream, bool naive_order) {
  Prepared pc;
  icl_status st = prep_harris(src, response, block, k, border, border_value, mask, threshold, band, &pc);
  if (st != ICL_OK) return st;
  pc.har.naive_order = naive_order;
  if (any_host(src, response, mask)) {
    const int a = block / 2, bb = block - 1 - a;
    return run_host(src, response, mask, band, a + 1, bb + 1,
                    [&](const icl_image* s, const icl_image* d, const icl_image* m, const icl_band* b, cudaStream_t cs) {
                      return harris_impl(s, d, block, k, border, border_value, m, threshold, b, cs, naive_order);
                    },
                    static_cast<cudaStream_t>(stream));
  }
  return dispatch(pc, static_cast<cudaStream_t>(stream));
}

extern "C++" {
namespace icl {
icl_status harris_naive_order(const icl_image* src, const icl_image* response, int block, float k, icl_border border,
                              float border_value, const icl_image* mask, float threshold, const icl_band* band,
                              void* stream) {
  return harris_impl(src, response, block, k, border, border_value, mask, threshold, band, stream, true);
}
}  // namespace icl
}  // extern "C++"

icl_status icl_harris(const icl_image* src, const icl_image* response, int block, float k, icl_border border,
                      float border_value, const icl_image* mask, float threshold, const icl_band* band,
                      void* stream) {
  return harris_impl(src, response, block, k, border, border_value, mask, threshold, band, stream, false);
}

icl_status icl_blur_harris(const icl_image* src, const icl_image* response, const float* taps_x, int rx,
                           const float* taps_y, int ry, icl_border blur_border, float blur_border_value, int block,
                           float k, icl_border border, float border_value, const icl_image* mask, float threshold,
                           const icl_band* band, void* workspace, size_t workspace_bytes, void* stream) {
  if (!src || !response) return fail(ICL_ERR_INVALID_ARG, "null image descriptor");
  if (!taps_x || !taps_y) return fail(ICL_ERR_INVALID_ARG, "null taps");
  if (rx < 0 || ry < 0) return fail(ICL_ERR_INVALID_ARG, "negative radius");
  if (rx > 3 || ry > 3) return fail(ICL_ERR_UNSUPPORTED, "blur radius > 3 (fused chain instantiations: 0..3)");
  for (int i = 0; i < 2 * rx + 1; ++i)
    if (!std::isfinite(taps_x[i])) return fail(ICL_ERR_INVALID_ARG, "non-finite tap");
  for (int i = 0; i < 2 * ry + 1; ++i)
    if (!std::isfinite(taps_y[i])) return fail(ICL_ERR_INVALID_ARG, "non-finite tap");
  if (block > 5 && block <= 7) return fail(ICL_ERR_UNSUPPORTED, "fused chain supports Harris blocks 1..5");
  if (blur_border != ICL_BORDER_CONSTANT && blur_border != ICL_BORDER_CLAMP)
    return fail(ICL_ERR_INVALID_ARG, "blur border must be ICL_BORDER_CONSTANT or ICL_BORDER_CLAMP");
  if (std::isnan(blur_border_value)) return fail(ICL_ERR_INVALID_ARG, "blur border_value is NaN");
  Prepared pc;
  icl_status st = prep_harris(src, response, block, k, border, border_value, mask, threshold, band, &pc);
  if (st != ICL_OK) return st;
  if (any_host(src, response, mask)) return fail(ICL_ERR_INVALID_ARG, "icl_blur_harris takes device images only");
  // the stencil of the chain: the Harris rows plus the blur radius
  const int a = block / 2, bb = block - 1 - a, R = std::max(rx, ry);
  if ((st = make_views(src, response, band, border, border_value, a + 1 + R, bb + 1 + R, &pc.har.src, &pc.har.dst)))
    return st;
  if (!pc.a16) return fail(ICL_ERR_UNSUPPORTED, "fused chain needs 16-byte aligned images, pitches and a 4-byte aligned mask");
  const int64_t Hg = band ? band->global_height : src->height, dy0 = band ? band->dst_y0 : 0;
  const int64_t sy0 = band ? band->src_y0 : 0;
  // Two-pass schedule when the caller gives room for the intermediate: the blurred rows Harris
  // reads (its halo, clipped to the image) through icl_sepconv, then icl_harris on them -- the
  // same values as the fused kernel, and faster on B200 (Harris is issue-bound)
  const int64_t m0 = std::max<int64_t>(0, dy0 - (a + 1)), m1 = std::min<int64_t>(Hg, dy0 + response->height + bb + 1);
  const int64_t mpitch = (src->width + 3) / 4 * 4 * 4, mrows = m1 - m0;
  const size_t need = (size_t)(mrows * mpitch * src->batch);
  if (workspace && workspace_bytes >= need) {
    Range w{reinterpret_cast<uintptr_t>(workspace), reinterpret_cast<uintptr_t>(workspace) + need};
    if (overlap(w, byte_range(src, 4)) || overlap(w, byte_range(response, 4)) ||
        (mask && mask->data && overlap(w, byte_range(mask, 1))))
      return fail(ICL_ERR_ALIASING, "workspace overlaps an image");
    if (reinterpret_cast<uintptr_t>(workspace) % 16) return fail(ICL_ERR_INVALID_ARG, "workspace not 16-byte aligned");
    icl_image mid{workspace, src->width, mrows, mpitch, src->batch, mrows * mpitch};
    icl_band bs{Hg, sy0, m0}, bh{Hg, m0, dy0};
    if ((st = icl_sepconv(src, &mid, taps_x, rx, taps_y, ry, blur_border, blur_border_value, &bs, nullptr, 0, stream)))
      return st;
    // the naive-order Harris variants: the fused kernel's consumer keeps that order (bit-identical)
    return harris_naive_order(&mid, response, block, k, border, border_value, mask, threshold, &bh, stream);
  }
  const int S = pc.pixels <= (1 << 25) ? 16 : 64;
  if (src->batch > 65535 || (pc.har.dst.H + S - 1) / S > 65535)
    return fail(ICL_ERR_UNSUPPORTED, "fused chain: batch > 65535 or image taller than 65535 row segments");
  SrcView raw = pc.har.src;
  raw.border = blur_border == ICL_BORDER_CLAMP ? kBorderClamp : kBorderConstant;
  raw.cval = blur_border_value;
  cudaError_t e = launch_blur_harris(pc.har, raw, taps_x, rx, taps_y, ry, S, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "blur_harris");
  return ICL_OK;
}

icl_status icl_sepconv3d(const icl_image* src, const icl_image* dst, const float* taps_x, int rx, const float* taps_y,
                         int ry, const float* taps_z, int rz, icl_border border, float border_value, void* stream) {
  icl_status st;
  if ((st = check_image(src, 4, "src")) || (st = check_image(dst, 4, "dst"))) return st;
  if (!taps_x || !taps_y || !taps_z) return fail(ICL_ERR_INVALID_ARG, "null taps");
  if (rx < 0 || ry < 0 || rz < 0) return fail(ICL_ERR_INVALID_ARG, "negative radius");
  if (rx > 7 || ry > 7 || rz > 7) return fail(ICL_ERR_UNSUPPORTED, "3-D radius > 7");
  for (int i = 0; i < 2 * rx + 1; ++i)
    if (!std::isfinite(taps_x[i])) return fail(ICL_ERR_INVALID_ARG, "non-finite tap");
  for (int i = 0; i < 2 * ry + 1; ++i)
    if (!std::isfinite(taps_y[i])) return fail(ICL_ERR_INVALID_ARG, "non-finite tap");
  for (int i = 0; i < 2 * rz + 1; ++i)
    if (!std::isfinite(taps_z[i])) return fail(ICL_ERR_INVALID_ARG, "non-finite tap");
  if (border != ICL_BORDER_CONSTANT && border != ICL_BORDER_CLAMP)
    return fail(ICL_ERR_INVALID_ARG, "border must be ICL_BORDER_CONSTANT or ICL_BORDER_CLAMP");
  if (std::isnan(border_value)) return fail(ICL_ERR_INVALID_ARG, "border_value is NaN");
  if (src->width != dst->width || src->height != dst->height || src->batch != dst->batch)
    return fail(ICL_ERR_INVALID_ARG, "src and dst volumes differ in shape");
  if (src->height > 524280) return fail(ICL_ERR_UNSUPPORTED, "volume slices taller than 524280 rows");
  if (src->height * src->pitch_bytes >= (1ll << 31))  // the tile loader's slice-relative offsets are int32
    return fail(ICL_ERR_UNSUPPORTED, "volume slices of 2 GiB or more");
  if (overlap(byte_range(src, 4), byte_range(dst, 4))) return fail(ICL_ERR_ALIASING, "src and dst overlap");
  if (any_host(src, dst, nullptr)) return fail(ICL_ERR_INVALID_ARG, "icl_sepconv3d takes device volumes only");
  Sep3Params p;
  p.src = static_cast<const char*>(src->data);
  p.spitch = src->pitch_bytes;
  p.sslice = src->batch > 1 ? src->batch_stride_bytes : 0;
  p.dst = static_cast<char*>(dst->data);
  p.dpitch = dst->pitch_bytes;
  p.dslice = dst->batch > 1 ? dst->batch_stride_bytes : 0;
  p.W = (int)src->width;
  p.H = (int)src->height;
  p.D = (int)src->batch;
  p.border = border == ICL_BORDER_CLAMP ? kBorderClamp : kBorderConstant;
  p.cval = border_value;
  p.rx = rx;
  p.ry = ry;
  p.rz = rz;
  for (int i = 0; i < 15; ++i) p.fx[i] = p.gy[i] = p.hz[i] = 0.0f;
  for (int i = 0; i < 2 * rx + 1; ++i) p.fx[i] = taps_x[i];
  for (int i = 0; i < 2 * ry + 1; ++i) p.gy[i] = taps_y[i];
  for (int i = 0; i < 2 * rz + 1; ++i) p.hz[i] = taps_z[i];
  const int vid = t_force[ICL_FILTER_SEPCONV3D] >= 0 ? t_force[ICL_FILTER_SEPCONV3D] : 1;
  cudaError_t e = launch_sep3d(p, vid, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "sepconv3d");
  t_last[ICL_FILTER_SEPCONV3D] = vid;
  return ICL_OK;
}

size_t icl_blur_harris_workspace_bytes(int64_t width, int64_t height, int64_t batch, int block) {
  if (width < 1 || height < 1 || batch < 1 || block < 1) return 0;
  return (size_t)((height + block + 1) * ((width + 3) / 4 * 4) * 4 * batch);
}

icl_status icl_nlm(const icl_image* src, const icl_image* dst, int patch_radius, int search_radius, float h,
                   icl_border border, float border_value, const icl_band* band, void* stream) {
  Prepared pc;
  icl_status st = prep_nlm(src, dst, patch_radius, search_radius, h, border, border_value, band, &pc);
  if (st != ICL_OK) return st;
  if (any_host(src, dst, nullptr)) {
    const int r = patch_radius + search_radius;
    return run_host(src, dst, nullptr, band, r, r,
                    [&](const icl_image* s, const icl_image* d, const icl_image*, const icl_band* b, cudaStream_t cs) {
                      return icl_nlm(s, d, patch_radius, search_radius, h, border, border_value, b, cs);
                    },
                    static_cast<cudaStream_t>(stream));
  }
  return dispatch(pc, static_cast<cudaStream_t>(stream));
}

icl_status icl_conv2d_u8(const icl_image* src, const icl_image* dst, const float* filter, int radius,
                         icl_border border, float border_value, const icl_band* band, void* stream) {
  Prepared pc;
  icl_status st = prep_conv2d(src, dst, filter, radius, border, border_value, band, &pc);
  if (st != ICL_OK) return st;
  if (any_host(src, dst, nullptr)) {
    return run_host(src, dst, nullptr, band, radius, radius,
                    [&](const icl_image* s, const icl_image* d, const icl_image*, const icl_band* b, cudaStream_t cs) {
                      return icl_conv2d_u8(s, d, filter, radius, border, border_value, b, cs);
                    },
                    static_cast<cudaStream_t>(stream), 1);
  }
  return dispatch(pc, static_cast<cudaStream_t>(stream));
}

static icl_status tune_entry(const icl_problem* p, unsigned flags, void* stream, icl_variant_info* chosen, int n1,
                             int topk, uint64_t seed);

icl_status icl_tune(const icl_problem* p, unsigned flags, void* stream, icl_variant_info* chosen) {
  return tune_entry(p, flags, stream, chosen, 0, 0, 0);
}

icl_status icl_tune_ann(const icl_problem* p, int n1, int topk, uint64_t seed, void* stream, icl_variant_info* chosen) {
  if (n1 < 1 || topk < 0) return fail(ICL_ERR_INVALID_ARG, "n1 must be >= 1 and topk >= 0");
  return tune_entry(p, ICL_TUNE_FORCE, stream, chosen, n1, topk, seed);
}

static icl_status tune_entry(const icl_problem* p, unsigned flags, void* stream, icl_variant_info* chosen, int n1,
                             int topk, uint64_t seed) {
  if (!p) return fail(ICL_ERR_INVALID_ARG, "null problem");
  if (any_host(&p->src, &p->dst, p->filter == ICL_FILTER_HARRIS ? &p->mask : nullptr))
    return fail(ICL_ERR_INVALID_ARG, "icl_tune needs device-resident images");
  Prepared pc;
  icl_status st;
  switch (p->filter) {
    case ICL_FILTER_SEPCONV:
      st = prep_sepconv(&p->src, &p->dst, p->taps_x, p->rx, p->taps_y, p->ry, p->border, p->border_value, nullptr,
                        p->workspace, p->workspace_bytes, &pc);
      break;
    case ICL_FILTER_CONV2D:
      st = prep_conv2d(&p->src, &p->dst, p->filter2d, p->radius2d, p->border, p->border_value, nullptr, &pc);
      break;
    case ICL_FILTER_HARRIS:
      st = prep_harris(&p->src, &p->dst, p->block, p->k, p->border, p->border_value, &p->mask, p->threshold,
                       nullptr, &pc);
      break;
    case ICL_FILTER_NLM:
      st = prep_nlm(&p->src, &p->dst, p->patch_radius, p->search_radius, p->h, p->border, p->border_value,
                    nullptr, &pc);
      break;
    default:
      return fail(ICL_ERR_INVALID_ARG, "unknown filter");
  }
  if (st != ICL_OK) return st;
  env_cache_load();
  const icl_status ts = tune_prepared(pc, flags, static_cast<cudaStream_t>(stream), chosen, n1, topk, seed);
  if (ts == ICL_OK) env_cache_save();
  return ts;
}

extern "C++" {
namespace icl {
// ICL_TUNE_CACHE=path: the tune cache persists across processes -- loaded (when the file exists
// and matches this device/build) before the first dispatch, saved after every tuning
static void env_cache_load() {
  static std::once_flag once;
  std::call_once(once, [] {
    const char* p = getenv("ICL_TUNE_CACHE");
    if (!p || !*p) return;
    FILE* f = fopen(p, "r");
    if (!f) return;
    fclose(f);
    if (icl_tune_cache_load(p) != ICL_OK && env_log())
      fprintf(stderr, "[icl] ICL_TUNE_CACHE %s not loaded: %s\n", p, icl_last_error());
  });
}

static void env_cache_save() {
  const char* p = getenv("ICL_TUNE_CACHE");
  if (p && *p && icl_tune_cache_save(p) != ICL_OK && env_log())
    fprintf(stderr, "[icl] ICL_TUNE_CACHE %s not saved: %s\n", p, icl_last_error());
}
}  // namespace icl
}  // extern "C++"

icl_status icl_tune_cache_save(const char* path) {
  if (!path) return fail(ICL_ERR_INVALID_ARG, "null path");
  std::ofstream f(path);
  if (!f) return fail(ICL_ERR_INVALID_ARG, "cannot open %s", path);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  f << "{\n\"device\": \"" << device_tag() << "\",\n\"entries\": {\n";
  size_t i = 0;
  for (auto& kv : g_cache) {
    int n;
    const Variant* vt = table(kv.first.rfind("sepconv", 0) == 0   ? ICL_FILTER_SEPCONV
                              : kv.first.rfind("harris", 0) == 0 ? ICL_FILTER_HARRIS
                              : kv.first.rfind("conv2d", 0) == 0 ? ICL_FILTER_CONV2D
                                                                  : ICL_FILTER_NLM,
                              &n);
    f << "\"" << kv.first << "\": [" << kv.second << ", \"" << (kv.second < n ? vt[kv.second].name : "?") << "\"]"
      << (++i < g_cache.size() ? "," : "") << "\n";
  }
  f << "}\n}\n";
  return f ? ICL_OK : fail(ICL_ERR_INVALID_ARG, "write failed: %s", path);
}

icl_status icl_tune_cache_load(const char* path) {
  if (!path) return fail(ICL_ERR_INVALID_ARG, "null path");
  std::ifstream f(path);
  if (!f) return fail(ICL_ERR_INVALID_ARG, "cannot open %s", path);
  std::string line, dev;
  std::map<std::string, int> entries;
  while (std::getline(f, line)) {
    if (line.rfind("\"device\": \"", 0) == 0) {
      const size_t e = line.rfind('"');
      dev = line.substr(11, e - 11);
    } else if (!line.empty() && line[0] == '"' && line.find("\": [") != std::string::npos) {
      const size_t q = line.find("\": [");
      const std::string key = line.substr(1, q - 1);
      const int id = atoi(line.c_str() + q + 4);
      entries[key] = id;
    }
  }
  if (dev != device_tag()) return fail(ICL_ERR_INVALID_ARG, "tune cache is for another device/build: %s", dev.c_str());
  std::lock_guard<std::mutex> lk(g_cache_mu);
  for (auto& kv : entries) g_cache[kv.first] = kv.second;
  return ICL_OK;
}

void icl_tune_cache_clear(void) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_cache.clear();
}

int icl_tune_cache_size(void) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  return (int)g_cache.size();
}

int icl_variant_count(icl_filter filter) {
  int n;
  table(filter, &n);
  return n;
}

icl_status icl_variant_name(icl_filter filter, int id, char* buf, size_t len) {
  int n;
  const Variant* vt = table(filter, &n);
  if (!vt || id < 0 || id >= n || !buf || !len) return fail(ICL_ERR_INVALID_ARG, "bad variant query");
  snprintf(buf, len, "%s", vt[id].name);
  return ICL_OK;
}

icl_status icl_force_variant(icl_filter filter, int id) {
  int n;
  if (!table(filter, &n)) return fail(ICL_ERR_INVALID_ARG, "unknown filter");
  if (id < -1 || id >= n) return fail(ICL_ERR_INVALID_ARG, "variant id %d out of range", id);
  t_force[filter] = id;
  return ICL_OK;
}

int icl_last_variant(icl_filter filter) {
  if (filter < 0 || filter >= kNFilters) return -1;
  return t_last[filter];
}

uint64_t icl_launch_count(void) { return g_launches.load(); }

void icl_transfer_bytes(uint64_t* h2d, uint64_t* d2h) {
  if (h2d) *h2d = g_h2d_bytes.load();
  if (d2h) *d2h = g_d2h_bytes.load();
}

const char* icl_last_error(void) { return t_err.c_str(); }

const char* icl_version(void) { return ICL_VERSION_STRING; }

icl_status icl_copy_2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width_bytes, int64_t rows,
                       void* stream) {
  if (!dst || !src || width_bytes < 0 || rows < 0 || dpitch < width_bytes || spitch < width_bytes)
    return fail(ICL_ERR_INVALID_ARG, "bad copy arguments");
  cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width_bytes, (size_t)rows,
                                    cudaMemcpyDefault, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? ICL_OK : cuda_fail(e, "icl_copy_2d");
}

icl_status icl_fill_uniform(const icl_image* img, uint64_t seed, int64_t row0, void* stream) {
  icl_status st = check_image(img, 4, "img");
  if (st != ICL_OK) return st;
  if (is_host_ptr(img->data)) return fail(ICL_ERR_INVALID_ARG, "icl_fill_uniform needs a device image");
  cudaError_t e = launch_fill_uniform(static_cast<float*>(img->data), img->width, img->height, img->pitch_bytes,
                                      img->batch, img->batch > 1 ? img->batch_stride_bytes : 0, seed, row0,
                                      static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fill_uniform");
  return ICL_OK;
}

}  // extern "C"
