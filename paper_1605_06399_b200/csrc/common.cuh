// common.cuh -- device-side helpers shared by the filter kernels (product code;
// nothing here is shared with oracle/).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace icl {

constexpr int kBorderConstant = 0;
constexpr int kBorderClamp = 1;
constexpr int kMaxRadius = 15;

// A source image as the kernels see it: band-aware, batch-aware.
//   global row y (0 <= y < Hg) lives at local row (y - y0) of `base`.
struct SrcView {
  const char* base;   // image 0, local row 0
  int64_t pitch;      // bytes
  int64_t bstride;    // bytes between images
  int W;              // width (global == local)
  int Hg;             // global height (boundary applies at 0 / Hg-1)
  int y0;             // global row of local row 0
  int border;         // kBorderConstant / kBorderClamp
  float cval;         // constant border value
  int Hl;             // rows held locally from y0 (a band buffer's rows; Hg - y0 .. for a whole image)
};

struct DstView {
  char* base;
  int64_t pitch;
  int64_t bstride;
  int H;   // rows to produce (local)
  int y0;  // global row of local row 0
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ const float* src_row(const SrcView& s, int b, int gy) {
  return reinterpret_cast<const float*>(s.base + (int64_t)b * s.bstride + (int64_t)(gy - s.y0) * s.pitch);
}
__device__ __forceinline__ float* dst_row(const DstView& d, int b, int ly) {
  return reinterpret_cast<float*>(d.base + (int64_t)b * d.bstride + (int64_t)ly * d.pitch);
}

// in_B(x, y) at GLOBAL coordinates (Fig. 3).
__device__ __forceinline__ float read_B(const SrcView& s, int b, int x, int gy) {
  if (x < 0 || x >= s.W || gy < 0 || gy >= s.Hg) {
    if (s.border == kBorderConstant) return s.cval;
    x = clampi(x, 0, s.W - 1);
    gy = clampi(gy, 0, s.Hg - 1);
  }
  // a row outside the band buffer is never inside an output's stencil (make_views checks the
  // stencil rows are held); tiles that over-reach the last output row read 0 there, not memory
  // past the buffer
  if ((unsigned)(gy - s.y0) >= (unsigned)s.Hl) return 0.0f;
  return __ldg(src_row(s, b, gy) + x);
}

// ---------------------------------------------------------------- cp.async
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte async copy global->shared with zero-fill of the bytes >= src_bytes.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Streaming (evict-first) vector store.
__device__ __forceinline__ void st_cs4(float* p, float4 v) { __stcs(reinterpret_cast<float4*>(p), v); }

}  // namespace icl

namespace icl {
// ---------------------------------------------------------------- mbarrier + TMA bulk copy
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(smem_u32(bar)), "r"(parity)
                 : "memory");
  } while (!done);
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`.
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// 3-D TMA tile load (cp.async.bulk.tensor: x = column, y = local row, z = image) into shared
// memory, completion counted on `bar` (expect_tx armed by the issuing thread).
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
}  // namespace icl
