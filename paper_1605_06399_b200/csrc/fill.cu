// fill.cu -- device implementation of the synthetic-input generator
// synth.uniform_image (SplitMix64 counter hash).  Input generation only: no
// filter arithmetic.  Tested equal to synth/ in tests/test_gpu_*.py.
#include "internal.h"

namespace icl {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_uniform_kernel(float* base, int64_t W, int64_t H, int64_t pitch, int64_t bstride,
                                    uint64_t seed, int64_t row0) {
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t y = blockIdx.y;
  const int64_t b = blockIdx.z;
  if (x >= W || y >= H) return;
  const uint64_t s = seed + (uint64_t)b;
  const uint64_t key = s * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
  const uint64_t idx = (uint64_t)((row0 + y) * W + x);
  const uint64_t z = splitmix64(idx ^ key);
  const float v = (float)(z >> 40) * 5.9604644775390625e-08f;  // 2^-24, exact
  reinterpret_cast<float*>(reinterpret_cast<char*>(base) + b * bstride + y * pitch)[x] = v;
}

cudaError_t launch_fill_uniform(float* base, int64_t W, int64_t H, int64_t pitch, int64_t batch,
                                int64_t bstride, uint64_t seed, int64_t row0, cudaStream_t s) {
  if (H > 65535 * 64) return cudaErrorInvalidValue;
  for (int64_t y0 = 0; y0 < H; y0 += 65535) {
    const int64_t h = (H - y0) < 65535 ? (H - y0) : 65535;
    dim3 grd((unsigned)((W + 255) / 256), (unsigned)h, (unsigned)batch);
    fill_uniform_kernel<<<grd, 256, 0, s>>>(
        reinterpret_cast<float*>(reinterpret_cast<char*>(base) + y0 * pitch), W, h, pitch, bstride, seed,
        row0 + y0);
    count_launch();
  }
  return cudaGetLastError();
}

}  // namespace icl
