// smem.cu -- shared-memory load bandwidth on B200: LDS.32 / LDS.64 / LDS.128,
// conflict-free, independent accumulators (no dependency chain), 8 warps x 4 CTAs/SM.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048
template <int V>
__global__ void k_lds(float* out) {
  __shared__ __align__(16) float sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 0.5f;
  __syncthreads();
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int base = w * 1024 / V;  // in units of V floats
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = ((base + k * 32 + lane + it) & (8192 / V - 1)) * V;
      if (V == 1) acc[k] += sm[idx];
      if (V == 2) { float2 v = *reinterpret_cast<const float2*>(sm + idx); acc[k] += v.x + v.y; }
      if (V == 4) { float4 v = *reinterpret_cast<const float4*>(sm + idx); acc[k] += (v.x + v.y) + (v.z + v.w); }
    }
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k];
  if (s == 1234.5f) out[0] = s;
}
template <int V>
void run(const char* name) {
  float* d; cudaMalloc(&d, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int B = sms * 4, T = 256;
  k_lds<V><<<B, T>>>(d); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k_lds<V><<<B, T>>>(d);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double bytes = 5.0 * B * T * ITERS * 8 * 4 * V;
  printf("%-8s %8.1f GB/s  %6.1f B/clk/SM\n", name, bytes / ms / 1e6, bytes / (ms * 1e-3) / (sms * clk * 1e3));
}
int main() { run<1>("LDS.32"); run<2>("LDS.64"); run<4>("LDS.128"); return 0; }
