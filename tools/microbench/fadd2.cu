// FADD2 vs FFMA2 forms on the FMA pipe (B200): which packed form reaches 128 lanes/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fadd2 fadd2.cu && ./fadd2
#include <cuda_runtime.h>
#include <cstdio>
constexpr int ITERS = 4096, ILP = 8;
__global__ void k_fadd2_rr(float* out, float a) {  // r[i] = r[i] + r[i+1]  (2 distinct register pairs)
  float2 r[ILP];
  for (int i = 0; i < ILP; ++i) r[i] = make_float2(threadIdx.x * 1e-3f + i * a, i * 0.5f);
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = __fadd2_rn(r[i], r[(i + 3) % ILP]);
  float s = 0;
  for (int i = 0; i < ILP; ++i) s += r[i].x + r[i].y;
  if (s == 1234.5f) out[0] = s;
}
__global__ void k_fma1_rr(float* out, float one) {  // r[i] = r[i+1] * (one, one) + r[i]  (FFMA2 with a uniform pair)
  float2 r[ILP];
  const float2 O = make_float2(one, one);
  for (int i = 0; i < ILP; ++i) r[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = __ffma2_rn(r[(i + 3) % ILP], O, r[i]);
  float s = 0;
  for (int i = 0; i < ILP; ++i) s += r[i].x + r[i].y;
  if (s == 1234.5f) out[0] = s;
}
__global__ void k_ffma2_3(float* out, float a) {  // r[i] = r[i+1] * r[i+2] + r[i]  (3 distinct pairs)
  float2 r[ILP];
  for (int i = 0; i < ILP; ++i) r[i] = make_float2(threadIdx.x * 1e-3f + i * a, i * 0.5f);
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = __ffma2_rn(r[(i + 3) % ILP], r[(i + 5) % ILP], r[i]);
  float s = 0;
  for (int i = 0; i < ILP; ++i) s += r[i].x + r[i].y;
  if (s == 1234.5f) out[0] = s;
}
__global__ void k_ffma2_sq(float* out, float a) {  // r[i] = r[i+1]^2 + r[i]  (2 distinct pairs)
  float2 r[ILP];
  for (int i = 0; i < ILP; ++i) r[i] = make_float2(threadIdx.x * 1e-3f + i * a, i * 0.5f);
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = __ffma2_rn(r[(i + 3) % ILP], r[(i + 3) % ILP], r[i]);
  float s = 0;
  for (int i = 0; i < ILP; ++i) s += r[i].x + r[i].y;
  if (s == 1234.5f) out[0] = s;
}
__global__ void k_ffma_3(float* out, float a) {  // scalar, 3 distinct registers
  float r[ILP];
  for (int i = 0; i < ILP; ++i) r[i] = threadIdx.x * 1e-3f + i * a;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = __fmaf_rn(r[(i + 3) % ILP], r[(i + 5) % ILP], r[i]);
  float s = 0;
  for (int i = 0; i < ILP; ++i) s += r[i];
  if (s == 1234.5f) out[0] = s;
}
template <typename K>
void run(const char* name, K k, float arg, int lanes_per_inst) {
  float* out;
  cudaMalloc(&out, 4);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = nsm * 8, threads = 256;
  k<<<blocks, threads>>>(out, arg);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(out, arg);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double inst = 5.0 * blocks * threads * (double)ITERS * ILP;  // thread-instructions
  const double per_clk_sm = inst / (ms * 1e-3) / nsm / (clk * 1e3);
  printf("%-40s %7.1f thread-inst/clk/SM = %6.1f lanes/clk/SM\n", name, per_clk_sm, per_clk_sm * lanes_per_inst);
  cudaFree(out);
}
int main() {
  run("FADD2 r = r + s (2 reg pairs)", k_fadd2_rr, 1.0f, 2);
  run("FFMA2 r = s * (1,1) + r (uniform pair)", k_fma1_rr, 1.0f, 2);
  run("FFMA2 r = s * t + r (3 reg pairs)", k_ffma2_3, 1.0f, 2);
  run("FFMA2 r = s * s + r (2 reg pairs)", k_ffma2_sq, 1.0f, 2);
  run("FFMA  r = s * t + r (3 regs)", k_ffma_3, 1.0f, 1);
  return 0;
}
