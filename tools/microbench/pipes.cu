// pipes.cu -- B200 microbenchmarks for the FP32 roof of the NLM/Harris kernels:
// FFMA vs packed FFMA2 vs FADD2 throughput, MUFU.EX2 throughput, and shared-memory
// LDS.32/LDS.128 throughput.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
template <int ILP>
__global__ void k_ffma(float* out, float a, float b) {
  float r[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) r[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = __fmaf_rn(r[i], a, b);
  }
  float s = 0; 
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += r[i];
  if (s == 1234.5f) out[0] = s;
}
template <int ILP>
__global__ void k_ffma_rr(float* out, const float* ab) {  // 3 distinct register operands
  float a = ab[0], b = ab[1];
  float r[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) r[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = __fmaf_rn(r[i], a, r[(i + 1) % ILP]);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += r[i];
  if (s == 1234.5f) out[0] = s;
}
template <int ILP>
__global__ void k_ffma2(float* out, float a, float b) {
  float2 r[ILP];
  const float2 A = make_float2(a, a), B = make_float2(b, b);
#pragma unroll
  for (int i = 0; i < ILP; ++i) r[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = __ffma2_rn(r[i], A, B);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += r[i].x + r[i].y;
  if (s == 1234.5f) out[0] = s;
}
template <int ILP>
__global__ void k_ffma2_rr(float* out, const float* ab) {
  float2 A = make_float2(ab[0], ab[1]);
  float2 r[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) r[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = __ffma2_rn(r[i], A, r[(i + 1) % ILP]);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += r[i].x + r[i].y;
  if (s == 1234.5f) out[0] = s;
}
template <int ILP>
__global__ void k_fadd2(float* out, float a) {
  float2 r[ILP];
  const float2 A = make_float2(a, -a);
#pragma unroll
  for (int i = 0; i < ILP; ++i) r[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = __fadd2_rn(r[i], A);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += r[i].x + r[i].y;
  if (s == 1234.5f) out[0] = s;
}
template <int ILP>
__global__ void k_ex2(float* out, float a) {
  float r[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) r[i] = -(threadIdx.x * 1e-3f + i);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(r[i]));
      r[i] = y;
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += r[i];
  if (s == 1234.5f) out[0] = s;
}
template <int ILP>
__global__ void k_mix_ex2_ffma2(float* out, float a) {  // 1 ex2 : 4 FFMA2
  float r[ILP];
  float2 q[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { r[i] = -(threadIdx.x * 1e-3f + i); q[i] = make_float2(i, i + 1); }
  const float2 A = make_float2(a, a);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(r[i]));
      r[i] = y;
      q[i] = __ffma2_rn(q[i], A, q[i]); q[i] = __ffma2_rn(q[i], A, q[i]);
      q[i] = __ffma2_rn(q[i], A, q[i]); q[i] = __ffma2_rn(q[i], A, q[i]);
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += r[i] + q[i].x + q[i].y;
  if (s == 1234.5f) out[0] = s;
}
__global__ void k_lds32(float* out) {
  __shared__ float sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
  __syncthreads();
  float s = 0;
  int idx = threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) s += sm[(idx + k * 32) & 4095];
    idx += 1;
  }
  if (s == 1234.5f) out[0] = s;
}
__global__ void k_lds128(float* out) {
  __shared__ float4 sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_float4(i, i, i, i);
  __syncthreads();
  float s = 0;
  int idx = threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { float4 v = sm[(idx + k * 32) & 1023]; s += v.x + v.w; }
    idx += 1;
  }
  if (s == 1234.5f) out[0] = s;
}
template <int ILP>
__global__ void k_shfl(float* out) {  // independent SHFL.IDX chains
  float r[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) r[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = __shfl_down_sync(0xffffffffu, r[i], 1 + (i & 3));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += r[i];
  if (s == 1234.5f) out[0] = s;
}
// 4 SHFL + 4 conflict-free LDS.32 per iteration: do they share the LSU/MIO path?
__global__ void k_shfl_lds(float* out) {
  __shared__ float sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
  __syncthreads();
  float r[4], s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) r[i] = threadIdx.x * 1e-3f + i;
  int idx = threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) r[i] = __shfl_down_sync(0xffffffffu, r[i], 1 + i);
#pragma unroll
    for (int k = 0; k < 4; ++k) s += sm[(idx + k * 32) & 4095];
    idx += 1;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) s += r[i];
  if (s == 1234.5f) out[0] = s;
}

// NA independent FFMA2 chains + NB independent scalar FFMA chains per iteration: do FFMA2 (FMA-heavy
// pipe) and scalar FFMA (heavy or lite) overlap?  Reported as FMA lanes (flop/2) per clk per SM.
template <int NA, int NB>
__global__ void k_mix2(float* out, float a, float b) {
  float2 r2[NA > 0 ? NA : 1];
  float r1[NB > 0 ? NB : 1];
  const float2 A = make_float2(a, a), B2 = make_float2(b, b);
#pragma unroll
  for (int i = 0; i < NA; ++i) r2[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
#pragma unroll
  for (int i = 0; i < NB; ++i) r1[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NA; ++i) r2[i] = __ffma2_rn(r2[i], A, B2);
#pragma unroll
    for (int i = 0; i < NB; ++i) r1[i] = __fmaf_rn(r1[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NA; ++i) s += r2[i].x + r2[i].y;
#pragma unroll
  for (int i = 0; i < NB; ++i) s += r1[i];
  if (s == 1234.5f) out[0] = s;
}

template <typename F>
double run(F launch, double ops_per_thread_iter, int blocks, int threads) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  launch(); cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) launch();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = ops_per_thread_iter * ITERS * (double)blocks * threads * 5;
  return ops / (ms * 1e-3);
}

int main() {
  float* d; cudaMalloc(&d, 64); float hab[2] = {0.999f, 0.001f}; float* ab; cudaMalloc(&ab, 8);
  cudaMemcpy(ab, hab, 8, cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int B = sms * 8, T = 256;
  printf("SMs %d, max clock %.0f MHz\n", sms, clk / 1e3);
  double per_sm_clk = sms * (clk * 1e3);
  double r;
  r = run([&] { k_ffma<8><<<B, T>>>(d, 0.999f, 0.001f); }, 8, B, T);
  printf("FFMA (imm/const operands) : %7.2f Tinst/s  %6.1f /clk/SM  = %6.1f TFLOP/s\n", r / 1e12, r / per_sm_clk, 2 * r / 1e12);
  r = run([&] { k_ffma_rr<8><<<B, T>>>(d, ab); }, 8, B, T);
  printf("FFMA (3 reg operands)     : %7.2f Tinst/s  %6.1f /clk/SM  = %6.1f TFLOP/s\n", r / 1e12, r / per_sm_clk, 2 * r / 1e12);
  r = run([&] { k_ffma2<8><<<B, T>>>(d, 0.999f, 0.001f); }, 8, B, T);
  printf("FFMA2 (uniform operands)  : %7.2f Tinst/s  %6.1f /clk/SM  = %6.1f TFLOP/s\n", r / 1e12, r / per_sm_clk, 4 * r / 1e12);
  r = run([&] { k_ffma2_rr<8><<<B, T>>>(d, ab); }, 8, B, T);
  printf("FFMA2 (reg operands)      : %7.2f Tinst/s  %6.1f /clk/SM  = %6.1f TFLOP/s\n", r / 1e12, r / per_sm_clk, 4 * r / 1e12);
  r = run([&] { k_fadd2<8><<<B, T>>>(d, 0.001f); }, 8, B, T);
  printf("FADD2                     : %7.2f Tinst/s  %6.1f /clk/SM  = %6.1f TFLOP/s\n", r / 1e12, r / per_sm_clk, 2 * r / 1e12);
  r = run([&] { k_ex2<8><<<B, T>>>(d, 0.5f); }, 8, B, T);
  printf("MUFU.EX2                  : %7.2f Tinst/s  %6.1f /clk/SM\n", r / 1e12, r / per_sm_clk);
  r = run([&] { k_mix_ex2_ffma2<4><<<B, T>>>(d, 0.999f); }, 4, B, T);
  printf("EX2 + 4 FFMA2 (per ex2)   : %7.2f Tinst/s  %6.1f ex2/clk/SM\n", r / 1e12, r / per_sm_clk);
  r = run([&] { k_lds32<<<B, T>>>(d); }, 8, B, T);
  printf("LDS.32 (conflict-free)    : %7.2f Tinst/s  %6.1f words/clk/SM\n", r / 1e12, r / per_sm_clk);
  r = run([&] { k_lds128<<<B, T>>>(d); }, 8, B, T);
  printf("LDS.128 (conflict-free)   : %7.2f Tinst/s  %6.1f words/clk/SM\n", r / 1e12, 4 * r / per_sm_clk);
  r = run([&] { k_mix2<8, 0><<<B, T>>>(d, 0.999f, 0.001f); }, 16, B, T);
  printf("FFMA2 only (8 chains)     : %6.1f FMA lanes/clk/SM\n", r / per_sm_clk);
  r = run([&] { k_mix2<4, 4><<<B, T>>>(d, 0.999f, 0.001f); }, 12, B, T);
  printf("4 FFMA2 + 4 FFMA          : %6.1f FMA lanes/clk/SM\n", r / per_sm_clk);
  r = run([&] { k_mix2<4, 8><<<B, T>>>(d, 0.999f, 0.001f); }, 16, B, T);
  printf("4 FFMA2 + 8 FFMA          : %6.1f FMA lanes/clk/SM\n", r / per_sm_clk);
  r = run([&] { k_mix2<2, 8><<<B, T>>>(d, 0.999f, 0.001f); }, 12, B, T);
  printf("2 FFMA2 + 8 FFMA          : %6.1f FMA lanes/clk/SM\n", r / per_sm_clk);
  r = run([&] { k_mix2<0, 8><<<B, T>>>(d, 0.999f, 0.001f); }, 8, B, T);
  printf("FFMA only (8 chains)      : %6.1f FMA lanes/clk/SM\n", r / per_sm_clk);
  r = run([&] { k_shfl<8><<<B, T>>>(d); }, 8, B, T);
  printf("SHFL.DOWN (independent)   : %7.2f Tinst/s  %6.1f lanes/clk/SM\n", r / 1e12, r / per_sm_clk);
  r = run([&] { k_shfl_lds<<<B, T>>>(d); }, 8, B, T);
  printf("4 SHFL + 4 LDS.32         : %7.2f Tinst/s  %6.1f lane-ops/clk/SM\n", r / 1e12, r / per_sm_clk);
  return 0;
}
