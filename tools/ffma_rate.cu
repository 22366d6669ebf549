// Harness-only: SIMT fp32 FMA throughput on sm_100a -- scalar FFMA (3-register form) vs packed
// fma.rn.f32x2 (FFMA2), many independent chains per thread, all SMs.  Control for the batched
// small-matrix path (config 4): is a SIMT product competitive with 3xTF32 mma.sync?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ffma_rate tools/ffma_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_loop(float* out, int iters, float x, float y) {
  float c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = threadIdx.x * 0.001f + i;
  float a = x + threadIdx.x, b = y;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(c[i]) : "f"(a), "f"(b));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 1.2345f) out[0] = s;
}

__global__ void ffma2_loop(float* out, int iters, float x, float y) {
  unsigned long long c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = ((unsigned long long)__float_as_uint(i * 1.f) << 32) | __float_as_uint(threadIdx.x * 1.f);
  const unsigned long long a = ((unsigned long long)__float_as_uint(x) << 32) | __float_as_uint(x + threadIdx.x);
  const unsigned long long b = ((unsigned long long)__float_as_uint(y) << 32) | __float_as_uint(y);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c[i]) : "l"(a), "l"(b));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += __uint_as_float((uint32_t)c[i]) + __uint_as_float((uint32_t)(c[i] >> 32));
  if (s == 1.2345f) out[0] = s;
}

// outer-product form as a SIMT GEMM would issue it: 4 x 8 register tile, operands from
// registers that change every k (a0..a3 broadcast pairs, b pairs)
__global__ void ffma2_outer(float* out, int iters, const float* __restrict__ in) {
  unsigned long long c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) c[i][j] = 0ull;
  __shared__ float sa[64], sb[64];
  if (threadIdx.x < 64) { sa[threadIdx.x] = in[threadIdx.x]; sb[threadIdx.x] = in[64 + threadIdx.x]; }
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 av = *reinterpret_cast<const float4*>(sa + (k & 7) * 4);
      const float4 b0 = *reinterpret_cast<const float4*>(sb + (k & 7) * 8);
      const float4 b1 = *reinterpret_cast<const float4*>(sb + (k & 7) * 8 + 4);
      const unsigned long long bp[4] = {
          ((unsigned long long)__float_as_uint(b0.y) << 32) | __float_as_uint(b0.x),
          ((unsigned long long)__float_as_uint(b0.w) << 32) | __float_as_uint(b0.z),
          ((unsigned long long)__float_as_uint(b1.y) << 32) | __float_as_uint(b1.x),
          ((unsigned long long)__float_as_uint(b1.w) << 32) | __float_as_uint(b1.z)};
      const float ar[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const unsigned long long ap = ((unsigned long long)__float_as_uint(ar[i]) << 32) | __float_as_uint(ar[i]);
#pragma unroll
        for (int j = 0; j < 4; ++j) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c[i][j]) : "l"(ap), "l"(bp[j]));
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += __uint_as_float((uint32_t)c[i][j]);
  if (s == 1.2345f) out[0] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 1024);
  cudaMemset(out, 0, 1024);
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int blocks = sms * 4, threads = 256, iters = 40000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  auto report = [&](const char* name, double fma_per_thread_iter) {
    const double fmas = fma_per_thread_iter * iters * (double)blocks * threads;
    printf("%-28s %8.2f ms  %7.2f TFLOP/s  %6.1f FMA/clk/SM (at %d MHz nominal)\n", name, ms,
           2 * fmas / ms / 1e9, fmas / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  };
  for (int rep = 0; rep < 2; ++rep) {
    ffma_loop<<<blocks, threads>>>(out, 100, 1.0001f, 0.9999f);
    cudaEventRecord(e0);
    ffma_loop<<<blocks, threads>>>(out, iters, 1.0001f, 0.9999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    report("FFMA (scalar, 16 chains)", 16);
    ffma2_loop<<<blocks, threads>>>(out, 100, 1.0001f, 0.9999f);
    cudaEventRecord(e0);
    ffma2_loop<<<blocks, threads>>>(out, iters, 1.0001f, 0.9999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    report("FFMA2 (f32x2, 16 chains)", 32);
    ffma2_outer<<<blocks, threads>>>(out, 10, out);
    cudaEventRecord(e0);
    ffma2_outer<<<blocks, threads>>>(out, iters / 8, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    report("FFMA2 outer 4x8 from LDS", 8 * 32 / 8.0);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
