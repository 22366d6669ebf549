// Harness-only: mma.sync m16n8k8 tf32 throughput with the batched kernel's operand pattern
// (2 m-tiles x NB n-tiles, 3 products per tile: lo*hi, hi*hi, hi*lo; every HMMA reads different
// A / B registers) vs the same-operand loop of mma_sync_rate.cu.  No loads, no other work.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_pattern_rate tools/mma_pattern_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int NB>
__global__ void pattern(float* out, int iters) {
  uint32_t ah[2][4], al[2][4], bh[NB][2], bl[NB][2];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 4; ++j) { ah[i][j] = threadIdx.x * 7 + i * 4 + j; al[i][j] = ah[i][j] ^ 0x55; }
  for (int i = 0; i < NB; ++i)
    for (int j = 0; j < 2; ++j) { bh[i][j] = threadIdx.x * 3 + i * 2 + j; bl[i][j] = bh[i][j] ^ 0x33; }
  float big[2][NB][4] = {}, sml[2][NB][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
#pragma unroll
      for (int mb = 0; mb < 2; ++mb)
#pragma unroll
        for (int j = 0; j < NB; ++j) mma(sml[mb][j], al[mb], bh[j][0], bh[j][1]);
#pragma unroll
      for (int mb = 0; mb < 2; ++mb)
#pragma unroll
        for (int j = 0; j < NB; ++j) mma(big[mb][j], ah[mb], bh[j][0], bh[j][1]);
#pragma unroll
      for (int mb = 0; mb < 2; ++mb)
#pragma unroll
        for (int j = 0; j < NB; ++j) mma(sml[mb][j], ah[mb], bl[j][0], bl[j][1]);
    }
  }
  float s = 0;
  for (int mb = 0; mb < 2; ++mb)
    for (int j = 0; j < NB; ++j)
      for (int e = 0; e < 4; ++e) s += big[mb][j][e] + sml[mb][j][e];
  if (s == 1.2345f) out[0] = s;
}

template <int NB>
void run(const char* name, int warps_per_sm) {
  float* out;
  cudaMalloc(&out, 64);
  const int blocks = 148, threads = 32 * warps_per_sm, iters = 4000;
  pattern<NB><<<blocks, threads>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  pattern<NB><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 16 * 8 * 8 * (3.0 * 2 * NB * 4) * iters * blocks * warps_per_sm;
  printf("%s warps/SM=%2d: %.1f TFLOP/s (%s)\n", name, warps_per_sm, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  for (int w : {4, 8, 16, 32}) run<2>("pattern 2x2 tiles (WPM=2)", w);
  for (int w : {4, 8, 16}) run<4>("pattern 2x4 tiles (WPM=1)", w);
  return 0;
}
