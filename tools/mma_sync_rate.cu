// Harness-only: legacy mma.sync throughput on sm_100a (tf32 m16n8k8, f32 FFMA reference).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void tf32_loop(float* out, int iters) {
  uint32_t a[4] = {threadIdx.x, 1u, 2u, 3u}, b[2] = {5u, 7u};
  float c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};"
        : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0; for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 1.2345f) out[0] = s;
}
int main() {
  float* out; cudaMalloc(&out, 64);
  int blocks = 148 * 4, threads = 256, iters = 20000;
  tf32_loop<<<blocks, threads>>>(out, 100); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); tf32_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 16 * 8 * 8 * 8.0 * iters * blocks * (threads / 32);
  printf("mma.sync m16n8k8 tf32: %.1f TFLOP/s (%s)\n", flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
