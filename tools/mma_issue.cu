// Harness-only: mma.sync m16n8k8 tf32 throughput vs resident warps per SM sub-partition, with
// the batched kernel's pattern (8 accumulator tiles x 3 products per k-step).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3},{%4,%5,%6,%7},{%8,%9},{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
template <int CH>
__global__ void loop(float* out, int iters) {
  uint32_t a[4] = {threadIdx.x, 1u, 2u, 3u}, b[2] = {5u, 7u};
  float c[CH][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) mma(c[i], a[0], a[1], a[2], a[3], b[0], b[1]);
  }
  float s = 0; for (int i = 0; i < CH; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 1.2345f) out[0] = s;
}
template <int CH>
void run(int warps_per_sm) {
  float* out; cudaMalloc(&out, 64);
  int iters = 4000;
  loop<CH><<<148, 32 * warps_per_sm>>>(out, 10); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); loop<CH><<<148, 32 * warps_per_sm>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double mmas = (double)CH * iters * warps_per_sm * 148;
  double tf = 2.0 * 16 * 8 * 8 * mmas / ms / 1e9;
  double cyc_per_mma_smsp = ms * 1e-3 * 1.965e9 / (mmas / (148 * 4));
  printf("chains %2d warps/SM %2d: %6.1f TFLOP/s  %.2f cycles per HMMA per SMSP (at 1.965 GHz)\n", CH, warps_per_sm, tf, cyc_per_mma_smsp);
  cudaFree(out);
}
int main() {
  for (int w : {4, 8, 16, 32}) { run<8>(w); run<16>(w); run<24>(w); }
  return 0;
}
