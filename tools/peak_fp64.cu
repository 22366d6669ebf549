// Microbenchmark: FP64 tensor (DMMA via mma.sync f64) and FP64 SIMT (DFMA) register-loop peaks
// on sm_100a. Harness-only (not part of the library). Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("{\"error\":\"%s\"}\n",cudaGetErrorString(e)); return 1;}}while(0)

template<int SHAPE>
__global__ void dmma_loop(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b0 = a0 * 0.5, b1 = b0 + 2;
  double c[8][4];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (SHAPE == 0) {  // m16n8k4: A 2 dbl, B 1 dbl, C 4 dbl
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
            : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b0));
      } else {           // m8n8k4: A 1, B 1, C 2
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
            : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a0), "d"(b1));
      }
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double x[16]; double a = 1.0000001, b = threadIdx.x * 1e-9;
  for (int i = 0; i < 16; ++i) x[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0; for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 4, threads = 256;
  float ms;
  // warm
  dmma_loop<0><<<blocks, threads>>>(out, 1000); CK(cudaDeviceSynchronize());
  double res[3];
  for (int shape = 0; shape < 2; ++shape) {
    int iters = 20000;
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) { if (shape == 0) dmma_loop<0><<<blocks, threads>>>(out, iters); else dmma_loop<1><<<blocks, threads>>>(out, iters); }
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double fma_per_mma = shape == 0 ? 16 * 8 * 4 : 8 * 8 * 4;
    double flops = 5.0 * blocks * (threads / 32) * (double)iters * 8 * fma_per_mma * 2;
    res[shape] = flops / (ms * 1e-3) / 1e12;
  }
  {
    int iters = 20000;
    dfma_loop<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) dfma_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double flops = 5.0 * blocks * threads * (double)iters * 16 * 2;
    res[2] = flops / (ms * 1e-3) / 1e12;
  }
  printf("{\"dmma_m16n8k4_tflops\": %.3f, \"dmma_m8n8k4_tflops\": %.3f, \"dfma_tflops\": %.3f, \"sms\": %d, \"clock_khz\": %d}\n",
         res[0], res[1], res[2], p.multiProcessorCount, p.clockRate);
  return 0;
}
