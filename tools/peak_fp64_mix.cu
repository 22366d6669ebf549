// Microbenchmark (harness only): do DMMA (mma.sync f64) and DFMA share one FP64 pipe on sm_100a,
// and are the larger f64 mma shapes (m16n8k8, m16n8k16) any faster than m8n8k4?
// Warps 0-3 of each 8-warp block run a DMMA register loop, warps 4-7 a DFMA loop (each SMSP gets
// both kinds); mode bit 0 enables the DMMA warps, bit 1 the DFMA warps.  If the pipes were
// separate T(both) = max(T(dmma), T(dfma)); if shared, T(both) = T(dmma) + T(dfma).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("{\"error\":\"%s\"}\n",cudaGetErrorString(e)); return 1;}}while(0)

__global__ void mix_loop(double* out, int mode, int itersD, int itersF) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp < 4) {
    if (!(mode & 1)) return;
    double a0 = threadIdx.x * 1e-3, b1 = a0 * 0.5 + 2;
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
    for (int it = 0; it < itersD; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a0), "d"(b1));
    }
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else {
    if (!(mode & 2)) return;
    double x[16]; double a = 1.0000001, b = threadIdx.x * 1e-9;
    for (int i = 0; i < 16; ++i) x[i] = i;
    for (int it = 0; it < itersF; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
    }
    for (int i = 0; i < 16; ++i) s += x[i];
  }
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int SHAPE>
__global__ void shape_loop(double* out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = threadIdx.x * 5e-4 + i;
  double c[8][4];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (SHAPE == 8)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = p.multiProcessorCount * 4, threads = 256;
  const int itersD = 20000, itersF = 4 * itersD;   // equal FMA counts per warp
  float ms[4] = {0, 0, 0, 0};
  mix_loop<<<blocks, threads>>>(out, 3, 1000, 4000); CK(cudaDeviceSynchronize());
  for (int mode = 1; mode <= 3; ++mode) {
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) mix_loop<<<blocks, threads>>>(out, mode, itersD, itersF);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms[mode], e0, e1);
  }
  const double fl_half = 5.0 * blocks * 4 * (double)itersD * 8 * 256 * 2;   // FLOP of one warp kind
  float ms8, ms16;
  shape_loop<8><<<blocks, threads>>>(out, 100); CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) shape_loop<8><<<blocks, threads>>>(out, 10000);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms8, e0, e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) shape_loop<16><<<blocks, threads>>>(out, 5000);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms16, e0, e1);
  const double fl8 = 5.0 * blocks * 8 * 10000.0 * 8 * (16 * 8 * 8) * 2;
  const double fl16 = 5.0 * blocks * 8 * 5000.0 * 8 * (16 * 8 * 16) * 2;
  printf("{\"dmma_only_ms\": %.3f, \"dfma_only_ms\": %.3f, \"both_ms\": %.3f, \"dmma_only_tflops\": %.3f, "
         "\"dfma_only_tflops\": %.3f, \"both_tflops\": %.3f, \"dmma_m16n8k8_tflops\": %.3f, "
         "\"dmma_m16n8k16_tflops\": %.3f, \"sms\": %d}\n",
         ms[1], ms[2], ms[3], fl_half / (ms[1] * 1e-3) / 1e12, fl_half / (ms[2] * 1e-3) / 1e12,
         2 * fl_half / (ms[3] * 1e-3) / 1e12, fl8 / (ms8 * 1e-3) / 1e12, fl16 / (ms16 * 1e-3) / 1e12,
         p.multiProcessorCount);
  return 0;
}
