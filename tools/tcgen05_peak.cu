// Harness-only: sustained tcgen05.mma .kind::tf32 (and .kind::f16 bf16 for reference) rate on
// every SM: one CTA per SM, one thread issues M = 128, N = 256, K = 8 (tf32) / K = 16 (bf16)
// MMAs from SW128 K-major SMEM tiles back to back into 2 alternating TMEM accumulators, for
// a requested wall time (>= 4 s for the "sustained" figure).  Prints TFLOP/s per kind.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tcgen05_peak tools/tcgen05_peak.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t sbo) {
  return ((uint64_t)(addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(sbo >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);   // SWIZZLE_128B, version 1
}

template <int KIND>   // 0: tf32 (K = 8 per MMA), 1: bf16 (K = 16 per MMA)
__global__ void __launch_bounds__(128, 1) peak(long long iters, unsigned long long* cycles, int rnd) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tb;
  // operands: zeros (minimum switching power) or pseudo-random values in (-1, 1) (the power a
  // real GEMM draws; bf16 reads the same bytes as pairs of random bf16 values)
  for (int i = threadIdx.x; i < (128 + 256) * 32; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ (blockIdx.x * 40503u + 12345u);
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    reinterpret_cast<float*>(base)[i] = rnd ? ((float)(h >> 8) / 8388608.0f - 1.0f) : 0.f;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tb;
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    const uint32_t a0 = sa(base), b0 = a0 + 128 * 128;
    const uint32_t idesc = KIND == 0 ? ((1u << 4) | (2u << 7) | (2u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24))
                                     : ((1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24));
    for (long long it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {   // 4 k-steps of one 128-byte swizzle row
        const uint64_t da = desc(a0 + 32 * ks, 1024), db = desc(b0 + 32 * ks, 1024);
        const uint32_t acc = ks ? 1u : 0u, t = tm + (uint32_t)(it & 1) * 256;
        if (KIND == 0)
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(t),
                       "l"(da), "l"(db), "r"(idesc), "r"(acc));
        else
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(t),
                       "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0,1,0,p;\n}"
                   : "=r"(ok) : "r"(sa(&bar)) : "memory");
    if (blockIdx.x == 0) *cycles = (unsigned long long)(clock64() - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int KIND>
double run(double seconds, int sms, unsigned long long* dcyc, double* clk_per_mma, int rnd) {
  const size_t smem = 1024 + (128 + 256) * 128;
  cudaFuncSetAttribute(peak<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  long long iters = 1000;
  float ms = 0;
  for (;;) {   // calibrate the loop to the requested time
    cudaEventRecord(e0);
    peak<KIND><<<sms, 128, smem>>>(iters, dcyc, rnd);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms > 1000.0 * seconds * 0.9 || iters > (1ll << 40)) break;
    iters = (long long)(iters * (1000.0 * seconds / (ms > 1 ? ms : 1)) * 1.05) + 1000;
  }
  unsigned long long cyc = 0;
  cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
  const double kper = KIND == 0 ? 8 : 16;
  const double flops = 2.0 * 128 * 256 * kper * 4 * (double)iters * sms;
  *clk_per_mma = (double)cyc / (4.0 * iters);
  printf("%s %s operands: %.2f s, %.1f TFLOP/s, %.1f cycles per M128 N256 MMA, implied SM clock %.0f MHz (%s)\n",
         KIND == 0 ? "tf32 (K=8)" : "bf16 (K=16)", rnd ? "random" : "zero", ms / 1e3, flops / (ms * 1e-3) / 1e12,
         *clk_per_mma, (double)cyc / (ms * 1e-3) / 1e6, cudaGetErrorString(cudaGetLastError()));
  return flops / (ms * 1e-3) / 1e12;
}

int main(int argc, char** argv) {
  const double seconds = argc > 1 ? atof(argv[1]) : 4.0;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* dcyc;
  cudaMalloc(&dcyc, 8);
  double c0, c1, c2, c3;
  const double tf = run<0>(seconds, sms, dcyc, &c0, 0);
  const double bf = run<1>(seconds, sms, dcyc, &c1, 0);
  const double tfr = run<0>(seconds, sms, dcyc, &c2, 1);
  const double bfr = run<1>(seconds, sms, dcyc, &c3, 1);
  printf("{\"tf32_tflops\": %.2f, \"tf32_clk_per_mma_n256\": %.1f, \"bf16_tflops\": %.2f, \"bf16_clk_per_mma_n256\": %.1f, "
         "\"tf32_tflops_random\": %.2f, \"tf32_clk_per_mma_n256_random\": %.1f, \"bf16_tflops_random\": %.2f, "
         "\"bf16_clk_per_mma_n256_random\": %.1f, \"seconds_each\": %.1f, \"sms\": %d}\n",
         tf, c0, bf, c1, tfr, c2, bfr, c3, seconds, sms);
  return 0;
}
