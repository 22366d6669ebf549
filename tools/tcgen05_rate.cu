// Harness-only: raw tcgen05.mma .kind::tf32 issue rate (SS operands, K-major SW128 tiles in
// SMEM, no TMA) for N = 64/128/192/256, M = 128, one CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p){return (uint32_t)__cvta_generic_to_shared(p);}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t layout, uint32_t sbo) {
  return ((uint64_t)(addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(sbo >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
template <int N, int SW, int PAT>
__global__ void rate(int iters, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2;
  __shared__ uint32_t tb;
  float* f = (float*)base;
  for (int i = threadIdx.x; i < 2 * (128 + N) * 32; i += blockDim.x) f[i] = 1.0f;
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000000;" :: "r"(sa(&bar2))); asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(sa(&tb))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = tb;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    // SW = 128: rows of 128 B (32 tf32, 4 k-steps), SW = 64: rows of 64 B (16 tf32, 2 k-steps)
    const uint32_t rowb = SW, atom = 8 * SW, layout = SW == 128 ? 2 : 4;
    const uint32_t a0 = sa(base), b0 = a0 + 128 * rowb, a1 = b0 + N * rowb, b1 = a1 + 128 * rowb;
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    const int KS = SW / 32;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        uint32_t acc = (it | ks) ? 1u : 0u;
        uint32_t tmb = tm;
        if (PAT >= 4) { tmb = tm + ((it & 3) * 128); acc = ks ? 1u : 0u; }
        if (PAT == 0) {
          uint64_t da = desc(a0 + 32 * ks, layout, atom), db = desc(b0 + 32 * ks, layout, atom);
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" :: "r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        } else {
          uint64_t ah = desc(a0 + 32 * ks, layout, atom), al = desc(a1 + 32 * ks, layout, atom);
          uint64_t bh = desc(b0 + 32 * ks, layout, atom), bl = desc(b1 + 32 * ks, layout, atom);
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" :: "r"(tmb), "l"(ah), "l"(bl), "r"(idesc), "r"(acc));
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" :: "r"(tmb), "l"(al), "l"(bh), "r"(idesc), "r"(1u));
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" :: "r"(tmb), "l"(ah), "l"(bh), "r"(idesc), "r"(1u));
          if (PAT == 2) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          if (PAT == 3) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(sa(&bar2)) : "memory");
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(sa(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(sa(&bar)) : "memory");
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (float)(t1 - t0) / (iters * (SW / 32) * (PAT ? 3 : 1));
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tm));
}
template <int N, int SW, int PAT> void run(float* out) {
  int smem = 2 * (128 + N) * 128 + 2048;
  cudaFuncSetAttribute(rate<N, SW, PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int iters = 20000;
  rate<N, SW, PAT><<<148, 128, smem>>>(100, out); cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); rate<N, SW, PAT><<<148, 128, smem>>>(iters, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 128 * N * 8 * (SW / 32) * (PAT ? 3.0 : 1.0) * iters * 148;
  printf("N=%d SW=%d pattern=%d: %.1f clk/instr (CTA0), %.1f TFLOP/s tf32 chip  err=%s\n", N, SW, PAT, out[0], flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

// PAT 5: STAGES-deep full/empty ring between a producer thread (warp 0) and the MMA thread
// (warp 1), 6 MMAs per stage (tf32 3-pass pattern, 2 k-steps), commit per stage -- no TMA.
template <int STAGES>
__global__ void ring(int iters, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[16], empty[16], done;
  __shared__ uint32_t tb;
  float* f = (float*)base;
  for (int i = threadIdx.x; i < 4 * 128 * 16; i += blockDim.x) f[i] = 1.0f;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&full[s]))); asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&empty[s]))); }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(sa(&tb))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = tb;
  auto wait = [](uint64_t* b, uint32_t ph) { uint32_t ok = 0; while (!ok) asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(sa(b)), "r"(ph) : "memory"); };
  long long t0 = clock64();
  const int n = iters;
  if (threadIdx.x == 0) {
    for (int kb = 0; kb < n; ++kb) { int s = kb % STAGES, r = kb / STAGES; if (r > 0) wait(&empty[s], (r - 1) & 1); asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(sa(&full[s]))); }
  } else if (threadIdx.x == 32) {
    const uint32_t a0 = sa(base), b0 = a0 + 8192, a1 = b0 + 8192, b1 = a1 + 8192;
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    for (int kb = 0; kb < n; ++kb) {
      int s = kb % STAGES, r = kb / STAGES; wait(&full[s], r & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t tmb = tm + (kb & 3) * 128;
      for (int ks = 0; ks < 2; ++ks) {
        uint64_t ah = desc(a0 + 32 * ks, 4, 512), al = desc(a1 + 32 * ks, 4, 512), bh = desc(b0 + 32 * ks, 4, 512), bl = desc(b1 + 32 * ks, 4, 512);
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" :: "r"(tmb), "l"(ah), "l"(bl), "r"(idesc), "r"((uint32_t)ks));
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" :: "r"(tmb), "l"(al), "l"(bh), "r"(idesc), "r"(1u));
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" :: "r"(tmb), "l"(ah), "l"(bh), "r"(idesc), "r"(1u));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(sa(&empty[s])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(sa(&done)) : "memory");
    wait(&done, 0);
    if (blockIdx.x == 0) out[0] = (float)(clock64() - t0) / (n * 6);
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tm));
}
template <int STAGES> void run_ring(float* out) {
  int smem = 4 * 8192 + 2048;
  cudaFuncSetAttribute(ring<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  ring<STAGES><<<148, 128, smem>>>(100, out); cudaDeviceSynchronize();
  ring<STAGES><<<148, 128, smem>>>(20000, out); cudaDeviceSynchronize();
  printf("ring STAGES=%d: %.1f clk/instr  err=%s\n", STAGES, out[0], cudaGetErrorString(cudaGetLastError()));
}
int main() { float* out; cudaMallocManaged(&out, 64);
  run<256, 64, 0>(out);   // back-to-back single MMAs
  run<256, 64, 1>(out);   // 3-pass pattern, no commits
  run<256, 64, 3>(out);   // 3-pass pattern, commit after every triple
  run<128, 64, 1>(out);
  run<128, 64, 3>(out);
  run_ring<2>(out); run_ring<4>(out); return 0; }
