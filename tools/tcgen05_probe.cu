// Harness-only probe of tcgen05 basics on sm_100a: TMEM st/ld roundtrip and one tf32 MMA with
// all-ones operands (layout independent: D must equal K = 8 everywhere).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p){return (uint32_t)__cvta_generic_to_shared(p);}
__global__ void probe(float* out, int variant) {
  __shared__ __align__(1024) float A[128 * 32];
  __shared__ __align__(1024) float B[32 * 128];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * 32; i += blockDim.x) { A[i] = 1.f; B[i] = 1.f; }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"(sa(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = tbase;
  if (tid == 0) out[2000] = (float)tm;
  // 1. st/ld roundtrip on columns 128..131
  {
    uint32_t taddr = tm + ((uint32_t)(warp * 32) << 16) + 128;
    uint32_t v0 = __float_as_uint(tid * 10.f), v1 = __float_as_uint(tid * 10.f + 1), v2 = __float_as_uint(tid * 10.f + 2), v3 = __float_as_uint(tid * 10.f + 3);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" :: "r"(taddr), "r"(v0), "r"(v1), "r"(v2), "r"(v3));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    uint32_t r0, r1, r2, r3;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    out[tid * 4 + 0] = __uint_as_float(r0); out[tid * 4 + 1] = __uint_as_float(r1);
    out[tid * 4 + 2] = __uint_as_float(r2); out[tid * 4 + 3] = __uint_as_float(r3);
  }
  __syncthreads();
  // 2. one MMA M=128 N=128 K=8 (tf32), all-ones operands
  if (tid == 0) {
    uint64_t da = 0, db = 0;
    uint32_t aa = sa(A), bb = sa(B);
    auto mk = [](uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) -> uint64_t {
      return ((uint64_t)(addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
             ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
    };
    uint32_t bmaj = 0;
    switch (variant) {
      case 0: da = mk(aa, 16, 1024, 2); db = mk(bb, 4096, 1024, 2); bmaj = 1; break;
      case 1: da = mk(aa, 128, 256, 0); db = mk(bb, 128, 256, 0); bmaj = 0; break;
      case 2: da = mk(aa, 16, 1024, 2); db = mk(bb, 16, 1024, 2); bmaj = 0; break;
      case 3: da = mk(aa, 128, 256, 0); db = mk(bb, 128, 256, 0); bmaj = 1; break;
      case 4: da = mk(aa, 16, 1024, 2); db = mk(bb, 1024, 4096, 2); bmaj = 1; break;
      case 5: da = mk(aa, 16, 1024, 2); db = mk(bb, 128, 256, 0); bmaj = 0; break;
      case 6: da = mk(aa, 128, 256, 0); db = mk(bb, 4096, 1024, 2); bmaj = 1; break;
      case 7: da = mk(aa, 16, 1024, 2); db = mk(bb, 4096, 1024, 2); bmaj = 0; break;
    }
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (bmaj << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    uint32_t acc = 0;
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" :: "r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(acc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(sa(&bar)) : "memory");
  }
  // wait
  {
    uint32_t ok = 0;
    for (int it = 0; it < (1 << 24) && !ok; ++it)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(sa(&bar)) : "memory");
    if (tid == 0) out[2001] = ok;
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    uint32_t taddr = tm + ((uint32_t)(warp * 32) << 16);
    uint32_t r0, r1, r2, r3;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    out[512 + tid * 4 + 0] = __uint_as_float(r0); out[512 + tid * 4 + 1] = __uint_as_float(r1);
    out[512 + tid * 4 + 2] = __uint_as_float(r2); out[512 + tid * 4 + 3] = __uint_as_float(r3);
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(tm));
}
int main() {
  float* out; cudaMallocManaged(&out, 4096 * 4);
  for (int variant = 0; variant < 8; ++variant) {
    for (int i = 0; i < 4096; ++i) out[i] = -1;
    probe<<<1, 128>>>(out, variant);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s tmem=%g barrier_ok=%g\n", variant, cudaGetErrorString(e), out[2000], out[2001]);
    printf(" st/ld: t0 %g %g %g %g | t37 %g %g %g %g\n", out[0], out[1], out[2], out[3], out[148], out[149], out[150], out[151]);
    printf(" mma D: t0 %g %g %g %g | t77 %g %g %g %g\n", out[512], out[513], out[514], out[515], out[512 + 308], out[513 + 308], out[514 + 308], out[515 + 308]);
  }
  return 0;
}
