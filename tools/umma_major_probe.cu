// Harness-only: which operand majorness does tcgen05.mma accept on this B200?  One M=128 MMA
// with all-ones operands (D must equal K everywhere for any in-bounds layout), for kind::tf32
// (K = 8) and kind::f16 with bf16 (K = 16), each operand K- or MN-major, SW128 or no swizzle.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
__device__ __forceinline__ uint32_t sa(const void* p){return (uint32_t)__cvta_generic_to_shared(p);}
struct V { int f16, amaj, bmaj, alay, blay, alo, aso, blo, bso, n; };
__global__ void probe(float* out, V v) {
  __shared__ __align__(1024) uint32_t A[128 * 32];   // 16 KB
  __shared__ __align__(1024) uint32_t B[32 * 128];   // 16 KB
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t one = v.f16 ? 0x3F803F80u : 0x3F800000u;   // two bf16 ones / one fp32 one
  for (int i = tid; i < 128 * 32; i += blockDim.x) { A[i] = one; B[i] = one; }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"(sa(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = tbase;
  if (tid == 0) {
    auto mk = [](uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) -> uint64_t {
      return ((uint64_t)(addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
             ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
    };
    uint64_t da = mk(sa(A), v.alo, v.aso, v.alay), db = mk(sa(B), v.blo, v.bso, v.blay);
    uint32_t fmt = v.f16 ? 1u : 2u;   // bf16 : tf32
    uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)v.amaj << 15) | ((uint32_t)v.bmaj << 16) |
                     (((uint32_t)v.n >> 3) << 17) | ((128u >> 4) << 24);
    if (v.f16)
      asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 0;\n" :: "r"(tm), "l"(da), "l"(db), "r"(idesc));
    else
      asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 0;\n" :: "r"(tm), "l"(da), "l"(db), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(sa(&bar)) : "memory");
  }
  uint32_t ok = 0;
  for (int it = 0; it < (1 << 24) && !ok; ++it)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(sa(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r0, r1, r2, r3;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(tm + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  out[tid * 4 + 0] = __uint_as_float(r0); out[tid * 4 + 3] = __uint_as_float(r3);
  asm volatile("tcgen05.fence::before_thread_sync;"); __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(tm));
}
int main() {
  float* out; cudaMallocManaged(&out, 4096 * 4);
  // f16 amaj bmaj alay blay alo aso blo bso n
  V vs[] = {
    {0, 0, 0, 2, 2, 16, 1024, 16, 1024, 128},     // tf32 K/K SW128 (known good)
    {0, 0, 1, 2, 2, 16, 1024, 4096, 1024, 128},   // tf32 B MN SW128
    {0, 0, 1, 2, 2, 16, 1024, 1024, 4096, 128},
    {0, 0, 1, 2, 2, 16, 1024, 1024, 1024, 32},    // tf32 B MN, one atom along N
    {0, 0, 1, 0, 0, 128, 256, 128, 256, 128},     // tf32 B MN no swizzle
    {0, 1, 0, 2, 2, 4096, 1024, 16, 1024, 128},   // tf32 A MN SW128
    {1, 0, 0, 2, 2, 16, 1024, 16, 1024, 128},     // bf16 K/K (known-good layout)
    {1, 0, 1, 2, 2, 16, 1024, 2048, 1024, 128},   // bf16 B MN SW128
    {1, 0, 1, 2, 2, 16, 1024, 1024, 2048, 128},
    {1, 0, 1, 0, 0, 128, 256, 128, 256, 128},     // bf16 B MN no swizzle
    {1, 1, 0, 2, 2, 2048, 1024, 16, 1024, 128},   // bf16 A MN SW128
  };
  for (auto& v : vs) {
    for (int i = 0; i < 4096; ++i) out[i] = -1;
    probe<<<1, 128>>>(out, v);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s amaj %d bmaj %d lay %d/%d lbo/sbo A %d/%d B %d/%d N %d: %s D[t0]=%g D[t77]=%g (expect %d)\n",
           v.f16 ? "bf16" : "tf32", v.amaj, v.bmaj, v.alay, v.blay, v.alo, v.aso, v.blo, v.bso, v.n,
           cudaGetErrorString(e), out[0], out[77 * 4], v.f16 ? 16 : 8);
    if (e != cudaSuccess) break;
  }
  return 0;
}
