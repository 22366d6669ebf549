// Harness-only: what bounds the fp32 engine's chunked 3xTF32 mainloop?
//   part 1: tcgen05.ld throughput per SM (32x32b.x32 loads, 4 / 8 / 16 warps, wait::ld per pair)
//   part 2: MMA issuer + drain warps with operands resident in SMEM (no TMA): a chunk of
//           KSC k-steps x 3 terms (hi*lo, lo*hi, hi*hi) into TMEM buffer c % NBUF, committed to
//           tmem_full; drain warps wait, optionally tcgen05.ld + FADD the chunk, arrive on
//           tmem_empty.  Reports cycles per MMA (raw floor: N/2 for M = 128).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/drain_rate tools/drain_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc64(uint32_t addr, uint32_t sbo) {   // K-major SWIZZLE_64B
  return ((uint64_t)(addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(sbo >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}"
                 : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
}
__device__ __forceinline__ uint32_t mbar_test(uint64_t* b, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}"
               : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
  return ok;
}
#define LD32(taddr, r)                                                                                     \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15," \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                   \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),      \
                 "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),  \
                 "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),            \
                 "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),            \
                 "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])             \
               : "r"(taddr) : "memory")

// ---------------- part 1: tcgen05.ld throughput
template <int W>
__global__ void ld_rate(int iters, float* out, long long* cyc) {
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tb + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * (512 / (W / 4));
  float s = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 512 / (W / 4) / 32; j += 2) {
      uint32_t v[32], w[32];
      LD32(tm + 32 * j, v);
      LD32(tm + 32 * (j + 1), w);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) s += __uint_as_float(v[i]) + __uint_as_float(w[i]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
  if (s == 1.2345f) out[0] = s;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

// ---------------- part 2: chunked MMA + drain pipeline
template <int N, int NBUF, int KSC, int DRAIN, int DW>
__global__ void pipe(int nchunks, float* out, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[NBUF], empty[NBUF];
  __shared__ uint32_t tb;
  constexpr int BK = 8 * KSC;                  // one "stage" holds exactly one chunk's k range
  constexpr uint32_t rowb = 64;                // SW64: rows of 16 tf32; KSC k-steps -> KSC/2 rows? (see below)
  // operand tiles: K-major SWIZZLE_64B, 16 k per 64-byte row, 8-row atoms (512 B); one 16-k
  // slab per tile (k-steps 0,1 inside the row); KSC > 2 reuses the same slab (values irrelevant)
  const uint32_t xh = sa(base), xl = xh + 128 * rowb, yh = xl + 128 * rowb, yl = yh + N * rowb;
  float* f = (float*)base;
  for (int i = threadIdx.x; i < (256 + 2 * N) * 16; i += blockDim.x) f[i] = 0.001f * (i & 7);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NBUF; ++b) { mbar_init(&full[b], 1); mbar_init(&empty[b], DW); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tb;
  constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  if (warp == 1) {
    long long t0 = clock64();
    uint32_t tm_ok = 1;
    for (int c = 0; c < nchunks; ++c) {
      const int b = c % NBUF, u = c / NBUF;
      if (u > 0 && !tm_ok) mbar_wait(&empty[b], (u - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (c + 1 < nchunks) {
        const int bn = (c + 1) % NBUF, un = (c + 1) / NBUF;
        tm_ok = un == 0 ? 1u : mbar_test(&empty[bn], (un - 1) & 1);
      }
      const uint32_t d = tm + b * N;
#pragma unroll
      for (int j = 0; j < KSC; ++j) {
        const uint32_t ko = 32 * (j & 1);
        const uint64_t dxh = desc64(xh + ko, 512), dxl = desc64(xl + ko, 512);
        const uint64_t dyh = desc64(yh + ko, 512), dyl = desc64(yl + ko, 512);
        asm volatile("{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
                     " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(dxh), "l"(dyl), "r"(idesc), "r"(j ? 1u : 0u));
        asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                     " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n}\n" ::"r"(d), "l"(dxl), "l"(dyh), "r"(idesc));
      }
#pragma unroll
      for (int j = 0; j < KSC; ++j) {
        const uint32_t ko = 32 * (j & 1);
        const uint64_t dxh = desc64(xh + ko, 512), dyh = desc64(yh + ko, 512);
        asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                     " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n}\n" ::"r"(d), "l"(dxh), "l"(dyh), "r"(idesc));
      }
      asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                   " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(sa(&full[b])) : "memory");
    }
    // wait for the last chunk's drain
    const int cl = nchunks - 1;
    mbar_wait(&empty[cl % NBUF], (cl / NBUF) & 1);
    long long t1 = clock64();
    if (lane == 0 && blockIdx.x == 0) *cyc = t1 - t0;
  } else if (warp >= 4 && warp < 4 + DW) {
    const int q = warp & 3, grp = (warp - 4) >> 2;
    constexpr int EC = N / (DW / 4);
    const uint32_t lo = (uint32_t)(q * 32) << 16;
    float acc[DRAIN ? EC : 1];
#pragma unroll
    for (int i = 0; i < (DRAIN ? EC : 1); ++i) acc[i] = 0.f;
    for (int c = 0; c < nchunks; ++c) {
      const int b = c % NBUF, u = c / NBUF;
      mbar_wait(&full[b], u & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (DRAIN) {
        const uint32_t ta = tm + lo + b * N + grp * EC;
#pragma unroll
        for (int j = 0; j < EC / 32; j += 2) {
          uint32_t v[32], w[32];
          LD32(ta + 32 * j, v);
          if (j + 1 < EC / 32) LD32(ta + 32 * (j + 1), w);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            acc[32 * j + i] += __uint_as_float(v[i]);
            if (j + 1 < EC / 32) acc[32 * (j + 1) + i] += __uint_as_float(w[i]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      if (lane == 0) mbar_arrive(&empty[b]);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < (DRAIN ? EC : 1); ++i) s += acc[i];
    if (s == 1.2345f) out[threadIdx.x] = s;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}


// ---------------- part 3: the same pipeline fed by a STAGES-deep ring of bulk copies from
// global memory (pre-swizzled 16-k tiles stored contiguously, d = 4096 planes: 4 x 64 MiB) into
// shared memory.  FEED 1: producer arrives without copying; 2: bulk copies, own B tile;
// 3: CTA pairs (cluster of 2 along M), each loading half of B and multicasting it.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(sa(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s_mc(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar, uint16_t mask) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], %4;"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(sa(bar)), "h"(mask) : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* m, uint64_t* bar, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(dst), "l"((uint64_t)m), "r"(sa(bar)), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void tma2d_mc(uint32_t dst, const CUtensorMap* m, uint64_t* bar, int x, int y, uint16_t mask) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;"
               ::"r"(dst), "l"((uint64_t)m), "r"(sa(bar)), "r"(x), "r"(y), "h"(mask) : "memory");
}
// FEED 4: 2D TMA boxes {16 k, rows} from row-major 4096 x 4096 planes (as the engine); 5: + pairs
template <int N, int NBUF, int STAGES, int FEED>
__global__ void pipe_fed(const uint8_t* __restrict__ gx, const uint8_t* __restrict__ gy, float* out, long long* cyc,
                         const __grid_constant__ CUtensorMap mxh, const __grid_constant__ CUtensorMap mxl,
                         const __grid_constant__ CUtensorMap myh, const __grid_constant__ CUtensorMap myl) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[NBUF], empty[NBUF], sfull[STAGES], sempty[STAGES];
  __shared__ uint32_t tb;
  constexpr int KSC = 2, KB = 256;                   // K = 4096 in 16-k blocks
  constexpr uint32_t ABYTES = 128 * 64, BBYTES = N * 64, STAGE = 2 * ABYTES + 2 * BBYTES;
  constexpr int CL = (FEED == 3 || FEED == 5) ? 2 : 1;
  uint32_t rank = 0;
  if (CL > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NBUF; ++b) { mbar_init(&full[b], 1); mbar_init(&empty[b], 8); }
    for (int s = 0; s < STAGES; ++s) { mbar_init(&sfull[s], 1); mbar_init(&sempty[s], CL); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&tb)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (CL > 1) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tb;
  const int tile_m = (blockIdx.x / CL) % 16 * CL + rank, tile_n = (blockIdx.x / CL) / 16;   // 32 x 16 tiles
  constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % STAGES, r = kb / STAGES;
        if (r > 0) mbar_wait(&sempty[s], (r - 1) & 1);
        const uint32_t st = sa(base) + s * STAGE;
        if (FEED == 1) { mbar_arrive(&sfull[s]); continue; }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&sfull[s])), "r"(STAGE) : "memory");
        // plane p of a 4096 x 4096 fp32 matrix, tile (row block of 128 | N, k block): contiguous
        const size_t pa = (size_t)64 << 20;
        const uint8_t* xa = gx + ((size_t)tile_m * KB + kb) * ABYTES;
        const uint8_t* yb = gy + ((size_t)tile_n * KB + kb) * BBYTES;
        if (FEED >= 4) {
          tma2d(st, &mxh, &sfull[s], kb * 16, tile_m * 128);
          tma2d(st + ABYTES, &mxl, &sfull[s], kb * 16, tile_m * 128);
          if (CL == 1) {
            tma2d(st + 2 * ABYTES, &myh, &sfull[s], kb * 16, tile_n * N);
            tma2d(st + 2 * ABYTES + BBYTES, &myl, &sfull[s], kb * 16, tile_n * N);
          } else {
            tma2d_mc(st + 2 * ABYTES + rank * (BBYTES / 2), &myh, &sfull[s], kb * 16, tile_n * N + rank * (N / 2), 3);
            tma2d_mc(st + 2 * ABYTES + BBYTES + rank * (BBYTES / 2), &myl, &sfull[s], kb * 16, tile_n * N + rank * (N / 2), 3);
          }
          continue;
        }
        bulk_g2s(st, xa, ABYTES, &sfull[s]);
        bulk_g2s(st + ABYTES, xa + pa, ABYTES, &sfull[s]);
        if (CL == 1) {
          bulk_g2s(st + 2 * ABYTES, yb, BBYTES, &sfull[s]);
          bulk_g2s(st + 2 * ABYTES + BBYTES, yb + pa, BBYTES, &sfull[s]);
        } else {
          const uint32_t hb = BBYTES / 2, o = rank * hb;
          bulk_g2s_mc(st + 2 * ABYTES + o, yb + o, hb, &sfull[s], 3);
          bulk_g2s_mc(st + 2 * ABYTES + BBYTES + o, yb + pa + o, hb, &sfull[s], 3);
        }
      }
    }
  } else if (warp == 1) {
    long long t0 = clock64();
    uint32_t tm_ok = 1;
    const int NCH = KB * (16 / (8 * KSC));
    for (int c = 0; c < NCH; ++c) {
      const int s = c % STAGES, r = c / STAGES;      // one chunk per stage (KSC = 2 = 16 k)
      const int b = c % NBUF, u = c / NBUF;
      mbar_wait(&sfull[s], r & 1);
      if (u > 0 && !tm_ok) mbar_wait(&empty[b], (u - 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (c + 1 < NCH) {
        const int bn = (c + 1) % NBUF, un = (c + 1) / NBUF;
        tm_ok = un == 0 ? 1u : mbar_test(&empty[bn], (un - 1) & 1);
      }
      const uint32_t st = sa(base) + s * STAGE, xh = st, xl = st + ABYTES, yh = st + 2 * ABYTES, yl = yh + BBYTES;
      const uint32_t d = tm + b * N;
#pragma unroll
      for (int j = 0; j < KSC; ++j) {
        const uint32_t ko = 32 * j;
        asm volatile("{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
                     " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(desc64(xh + ko, 512)), "l"(desc64(yl + ko, 512)), "r"(idesc), "r"(j ? 1u : 0u));
        asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                     " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n}\n" ::"r"(d), "l"(desc64(xl + ko, 512)), "l"(desc64(yh + ko, 512)), "r"(idesc));
      }
#pragma unroll
      for (int j = 0; j < KSC; ++j) {
        const uint32_t ko = 32 * j;
        asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                     " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n}\n" ::"r"(d), "l"(desc64(xh + ko, 512)), "l"(desc64(yh + ko, 512)), "r"(idesc));
      }
      asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                   " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(sa(&full[b])) : "memory");
      if (CL > 1)
        asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                     " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(sa(&sempty[s])), "h"((uint16_t)3) : "memory");
      else
        asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
                     " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(sa(&sempty[s])) : "memory");
    }
    const int cl = NCH - 1;
    mbar_wait(&empty[cl % NBUF], (cl / NBUF) & 1);
    long long t1 = clock64();
    if (lane == 0) atomicAdd((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
  } else if (warp >= 4 && warp < 12) {
    const int q = warp & 3, grp = (warp - 4) >> 2;
    constexpr int EC = N / 2;
    const uint32_t lo = (uint32_t)(q * 32) << 16;
    float acc[EC];
#pragma unroll
    for (int i = 0; i < EC; ++i) acc[i] = 0.f;
    const int NCH = KB * (16 / (8 * KSC));
    for (int c = 0; c < NCH; ++c) {
      const int b = c % NBUF, u = c / NBUF;
      mbar_wait(&full[b], u & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t ta = tm + lo + b * N + grp * EC;
#pragma unroll
      for (int j = 0; j < EC / 32; j += 2) {
        uint32_t v[32], w[32];
        LD32(ta + 32 * j, v);
        LD32(ta + 32 * (j + 1), w);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 32; ++i) { acc[32 * j + i] += __uint_as_float(v[i]); acc[32 * (j + 1) + i] += __uint_as_float(w[i]); }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      if (lane == 0) mbar_arrive(&empty[b]);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < EC; ++i) s += acc[i];
    if (s == 1.2345f) out[threadIdx.x] = s;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (CL > 1) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

static CUtensorMap make_map(const void* base, int rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  CUtensorMap m;
  cuuint64_t dims[2] = {4096, 4096};
  cuuint64_t strides[1] = {4096 * 4};
  cuuint32_t box[2] = {16, (cuuint32_t)rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("tensor map error %d\n", (int)r);
  return m;
}
template <int N, int NBUF, int STAGES, int FEED>
void run_fed(const uint8_t* gx, const uint8_t* gy, float* out, long long* cyc, int grid) {
  const size_t pl = (size_t)64 << 20;
  const int brows = (FEED == 5) ? N / 2 : N;
  CUtensorMap mxh = make_map(gx, 128), mxl = make_map(gx + pl, 128), myh = make_map(gy, brows), myl = make_map(gy + pl, brows);
  constexpr uint32_t STAGE = 2 * 128 * 64 + 2 * N * 64;
  const size_t smem = 1024 + STAGES * STAGE;
  auto k = pipe_fed<N, NBUF, STAGES, FEED>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(384);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (FEED == 3 || FEED == 5) ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, gx, gy, out, cyc, mxh, mxl, myh, myl);
  cudaDeviceSynchronize();
  cudaMemset(cyc, 0, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k, gx, gy, out, cyc, mxh, mxl, myh, myl);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double mmas = 256.0 * 6;
  printf("fed N=%d NBUF=%d STAGES=%d FEED=%d grid=%d: %.1f clk/MMA avg over CTAs (floor %d), kernel %.3f ms = %.0f TF/s tensor %s\n", N, NBUF,
         STAGES, FEED, grid, c / (double)grid / mmas, N / 2, ms, grid * 2.0 * 128 * N * 4096 * 3 / ms / 1e9,
         e ? cudaGetErrorString(e) : "");
}

template <int N, int NBUF, int KSC, int DRAIN, int DW>
void run_pipe(float* out, long long* cyc) {
  const int nchunks = 2048 / KSC;
  const size_t smem = 1024 + (256 + 2 * N) * 64;
  auto k = pipe<N, NBUF, KSC, DRAIN, DW>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<148, 128 + 32 * DW, smem>>>(nchunks, out, cyc);
  cudaDeviceSynchronize();
  k<<<148, 128 + 32 * DW, smem>>>(nchunks, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double mmas = (double)nchunks * KSC * 3;
  printf("pipe N=%d NBUF=%d KSC=%d drain=%d warps=%d: %.1f clk/MMA (floor %d), drained %.1f B/clk %s\n", N, NBUF, KSC,
         DRAIN, DW, c / mmas, N / 2, DRAIN ? (double)nchunks * 128 * N * 4 / c : 0.0, e ? cudaGetErrorString(e) : "");
}

template <int W>
void run_ld(float* out, long long* cyc) {
  const int iters = 200;
  ld_rate<W><<<148, 32 * W>>>(iters, out, cyc);
  cudaDeviceSynchronize();
  ld_rate<W><<<148, 32 * W>>>(iters, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("tcgen05.ld 32x32b.x32 pairs, %d warps: %.1f B/clk/SM (%lld clk for %d x 256 KiB) %s\n", W,
         (double)iters * 128 * 512 * 4 / c, c, iters, e ? cudaGetErrorString(e) : "");
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4096 * 4);
  cudaMalloc(&cyc, 8);
  uint8_t *gx, *gy;
  cudaMalloc(&gx, (size_t)128 << 20);
  cudaMalloc(&gy, (size_t)128 << 20);
  cudaMemset(gx, 0, (size_t)128 << 20);
  cudaMemset(gy, 0, (size_t)128 << 20);
  run_fed<256, 2, 4, 1>(gx, gy, out, cyc, 512);
  run_fed<256, 2, 4, 4>(gx, gy, out, cyc, 512);
  run_fed<256, 2, 4, 4>(gx, gy, out, cyc, 148);
  run_fed<256, 2, 4, 5>(gx, gy, out, cyc, 148);
  run_fed<256, 2, 4, 2>(gx, gy, out, cyc, 148);
  run_fed<256, 2, 4, 1>(gx, gy, out, cyc, 148);
  run_fed<256, 2, 4, 2>(gx, gy, out, cyc, 148);
  run_fed<256, 2, 4, 3>(gx, gy, out, cyc, 148);
  run_fed<256, 2, 3, 2>(gx, gy, out, cyc, 148);
  run_fed<256, 2, 4, 2>(gx, gy, out, cyc, 74);
  run_fed<256, 2, 4, 2>(gx, gy, out, cyc, 32);
  run_fed<128, 4, 6, 2>(gx, gy, out, cyc, 148);
  run_fed<128, 4, 6, 3>(gx, gy, out, cyc, 148);
  return 0;
}
