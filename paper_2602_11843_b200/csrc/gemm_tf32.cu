// gemm_tf32.cu -- FP32 engine: 3xTF32 products on the 5th-generation tensor cores (sm_100a).
//
// acc = X * Y (d x d x d) with fp32 accuracy from three tcgen05.mma .kind::tf32 passes
//   acc = Xhi*Yhi + (Xhi*Ylo + Xlo*Yhi)        (hi = rn_tf32(x), lo = rn_tf32(x - hi), round to nearest even)
// Operands live in HBM as tf32 "planes" (hi and lo, fp32 containers, leading dimension ldp,
// a multiple of 32) written by the producing epilogue (or by the one-off split of the user's
// A), so the mainloop is pure TMA -> SMEM -> tcgen05 with no conversion work (DESIGN.md
// "FP32 engine").
//
// Tensor-core accumulation truncates toward zero (profiles/r01_tf32_accumulation_probe.txt),
// which biases long accumulations (~0.3 ulp of the accumulator per instruction).  The K loop
// is therefore split into chunks of CK k-blocks: each chunk accumulates in its own TMEM
// buffer -- the two small cross terms first (while the accumulator is still small), then
// hi*hi -- and the epilogue warps drain every chunk into fp32 register sums with IEEE adds
// while the tensor core fills the next of NBUF buffers.
//
// CTA: 128x128 output tile, BK = 32 (one 128-byte swizzle row of fp32), 3-stage TMA ring of
// {Xhi, Xlo, Yhi, Ylo} tiles (64 KB / stage).  Warp roles: w0 TMA producer, w1 MMA issuer,
// w2 TMEM allocator, w4..w7 epilogue (TMEM lane quarter = warp % 4).
// Both operands are K-major SWIZZLE_128B tiles (rows of 32 k-values, 8-row atoms, SBO = 1 KB,
// +32 B per k-step).  .kind::tf32 with an MN-major B operand from SMEM returned all zeros on
// this B200 (tools/tcgen05_probe.cu, profiles/r01_tcgen05_probe.txt), so the B role reads
// TRANSPOSED planes Y^T (row n holds column n of Y); producing epilogues write them.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <map>
#include <cstdlib>
#include <mutex>
#include <tuple>

#include "internal.h"

// A second translation unit (gemm_tf32_b128.cu) compiles this file again with another tile
// configuration: NSERIES_TF32_API renames its entry points, NSERIES_TF32_VARIANT drops the
// configuration-independent kernels (plane split, axpby) from it.
#ifndef NSERIES_TF32_API
#define NSERIES_TF32_API(name) name
#endif

namespace nseries {
namespace {

#ifndef NSERIES_TF32_XACC
#define NSERIES_TF32_XACC 0   // cross terms hi*lo + lo*hi in their own TMEM accumulator (below);
#endif                        // needs BN = 128: d = 4096 GEMM 0.717 -> 0.802 ms, d = 1024 0.054 -> 0.040
#ifndef NSERIES_TF32_BN
#if NSERIES_TF32_XACC
#define NSERIES_TF32_BN 128
#define NSERIES_TF32_BK 32
#define NSERIES_TF32_STAGES 3
#define NSERIES_TF32_KSC 4
#else
#define NSERIES_TF32_BN 256   // (BN = 192 -- 4.76 waves instead of 3.46 at d = 4096 -- measured
#define NSERIES_TF32_BK 16    //  11% slower: lower operand reuse per TMA byte)
#define NSERIES_TF32_STAGES 4
#endif
#endif
#ifndef NSERIES_TF32_CLUSTER
#define NSERIES_TF32_CLUSTER 2   // CTA pairs along M share (TMA-multicast) the B operand tile
#endif
#ifndef NSERIES_TF32_RU
#define NSERIES_TF32_RU 2   // rows per epilogue aux-load batch
#endif
constexpr int BM = 128, BN = NSERIES_TF32_BN, BK = NSERIES_TF32_BK, STAGES = NSERIES_TF32_STAGES;
constexpr int CL = NSERIES_TF32_CLUSTER;     // 1 or 2 CTAs per cluster
// (A 2-SM UMMA variant -- tcgen05.mma.cta_group::2, M = 256 from the leader CTA -- was correct
// but 1.8x slower: with the per-16-K drain the leader waits for both CTAs' drains every chunk.
// Removed in round 2.)
#ifndef NSERIES_TF32_PREFETCH
#define NSERIES_TF32_PREFETCH 0   // (8 measured 19% slower at d = 4096: extra L2 traffic)
#endif
constexpr int kPrefetchKB = NSERIES_TF32_PREFETCH;   // L2 prefetch distance (k-blocks) of the producer
#ifndef NSERIES_TF32_RASTER
#define NSERIES_TF32_RASTER 8   // pair rows per raster band (1: row-major tile order)
#endif
constexpr int kRasterGroup = NSERIES_TF32_RASTER;
// BK = 16 fp32 = 64-byte rows -> SWIZZLE_64B tiles (8-row atoms of 512 B).  Each 16-wide K
// chunk is one accumulation unit; NBUF = 4 chunk accumulators keep 4 chunks (24 MMAs) queued
// ahead of the drain round trip (commit -> epilogue tcgen05.ld -> arrive), which a 2-deep
// buffer (128x256 tiles) could not hide (tools/tf32_timing.cu).
#ifndef NSERIES_TF32_KSC
#define NSERIES_TF32_KSC 2
#endif
constexpr int KSC = NSERIES_TF32_KSC;        // k-steps (of 8) per accumulation chunk (Kc = 8 KSC)
constexpr int CPS = (BK / 8) / KSC;          // chunks per smem stage
// XACC: the cross terms (hi*lo + lo*hi, ~2^-11 of the product) accumulate over the whole K
// range in one TMEM accumulator -- their truncation bias is ~2^-11 of a full-K chain, far below
// fp32 rounding -- and only the hi*hi chunks (KSC MMAs each) go through the per-chunk drain.
// Same bias per chunk as KSC = 2 with all three terms, with half the drains per K.
constexpr bool XACC = NSERIES_TF32_XACC != 0;
constexpr int NBUF = XACC ? (512 - BN) / BN : 512 / BN;   // TMEM chunk accumulators of BN columns
#ifndef NSERIES_TF32_EPI_WARPS
#define NSERIES_TF32_EPI_WARPS 8   // (16: 11% slower -- the single MMA-issue thread competes with 20 warps)
#endif
constexpr int kEpiWarps = NSERIES_TF32_EPI_WARPS;   // 8: 2 per TMEM lane quarter; 16: 4 per quarter
constexpr int NG = kEpiWarps / 4;            // column groups of the tile (one per warp of a quarter)
constexpr int EC = BN / NG;                  // columns per epilogue thread
constexpr int kThreads = 128 + 32 * kEpiWarps;
constexpr int kFinalWarps = kThreads / 32;    // every warp runs the final epilogue passes
constexpr uint32_t kATileBytes = BM * BK * 4;   // 8 KB  (128 rows x 16 k)
constexpr uint32_t kBTileBytes = BN * BK * 4;   // 8 KB (128 rows of Y^T x 16 k)
constexpr uint32_t kStageBytes = 2 * kATileBytes + 2 * kBTileBytes;
constexpr uint32_t kTmemCols = (NBUF + (XACC ? 1 : 0)) * BN <= 256 ? 256 : 512;   // power of two >= used
constexpr uint32_t kSwizzleLayout = BK == 32 ? 2 : 4;   // UMMA layout: SWIZZLE_128B / _64B
constexpr uint32_t kAtomBytes = 8 * BK * 4;     // 8 rows x 64 B = 512 B (SBO)
constexpr int kStageLd = EC + 4;                // epilogue staging row (floats, 16-byte aligned)

struct Smem {
  alignas(1024) uint8_t xh[STAGES][kATileBytes];
  alignas(1024) uint8_t xl[STAGES][kATileBytes];
  alignas(1024) uint8_t yh[STAGES][kBTileBytes];
  alignas(1024) uint8_t yl[STAGES][kBTileBytes];
  uint8_t epi_extra[8192];   // the epilogue staging ((NG+1) x [128][EC+4] fp32) spills past the ring
  alignas(8) uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t tmem_full[NBUF];
  uint64_t tmem_empty[NBUF];
  uint32_t tmem_base;
  int sk_last;               // split-K: this CTA finishes the tile (1) or only leaves its partial (0)
};
static_assert((NG + 1) * BM * kStageLd * 4 <= STAGES * kStageBytes + 8192, "epilogue staging must fit the TMA ring + epi_extra");

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(saddr(b)));
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(saddr(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// non-blocking probe: issue early, consume the predicate later (hides the ~100-cycle
// barrier round trip behind MMA issue)
__device__ __forceinline__ uint32_t mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(saddr(b)), "r"(parity)
      : "memory");
  return ok;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  // bounded spin: a protocol bug traps instead of hanging the device
  for (uint32_t i = 0; !mbar_try_wait(b, parity); ++i)
    if (i > (1u << 26)) __trap();
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x,
                                            int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
          saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(saddr(bar)), "r"(x), "r"(y)
      : "memory");
}

// multicast variant: the box lands at the same shared offset in every CTA of ctaMask, and each
// destination's mbarrier (same offset) receives the complete_tx
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;\n" ::"r"(saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(saddr(bar)), "r"(x), "r"(y), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// SM100 shared-memory matrix descriptor (K-major, swizzled, version 1).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;          // version = 1 (Blackwell)
  d |= (uint64_t)kSwizzleLayout << 61;
  return d;
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = BN.
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (0u << 16) |
                            ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

// Warp-converged issue: every lane of the MMA warp runs the loop (so descriptors and TMEM
// addresses stay warp-uniform and live in uniform registers) and one elected lane issues.
__device__ __forceinline__ void mma_tf32_w(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p, e;\n setp.ne.b32 p, %4, 0;\n elect.sync _|e, 0xffffffff;\n"
      " @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit_w(uint64_t* bar) {
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
               " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(saddr(bar))
               : "memory");
}
__device__ __forceinline__ void mma_commit_mc_w(uint64_t* bar, uint16_t mask) {
  asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n"
               " @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
                   saddr(bar)), "h"(mask)
               : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}
// arrive on the mbarrier at the same offset in every CTA of ctaMask once the MMAs complete
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                   saddr(bar)), "h"(mask)
               : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   saddr(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// issue a 32-column TMEM load without waiting (pair with tmem_wait_ld before use)
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_ld16_async(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// packed fp32 add (SASS FADD2): acc[0:1] += (x, y), IEEE round-to-nearest
__device__ __forceinline__ void fadd2(float& a0, float& a1, float x, float y) {
  unsigned long long ua, ub;
  ua = ((unsigned long long)__float_as_uint(a1) << 32) | __float_as_uint(a0);
  ub = ((unsigned long long)__float_as_uint(y) << 32) | __float_as_uint(x);
  unsigned long long uc;
  asm("add.rn.f32x2 %0, %1, %2;\n" : "=l"(uc) : "l"(ua), "l"(ub));
  a0 = __uint_as_float((uint32_t)uc);
  a1 = __uint_as_float((uint32_t)(uc >> 32));
}

// tf32 round to nearest even: cvt.rn.tf32.f32 is ONE F2FP.TF32 instruction on sm_100a
// (cvt.rna is emulated by 4, the rna bit-pattern trick takes 2; tools/f2fp_split.cu)
__device__ __forceinline__ float rn_tf32(float x) {
  uint32_t r;
  asm("cvt.rn.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

#ifdef NSERIES_TF32_DEBUG
__device__ float* g_dbg = nullptr;
__device__ unsigned long long* g_tl = nullptr;   // per CTA: globaltimer at start / end, SM id
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

// Fused epilogue of one tile (after both accumulator halves are staged in shared memory).
// Inlined: an out-of-line version reads the __grid_constant__ parameters through generic loads
// (~10 K cycles per pass); the drain loop stays spill-free as long as the staging pointer is
// derived without an integer round trip through the shared-window address.
//
// Vectorised (round 2): a lane owns a quad of 4 consecutive columns, so one warp-wide access
// covers a whole staged row (EC = 128) or two (EC = 64): LDS.128 of the staged accumulator,
// coalesced LDG.128 of the aux rows and STG.128 of the x / hi / lo planes, with 16-byte aligned
// staging rows (kStageLd = EC + 4: row-wise and quad-per-row column reads are conflict-free).
// The transposed planes (and the symmetric mirror) are written by a column pass in which lane =
// row, reading its row's quad with one LDS.128 and storing 4 coalesced 128-byte columns.
// Misaligned or ragged quads (d % 4 != 0, tile edges) take a scalar path with the same formulas.
__device__ __forceinline__ float4 ld4g(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float q4(const float4& v, int e) { return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w; }
__device__ __forceinline__ float4 rn4(const float4& v) {
  return make_float4(rn_tf32(v.x), rn_tf32(v.y), rn_tf32(v.z), rn_tf32(v.w));
}
__device__ __forceinline__ float4 sub4(const float4& a, const float4& b) {
  return make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
}
// store the elements of quad t selected by mask (bit e: column c + e) at row pointer p + c
__device__ __forceinline__ void st_quad(float* p, int c, const float4& t, unsigned mask, bool vec) {
  if (vec && mask == 0xFu) {
    *reinterpret_cast<float4*>(p + c) = t;
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (mask & (1u << e)) p[c + e] = q4(t, e);
  }
}

template <int NO>   // number of outputs (compile-time: the per-element loops fully unroll)
__device__ __forceinline__ void tile_epilogue(const uint32_t tiles_off, const int m0, const int n0, const int d,
                                           const int ew, const int lane, const EpiParamsF32& ep,
                                           const int warp, const long long t_drained, const bool diag_pair) {
  // re-derive the staging pointer from the dynamic shared array so that accesses compile to
  // LDS / STS (a generic pointer passed in would not)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  float* const tiles = reinterpret_cast<float*>(smem_raw + tiles_off);
  float* const vt = tiles + NG * BM * kStageLd;   // output values of the current output
  constexpr int kQ = EC / 4;                      // column quads per staged row (32 or 16)
  constexpr int kRPI = 32 / kQ;                   // rows per warp-wide access (1 or 2)
  const int n_aux = ep.n_aux, ldp = ep.ldp;
  constexpr int n_out = NO;
  const float* auxb[kMaxAux];
  int auxld[kMaxAux];
  // vector path: every aux row and every row-major output row this epilogue touches starts on
  // a 16-byte boundary (hn0 is a multiple of 4; ldp is a multiple of 32)
  bool vec = (reinterpret_cast<uintptr_t>(ep.out_hi[0]) | reinterpret_cast<uintptr_t>(ep.out_lo[0])) % 16 == 0;
#pragma unroll
  for (int x = 0; x < kMaxAux; ++x) {
    auxb[x] = x < n_aux ? ep.aux[x] : nullptr;
    auxld[x] = x < n_aux ? ep.aux_ld[x] : 0;
    if (x < n_aux) vec = vec && (reinterpret_cast<uintptr_t>(auxb[x]) % 16 == 0) && (auxld[x] % 4 == 0);
  }
#pragma unroll
  for (int o = 0; o < kMaxOut; ++o)
    if (o < n_out)
      vec = vec && ((reinterpret_cast<uintptr_t>(ep.out_x[o]) | reinterpret_cast<uintptr_t>(ep.out_hi[o]) |
                     reinterpret_cast<uintptr_t>(ep.out_lo[o])) % 16 == 0) && (ep.out_ld[o] % 4 == 0);
#ifdef NSERIES_TF32_DEBUG
  __shared__ long long s_tp[8];
#define NSERIES_TP(i) do { if (warp == 4 && lane == 0) s_tp[i] = clock64(); } while (0)
#else
#define NSERIES_TP(i) do { } while (0)
#endif
  NSERIES_TP(0);
  const int qc = 4 * (lane % kQ);                 // this lane's quad: columns qc .. qc+3 of the half
  const int rsub = lane / kQ;                     // its row within a warp-wide access
  for (int hh = 0; hh < NG; ++hh) {
    const int hn0 = n0 + hh * EC;            // global column of this column group
    float* const tile = tiles + hh * BM * kStageLd;
    asm volatile("bar.sync 1, %0;\n" ::"n"(kThreads));
    NSERIES_TP(1 + 3 * hh);
    const int ncol = min(EC, d - hn0);       // valid columns of this half (> 0 for launched tiles)
    const int nrow = min(BM, d - m0);
    // valid columns of this lane's quad
    const unsigned cmask = qc + 4 <= ncol ? 0xFu : (qc < ncol ? (1u << (ncol - qc)) - 1u : 0u);
    // Pass 0 computes EVERY output from one read of the aux tiles (row-major x / hi / lo planes)
    // and stages the first output that needs transposed planes; each further transposed output
    // gets its own pass (staging only).  fp32 combination (binary64 epilogue arithmetic
    // measured no accuracy gain at config 3 and its F2F conversions were ~5x slower).
    for (int pass = 0, tnext = 0; pass < 1 + kMaxOut; ++pass) {
      int tout = -1;                         // output staged for the column pass in this pass
      for (int o = tnext; o < n_out; ++o)
        if (ep.sym || ep.out_hiT[o]) { tout = o; break; }
      if (pass > 0 && tout < 0) break;
      tnext = tout + 1;
      float al[kMaxOut], ga[kMaxOut], be[kMaxOut][kMaxAux];
      float *ox[kMaxOut], *oh[kMaxOut], *ol[kMaxOut];
      int old_[kMaxOut];
#pragma unroll
      for (int o = 0; o < kMaxOut; ++o) {
        const bool on = o < n_out && (pass == 0 || o == tout);
        al[o] = on ? (float)ep.alpha[o] : 0.f;
        ga[o] = on ? (float)ep.gamma[o] : 0.f;
#pragma unroll
        for (int x = 0; x < kMaxAux; ++x) be[o][x] = (on && x < n_aux) ? (float)ep.beta[o][x] : 0.f;
        ox[o] = (on && pass == 0) ? ep.out_x[o] : nullptr;
        oh[o] = (on && pass == 0) ? ep.out_hi[o] : nullptr;
        ol[o] = (on && pass == 0) ? ep.out_lo[o] : nullptr;
        old_[o] = o < n_out ? ep.out_ld[o] : 0;
      }
      // row pass: lanes along column quads; batches of RU warp-wide row accesses whose aux
      // loads are all issued before any use
      constexpr int RU = NSERIES_TF32_RU;
      constexpr int kStep = kFinalWarps * kRPI;   // rows advanced per warp per batch element
      for (int rb = ew * kRPI + rsub; rb < BM; rb += kStep * RU) {
        float4 av[RU][kMaxAux];
#pragma unroll
        for (int u = 0; u < RU; ++u) {
          const int rr = rb + u * kStep, r = m0 + rr;
          const bool ok = rr < nrow && cmask != 0u;
#pragma unroll
          for (int x = 0; x < kMaxAux; ++x) {
            av[u][x] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (x < n_aux && ok) {
              const float* ar = auxb[x] + (size_t)r * auxld[x] + hn0 + qc;
              if (vec && cmask == 0xFu) {
                av[u][x] = ld4g(ar);
              } else {
                float tmp[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int e = 0; e < 4; ++e)
                  if (cmask & (1u << e)) tmp[e] = __ldg(ar + e);
                av[u][x] = make_float4(tmp[0], tmp[1], tmp[2], tmp[3]);
              }
            }
          }
        }
#pragma unroll
        for (int u = 0; u < RU; ++u) {
          const int rr = rb + u * kStep, r = m0 + rr;
          if (rr >= nrow || cmask == 0u) continue;
          const int dq = r - hn0 - qc;             // quad element on the diagonal (if 0..3)
          // symmetric diagonal tiles: the upper part (column >= row) only
          unsigned smask = cmask;
          if (diag_pair) smask &= dq <= 0 ? 0xFu : (dq >= 4 ? 0u : (0xFu << dq) & 0xFu);
          const float4 a = *reinterpret_cast<const float4*>(tile + rr * kStageLd + qc);
#pragma unroll
          for (int o = 0; o < kMaxOut; ++o) {
            if (o >= n_out) break;
            float4 t = make_float4(al[o] * a.x, al[o] * a.y, al[o] * a.z, al[o] * a.w);
#pragma unroll
            for (int x = 0; x < kMaxAux; ++x) {   // be = 0 beyond n_aux
              t.x = fmaf(be[o][x], av[u][x].x, t.x);
              t.y = fmaf(be[o][x], av[u][x].y, t.y);
              t.z = fmaf(be[o][x], av[u][x].z, t.z);
              t.w = fmaf(be[o][x], av[u][x].w, t.w);
            }
            if (dq == 0) t.x += ga[o];
            if (dq == 1) t.y += ga[o];
            if (dq == 2) t.z += ga[o];
            if (dq == 3) t.w += ga[o];
            if (ox[o]) st_quad(ox[o] + (size_t)r * old_[o] + hn0, qc, t, smask, vec);
            if (oh[o]) {
              const float4 hi = rn4(t);
              st_quad(oh[o] + (size_t)r * ldp + hn0, qc, hi, smask, vec);
              st_quad(ol[o] + (size_t)r * ldp + hn0, qc, rn4(sub4(t, hi)), smask, vec);
            }
            if (o == tout) *reinterpret_cast<float4*>(vt + rr * kStageLd + qc) = t;
          }
        }
      }
      if (pass == 0) NSERIES_TP(2 + 3 * hh);
      if (tout >= 0) {
        asm volatile("bar.sync 1, %0;\n" ::"n"(kThreads));
        // column pass: lane = row of a 32-row group, one LDS.128 of its row's quad, then four
        // coalesced 128-byte columns -- of the transposed operand planes, or (symmetric mode)
        // the mirror image (c, r) of every element (r, c) (strictly upper part in diagonal
        // tiles) in the output's own x / hi / lo planes
        float* const tx = ep.sym ? ep.out_x[tout] : nullptr;
        float* const th = ep.sym ? ep.out_hi[tout] : ep.out_hiT[tout];
        float* const tl = ep.sym ? ep.out_lo[tout] : ep.out_loT[tout];
        const int tld = ep.sym ? ep.out_ld[tout] : ldp;   // ld of the x mirror (hi / lo: ldp)
        for (int item = ew; item < (BM / 32) * kQ; item += kFinalWarps) {
          const int rr = (item / kQ) * 32 + lane, c0 = 4 * (item % kQ);
          if (rr >= nrow || c0 >= ncol) continue;
          const int r = m0 + rr;
          const float4 v = *reinterpret_cast<const float4*>(vt + rr * kStageLd + c0);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int c = hn0 + c0 + e;
            if (c0 + e >= ncol) break;
            if (ep.sym && diag_pair && r >= c) continue;
            const float val = q4(v, e);
            if (tx) tx[(size_t)c * tld + r] = val;
            if (th) {
              const float hi = rn_tf32(val);
              th[(size_t)c * ldp + r] = hi;
              tl[(size_t)c * ldp + r] = rn_tf32(val - hi);
            }
          }
        }
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(kThreads));
      if (pass == 0) NSERIES_TP(3 + 3 * hh);
    }
  }
#ifdef NSERIES_TF32_DEBUG
  NSERIES_TP(7);
  if (warp == 4 && lane == 0 && g_dbg)
    for (int i = 1; i < 8; ++i)
      atomicAdd(reinterpret_cast<unsigned long long*>(g_dbg) + 7 + i, (unsigned long long)(s_tp[i] - s_tp[i - 1]));
#endif
#undef NSERIES_TP
}

__global__ void __launch_bounds__(kThreads, 1) __cluster_dims__(CL, 1, 1)
gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap mXh, const __grid_constant__ CUtensorMap mXl,
                   const __grid_constant__ CUtensorMap mYh, const __grid_constant__ CUtensorMap mYl,
                   int d, const __grid_constant__ EpiParamsF32 ep) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntn = (d + BN - 1) / BN;
  // cluster of CL CTAs: same n0, consecutive row tiles; each CTA TMA-loads 1/CL of the B tile
  // and multicasts it to the pair (a CTA whose rows fall past d still runs the protocol)
  const int rank = CL > 1 ? (int)cluster_ctarank() : 0;
  // split-K units of the last partial wave: unit u >= sk_first covers K range sp of pair tile
  // sk_first + (u - sk_first) / sk_split
  const int unit = blockIdx.x / CL;
  const bool split = ep.sk_split > 1 && unit >= ep.sk_first;
  const int pair = split ? ep.sk_first + (unit - ep.sk_first) / ep.sk_split : unit;
  const int sp = split ? (unit - ep.sk_first) % ep.sk_split : 0;
  int m0, n0;
  bool diag_pair = false;
  if (ep.sym) {
    // symmetric mode (CL * BM == BN): square CL*BM x BN pair tiles on/above the diagonal,
    // enumerated row after row
    int rem = pair, pr = 0;
    while (rem >= ntn - pr) { rem -= ntn - pr; ++pr; }
    const int tn = pr + rem;
    m0 = (pr * CL + rank) * BM;
    n0 = tn * BN;
    diag_pair = tn == pr;
  } else if (kRasterGroup > 1) {
    // grouped raster: bands of kRasterGroup pair rows, column-major inside a band, so the
    // concurrently resident tiles share their X and Y^T panels in L2
    const int npr = ((d + BM - 1) / BM + CL - 1) / CL;
    const int band = kRasterGroup * ntn;
    const int first = (pair / band) * kRasterGroup;
    const int gsz = min(npr - first, kRasterGroup);
    m0 = ((first + (pair % band) % gsz) * CL + rank) * BM;
    n0 = ((pair % band) / gsz) * BN;
  } else {
    m0 = ((pair / ntn) * CL + rank) * BM;
    n0 = (pair % ntn) * BN;
  }
  const int KBt = (d + BK - 1) / BK;
  const int kb0 = split ? KBt * sp / ep.sk_split : 0;
  const int KB = split ? KBt * (sp + 1) / ep.sk_split - kb0 : KBt;   // this unit's k-blocks
  const int NC = KB * CPS;                   // accumulation chunks
#ifdef NSERIES_TF32_DEBUG
  const long long t_kernel0 = clock64();
  unsigned long long* const dbgp = reinterpret_cast<unsigned long long*>(g_dbg);   // loaded once
  if (threadIdx.x == 0 && g_tl) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_tl[3 * blockIdx.x] = gtimer();
    g_tl[3 * blockIdx.x + 2] = smid;
  }
  long long t_drained = 0;
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&sm.full[s], 1); mbar_init(&sm.empty[s], CL); }
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&sm.tmem_full[b], 1);
      mbar_init(&sm.tmem_empty[b], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     saddr(&sm.tmem_base)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  fence_before();
  if (CL > 1) cluster_sync_all();   // the peer's barriers are initialised before any multicast
  else __syncthreads();
  fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % STAGES, r = kb / STAGES;
        NSERIES_SHAKE_POINT(1000 + kb);
        if (r > 0) mbar_wait(&sm.empty[s], (r - 1) & 1);
#ifdef NSERIES_TF32_NO_TMA
        mbar_arrive(&sm.full[s]);
#else
        mbar_expect_tx(&sm.full[s], kStageBytes);
        const int k0 = (kb0 + kb) * BK;
        tma_load_2d(sm.xh[s], &mXh, &sm.full[s], k0, m0);
        tma_load_2d(sm.xl[s], &mXl, &sm.full[s], k0, m0);
        if (kPrefetchKB > 0 && kb + kPrefetchKB < KB) {   // pull a later k-block into L2 (DRAM latency)
          const int kp = (kb0 + kb + kPrefetchKB) * BK;
          tma_prefetch_2d(&mXh, kp, m0);
          tma_prefetch_2d(&mXl, kp, m0);
          tma_prefetch_2d(&mYh, kp, n0 + rank * (BN / CL));
          tma_prefetch_2d(&mYl, kp, n0 + rank * (BN / CL));
        }
        if (CL > 1) {   // this CTA's slice of Y^T rows n0 .. n0+BN-1, multicast to the pair
          const int nb = rank * (BN / CL);
          tma_load_2d_mc(sm.yh[s] + rank * (kBTileBytes / CL), &mYh, &sm.full[s], k0, n0 + nb, (1u << CL) - 1);
          tma_load_2d_mc(sm.yl[s] + rank * (kBTileBytes / CL), &mYl, &sm.full[s], k0, n0 + nb, (1u << CL) - 1);
        } else {
          tma_load_2d(sm.yh[s], &mYh, &sm.full[s], k0, n0);   // Y^T rows n0..n0+BN-1
          tma_load_2d(sm.yl[s], &mYl, &sm.full[s], k0, n0);
        }
#endif
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: the whole warp runs the loop, one elected lane issues
    {
#ifdef NSERIES_TF32_DEBUG
      long long tstart = clock64();
      if (dbgp && lane == 0) atomicAdd(dbgp + 4, (unsigned long long)(tstart - t_kernel0));
#endif
      // The tensor pipe queues only a couple of MMAs, so a blocking barrier wait between two
      // chunks drains it (tools/tcgen05_rate.cu: 97 clk per N=128 MMA in a producer/consumer
      // ring vs 64 back to back).  The barriers of the NEXT chunk (stage full, TMEM buffer
      // empty) are therefore probed with a non-blocking test_wait right after this chunk's
      // barriers are satisfied and BEFORE its MMAs are issued; the probe results are consumed
      // one chunk later and a blocking wait happens only if a probe failed.
      uint32_t full_ok = mbar_test(&sm.full[0], 0);
      uint32_t tm_ok = 1;                        // chunk 0 uses a fresh buffer
#ifdef NSERIES_TF32_DEBUG
      long long dbg_wfull = 0, dbg_wempty = 0;   // local sums: one atomic per CTA at the end
#endif
      for (int c = 0; c < NC; ++c) {
        const int kb = c / CPS, h = c % CPS, s = kb % STAGES, r = kb / STAGES;
        const int b = c % NBUF, u = c / NBUF;     // accumulator b, use count u
        NSERIES_SHAKE_POINT(3000 + c);
        if (h == 0 && !full_ok) {
#ifdef NSERIES_TF32_DEBUG
          long long t1 = clock64();
#endif
          mbar_wait(&sm.full[s], r & 1);
#ifdef NSERIES_TF32_DEBUG
          dbg_wfull += clock64() - t1;
#endif
        }
        if (u > 0 && !tm_ok) {
#ifdef NSERIES_TF32_DEBUG
          long long t0 = clock64();
#endif
          mbar_wait(&sm.tmem_empty[b], (u - 1) & 1);
#ifdef NSERIES_TF32_DEBUG
          dbg_wempty += clock64() - t0;
#endif
        }
        fence_after();
        if (c + 1 < NC) {                         // probe the next chunk's barriers now
          const int cn = c + 1, kbn = cn / CPS, bn = cn % NBUF, un = cn / NBUF;
          full_ok = (cn % CPS) ? 1u : mbar_test(&sm.full[kbn % STAGES], (kbn / STAGES) & 1);
          tm_ok = un == 0 ? 1u : mbar_test(&sm.tmem_empty[bn], (un - 1) & 1);
        }
        const uint64_t dxh = smem_desc(saddr(sm.xh[s]), 16, kAtomBytes), dxl = smem_desc(saddr(sm.xl[s]), 16, kAtomBytes);
        const uint64_t dyh = smem_desc(saddr(sm.yh[s]), 16, kAtomBytes), dyl = smem_desc(saddr(sm.yl[s]), 16, kAtomBytes);
        const uint32_t t_acc = tmem + b * BN;
        // small cross terms first (accumulator still small), hi*hi last; K-major swizzled
        // tiles advance 32 B (8 tf32, +2 in the >>4 address field) per k-step
        if constexpr (XACC) {
          // hi*hi into this chunk's buffer, then the cross terms into the full-K accumulator
          const uint32_t t_x = tmem + NBUF * BN;
#pragma unroll
          for (int j = 0; j < KSC; ++j) {
            const int ks = h * KSC + j;
            mma_tf32_w(t_acc, dxh + 2 * ks, dyh + 2 * ks, j == 0 ? 0u : 1u);
          }
#pragma unroll
          for (int j = 0; j < KSC; ++j) {
            const int ks = h * KSC + j;
            mma_tf32_w(t_x, dxh + 2 * ks, dyl + 2 * ks, (c == 0 && j == 0) ? 0u : 1u);
            mma_tf32_w(t_x, dxl + 2 * ks, dyh + 2 * ks, 1u);
          }
          mma_commit_w(&sm.tmem_full[b]);          // chunk accumulator ready for the epilogue
          if (h == CPS - 1) {
            if (CL > 1) mma_commit_mc_w(&sm.empty[s], (1u << CL) - 1);
            else mma_commit_w(&sm.empty[s]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < KSC; ++j) {
            const int ks = h * KSC + j;
            mma_tf32_w(t_acc, dxh + 2 * ks, dyl + 2 * ks, j == 0 ? 0u : 1u);
            mma_tf32_w(t_acc, dxl + 2 * ks, dyh + 2 * ks, 1u);
          }
#pragma unroll
          for (int j = 0; j < KSC; ++j) {
            const int ks = h * KSC + j;
            mma_tf32_w(t_acc, dxh + 2 * ks, dyh + 2 * ks, 1u);
          }
          mma_commit_w(&sm.tmem_full[b]);          // chunk accumulator ready for the epilogue
          if (h == CPS - 1) {
            // frees the smem stage (in every CTA of the cluster: the pair multicasts into it)
            // once these MMAs finish
            if (CL > 1) mma_commit_mc_w(&sm.empty[s], (1u << CL) - 1);
            else mma_commit_w(&sm.empty[s]);
          }
        }
      }
#ifdef NSERIES_TF32_DEBUG
      if (dbgp && lane == 0) {
        atomicAdd(dbgp + 2, 1ull);
        atomicAdd(dbgp + 3, (unsigned long long)(clock64() - tstart));
        atomicAdd(dbgp + 0, (unsigned long long)dbg_wempty);
        atomicAdd(dbgp + 1, (unsigned long long)dbg_wfull);
      }
#endif
    }
  } else if (warp == 3) {
    // ---------------- idle warp: pull this tile's aux rows into L2 while the mainloop runs, so
    // the (latency-bound) epilogue reads hit L2
    const int ncols = min(BN, d - n0);
    for (int x = 0; x < ep.n_aux; ++x) {
      const float* base = ep.aux[x];
      const size_t ld = (size_t)ep.aux_ld[x];
      if (((reinterpret_cast<uintptr_t>(base) | (ld * 4) | (size_t)(n0 * 4)) & 15) != 0) continue;
      for (int rr = lane; rr < BM && m0 + rr < d; rr += 32) {
        const float* row = base + (size_t)(m0 + rr) * ld + n0;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(row), "r"((ncols * 4) & ~15) : "memory");
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: drain chunks into fp32 registers, then the fused outputs
    const int q = warp & 3;                    // TMEM lane quarter (hardware: warp % 4)
    const int half = (warp - 4) >> 2;          // this warp's column group of the tile
    const int cb = half * EC;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    float acc[EC];
#pragma unroll
    for (int i = 0; i < EC; ++i) acc[i] = 0.f;
    for (int c = 0; c < NC; ++c) {
      const int b = c % NBUF, u = c / NBUF;
      NSERIES_SHAKE_POINT(5000 + c);
      mbar_wait(&sm.tmem_full[b], u & 1);
      fence_after();
      const uint32_t t_acc = tmem + lane_off + b * BN + cb;
#ifndef NSERIES_TF32_NO_DRAIN
#if NSERIES_TF32_BN == 256 && NSERIES_TF32_EPI_WARPS == 8
#pragma unroll
      for (int j = 0; j < EC / 32; j += 2) {   // two 32-column loads in flight
        uint32_t v[32], w[32];
        tmem_ld32_async(t_acc + 32 * j, v);
        tmem_ld32_async(t_acc + 32 * (j + 1), w);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          fadd2(acc[32 * j + i], acc[32 * j + i + 1], __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
          fadd2(acc[32 * (j + 1) + i], acc[32 * (j + 1) + i + 1], __uint_as_float(w[i]), __uint_as_float(w[i + 1]));
        }
      }
#else
#pragma unroll
      for (int j = 0; j < EC / 32; ++j) {      // one 32-column group (two x16 loads) in flight
        uint32_t v[16], w[16];
        tmem_ld16_async(t_acc + 32 * j, v);
        tmem_ld16_async(t_acc + 32 * j + 16, w);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          fadd2(acc[32 * j + i], acc[32 * j + i + 1], __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
          fadd2(acc[32 * j + 16 + i], acc[32 * j + 16 + i + 1], __uint_as_float(w[i]), __uint_as_float(w[i + 1]));
        }
      }
#endif
#endif
      fence_before();
      NSERIES_SHAKE_POINT(7000 + c);
      if (lane == 0) {
        mbar_arrive(&sm.tmem_empty[b]);
      }
    }
    if constexpr (XACC) {
      // the last chunk's commit covered every MMA: the cross accumulator is complete
      const uint32_t t_x = tmem + lane_off + NBUF * BN + cb;
#pragma unroll
      for (int j = 0; j < EC / 32; ++j) {
        uint32_t v[16], w[16];
        tmem_ld16_async(t_x + 32 * j, v);
        tmem_ld16_async(t_x + 32 * j + 16, w);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          fadd2(acc[32 * j + i], acc[32 * j + i + 1], __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
          fadd2(acc[32 * j + 16 + i], acc[32 * j + 16 + i + 1], __uint_as_float(w[i]), __uint_as_float(w[i + 1]));
        }
      }
    }
#ifdef NSERIES_TF32_DEBUG
    t_drained = clock64();
#endif
    // ---- fused epilogue, staged through shared memory one column half at a time (the TMA
    // ring is idle: every MMA has completed and every stage was consumed).  Staging tiles
    // [128][EC+1] (acc, then the output value); the +1 pad keeps row- and column-wise
    // accesses conflict-free.  All per-output parameters are hoisted into registers (the
    // pass is instruction-bound), tf32 splits are one F2FP each (cvt.rn).
    // both column halves are staged at once (the accumulator registers die here); the
    // current output's values go to a third staging tile for the transposed column pass
    float* const tiles = reinterpret_cast<float*>(smem_raw + (reinterpret_cast<uint8_t*>(&sm.xh[0][0]) - smem_raw));
    const int rl = q * 32 + lane;
#pragma unroll
    for (int i = 0; i < EC; i += 4)   // STS.128: 8-lane phases hit 8 distinct bank quads (pitch EC + 4)
      *reinterpret_cast<float4*>(tiles + (half * BM + rl) * kStageLd + i) = make_float4(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]);
    if (split) {
      // split-K (2 K ranges): the first CTA of the tile to finish leaves its partial, the
      // second adds it (p_0 + p_1 is exact-commutative, so the result does not depend on who
      // finishes first).  Partials are stored as [tile][BN/4][BM][4] floats: a warp's float4
      // accesses are contiguous.  Works on the staged values (accumulator registers are dead).
      const int tile = (pair - ep.sk_first) * CL + rank;
      unsigned* cnt = ep.sk_cnt + 2 * tile;
      float4* const pt = reinterpret_cast<float4*>(ep.sk_part + (size_t)tile * (BN * BM)) + (size_t)(cb / 4) * BM + rl;
      float* const st = tiles + (half * BM + rl) * kStageLd;
      NSERIES_SHAKE_POINT(9000);
      if (warp == 4 && lane == 0) sm.sk_last = atomicAdd(cnt, 1u) == 1u;
      asm volatile("bar.sync 2, %0;\n" ::"n"(32 * kEpiWarps) : "memory");
      if (!sm.sk_last) {
#pragma unroll
        for (int i = 0; i < EC; i += 4) __stcg(pt + (size_t)(i / 4) * BM, make_float4(st[i], st[i + 1], st[i + 2], st[i + 3]));
        __threadfence();
        NSERIES_SHAKE_POINT(9001);
        asm volatile("bar.sync 2, %0;\n" ::"n"(32 * kEpiWarps) : "memory");
        if (warp == 4 && lane == 0) atomicAdd(cnt + 1, 1u);
      } else {
        if (warp == 4 && lane == 0) {
          unsigned v;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(cnt + 1) : "memory");
          } while (v != 1u);
          cnt[0] = 0u;     // the other unit of this tile is done with the counters
          cnt[1] = 0u;
        }
        asm volatile("bar.sync 2, %0;\n" ::"n"(32 * kEpiWarps) : "memory");
#pragma unroll
        for (int i0 = 0; i0 < EC; i0 += 64) {          // 16 independent float4 loads in flight
          float4 v[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) v[u] = __ldcg(pt + (size_t)((i0 + 4 * u) / 4) * BM);
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int i = i0 + 4 * u;
            st[i] += v[u].x;
            st[i + 1] += v[u].y;
            st[i + 2] += v[u].z;
            st[i + 3] += v[u].w;
          }
        }
      }
    }
  }
  {
    // ---- final epilogue passes on ALL warps (the producer / MMA / allocator / prefetch warps
    // are idle by now); the first barrier inside orders the staging above
#ifdef NSERIES_TF32_DEBUG
    const long long td = t_drained;
#else
    const long long td = 0;
#endif
    const uint32_t tiles_off = (uint32_t)(reinterpret_cast<uint8_t*>(&sm.xh[0][0]) - smem_raw);
    const int ew = warp >= 4 ? warp - 4 : warp + kEpiWarps;   // 0 .. kFinalWarps-1
    if (split) __syncthreads();      // sm.sk_last is visible to every warp
    if (split && !sm.sk_last) {
      // partial written: nothing more for this CTA
    } else if (ep.n_out == 1) tile_epilogue<1>(tiles_off, m0, n0, d, ew, lane, ep, warp, td, diag_pair);
    else if (ep.n_out == 2) tile_epilogue<2>(tiles_off, m0, n0, d, ew, lane, ep, warp, td, diag_pair);
    else tile_epilogue<3>(tiles_off, m0, n0, d, ew, lane, ep, warp, td, diag_pair);
  }
#ifdef NSERIES_TF32_DEBUG
  if (warp == 4 && lane == 0 && dbgp) {
    atomicAdd(dbgp + 5, (unsigned long long)(clock64() - t_drained));
    atomicAdd(dbgp + 6, (unsigned long long)(t_drained - t_kernel0));
  }
#endif
  fence_before();
  if (CL > 1) cluster_sync_all();   // no CTA leaves while its pair may still signal its barriers
  else __syncthreads();
  if (warp == 2) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTmemCols));
#ifdef NSERIES_TF32_DEBUG
    if (lane == 0 && g_tl) g_tl[3 * blockIdx.x + 1] = gtimer();
#endif
  }
}

#ifndef NSERIES_TF32_VARIANT
// split x (ld_in) into tf32 planes hi/lo and/or transposed planes hiT/loT (ld_out);
// identity != 0 splits I instead of x.  32x32 tiles through shared memory keep both the
// row-major and the transposed writes coalesced.
__global__ void split_planes_kernel(const float* __restrict__ x, int ld_in, float* __restrict__ hi,
                                    float* __restrict__ lo, float* __restrict__ hiT,
                                    float* __restrict__ loT, int ld_out, int d, int identity) {
  __shared__ float th[32][33], tl[32][33];
  const int tiles = (d + 31) / 32;
  for (int t = blockIdx.x; t < tiles * tiles; t += gridDim.x) {
    const int r0 = (t / tiles) * 32, c0 = (t % tiles) * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
      const int r = r0 + i, c = c0 + threadIdx.x;
      float h = 0.f, l = 0.f;
      if (r < d && c < d) {
        const float v = identity ? (r == c ? 1.f : 0.f) : x[(size_t)r * ld_in + c];
        h = rn_tf32(v);
        l = rn_tf32(v - h);
        if (hi) { hi[(size_t)r * ld_out + c] = h; lo[(size_t)r * ld_out + c] = l; }
      }
      th[i][threadIdx.x] = h;
      tl[i][threadIdx.x] = l;
    }
    __syncthreads();
    if (hiT) {
      for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, r = r0 + threadIdx.x;   // write row c of the transpose
        if (r < d && c < d) {
          hiT[(size_t)c * ld_out + r] = th[threadIdx.x][i];
          loT[(size_t)c * ld_out + r] = tl[threadIdx.x][i];
        }
      }
    }
    __syncthreads();
  }
}

__global__ void axpby_f32_kernel(int d, const __grid_constant__ EpiParamsF32 ep) {
  const size_t n = (size_t)d * d;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / d), c = (int)(i % d);
    for (int o = 0; o < ep.n_out; ++o) {
      double t = 0.0;
      for (int x = 0; x < ep.n_aux; ++x) t = fma(ep.beta[o][x], (double)ep.aux[x][(size_t)r * ep.aux_ld[x] + c], t);
      if (r == c) t += ep.gamma[o];
      const float v = (float)t;
      const float h = rn_tf32(v), l = rn_tf32(v - h);
      if (ep.out_x[o]) ep.out_x[o][(size_t)r * ep.out_ld[o] + c] = v;
      if (ep.out_hi[o]) { ep.out_hi[o][(size_t)r * ep.ldp + c] = h; ep.out_lo[o][(size_t)r * ep.ldp + c] = l; }
      if (ep.out_hiT[o]) { ep.out_hiT[o][(size_t)c * ep.ldp + r] = h; ep.out_loT[o][(size_t)c * ep.ldp + r] = l; }
    }
  }
}

#endif  // NSERIES_TF32_VARIANT

// ---------------------------------------------------------------- host: tensor maps
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// role 0: A operand box {BK k, BM rows}; role 1: B operand (transposed planes) box {BK k, BN rows}
int make_map(CUtensorMap* m, const float* base, int d, int ld, int role) {
  auto enc = get_encode();
  if (!enc) return (int)cudaErrorNotSupported;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)d};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)BK, role == 0 ? (cuuint32_t)BM : (cuuint32_t)(BN / CL)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, BK == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

struct MapCache {
  std::mutex mu;
  std::map<std::tuple<const void*, int, int, int>, CUtensorMap> maps;
  int get(const float* p, int d, int ld, int role, CUtensorMap* out) {
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple((const void*)p, d, ld, role);
    auto it = maps.find(key);
    if (it == maps.end()) {
      CUtensorMap m;
      int rc = make_map(&m, p, d, ld, role);
      if (rc) return rc;
      it = maps.emplace(key, m).first;
    }
    *out = it->second;
    return 0;
  }
};
MapCache g_maps;

// concurrently resident clusters of the GEMM kernel (one wave)
int wave_clusters() {
  static int w = -1;
  if (w < 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(148 * CL);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = sizeof(Smem) + 1024;
    smem_attr_once<gemm_tf32x3_kernel>((int)cfg.dynamicSmemBytes);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, gemm_tf32x3_kernel, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 0;
    }
    w = n;
  }
  return w;
}

// split-K of the tail: with T pair tiles and W resident clusters the last wave holds
// t = T mod W tiles; each is split into S = min(W / t, kMaxSplit) K ranges when S >= 2
constexpr int kMaxSplit = 2;            // the combine relies on p_0 + p_1 = p_1 + p_0
constexpr int kSplitMinKB = 16;            // keep at least 16 k-blocks (K = 256) per unit
void splitk_plan(int d, bool sym, int* first, int* S) {
  *first = 0;
  *S = 1;
  static const bool off = std::getenv("NSERIES_TF32_SPLITK") && std::atoi(std::getenv("NSERIES_TF32_SPLITK")) == 0;
  if (sym || off) return;
  const int ntn = (d + BN - 1) / BN;
  const int T = ((d + BM - 1) / BM + CL - 1) / CL * ntn;
  const int W = wave_clusters();
  if (W <= 0) return;
  const int t = T % W;                     // T < W: a single partial wave, split all of it
  if (t == 0) return;
  int s = std::min(W / t, kMaxSplit);
  while (s > 1 && (d + BK - 1) / BK / s < kSplitMinKB) --s;
  if (s < 2 || (size_t)t * CL * 2 * sizeof(unsigned) > 8192) return;
  *first = T - t;
  *S = s;
}

// split-K workspace layout: [counters: 2 x unsigned per CTA tile, fixed 8 KiB area][partials].
// The counter area is at the same place for every d (the partials of one size must never land
// on counters another size expects to be zero); split tiles < one wave <= 1024 CTA tiles.
constexpr size_t kSplitCntBytes = 8192;
size_t splitk_cnt_bytes(size_t) { return kSplitCntBytes; }

}  // namespace

size_t NSERIES_TF32_API(tf32_splitk_ws_bytes)(int d) {
  int first, S;
  splitk_plan(d, false, &first, &S);
  if (S < 2) return 0;
  const int ntn = (d + BN - 1) / BN;
  const int T = ((d + BM - 1) / BM + CL - 1) / CL * ntn;
  const size_t tiles = (size_t)(T - first) * CL;
  return splitk_cnt_bytes(tiles) + tiles * (size_t)(BN * BM) * sizeof(float);
}

int NSERIES_TF32_API(launch_gemm_tf32x3)(const float* Xh, const float* Xl, const float* Yh, const float* Yl, int d,
                                         int ldp, const EpiParamsF32& ep_in, void* stream, void* sk_ws) {
  EpiParamsF32 ep = ep_in;
  ep.sk_first = 0;
  ep.sk_split = 1;
  ep.sk_part = nullptr;
  ep.sk_cnt = nullptr;
  if (sk_ws && !ep.sym) {
    int first, S;
    splitk_plan(d, false, &first, &S);
    if (S > 1) {
      const int ntn = (d + BN - 1) / BN;
      const int T = ((d + BM - 1) / BM + CL - 1) / CL * ntn;
      const size_t tiles = (size_t)(T - first) * CL;
      ep.sk_first = first;
      ep.sk_split = S;
      ep.sk_cnt = static_cast<unsigned*>(sk_ws);
      const size_t off = splitk_cnt_bytes(tiles);
      ep.sk_part = reinterpret_cast<float*>(static_cast<char*>(sk_ws) + off);
    }
  }
  CUtensorMap mxh, mxl, myh, myl;
  int rc = g_maps.get(Xh, d, ldp, 0, &mxh);
  if (!rc) rc = g_maps.get(Xl, d, ldp, 0, &mxl);
  if (!rc) rc = g_maps.get(Yh, d, ldp, 1, &myh);   // transposed planes, K-major box of BN rows
  if (!rc) rc = g_maps.get(Yl, d, ldp, 1, &myl);
  if (rc) return rc;
  const size_t smem = sizeof(Smem) + 1024;
  if (int e = smem_attr_once<gemm_tf32x3_kernel>((int)smem)) return e;
  const int row_groups = ((d + BM - 1) / BM + CL - 1) / CL;   // clusters of CL row tiles
  const int ntn = (d + BN - 1) / BN;
  if (ep.sym && CL * BM != BN) return (int)cudaErrorInvalidValue;   // square pair tiles needed
  int ctas = ep.sym ? ntn * (ntn + 1) / 2 * CL : row_groups * ntn * CL;
  if (ep.sk_split > 1) ctas += (row_groups * ntn - ep.sk_first) * (ep.sk_split - 1) * CL;
  gemm_tf32x3_kernel<<<ctas, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(mxh, mxl, myh, myl, d, ep);
  return (int)cudaGetLastError();
}

#ifndef NSERIES_TF32_VARIANT
int launch_split_f32(const float* x, int ld_in, float* hi, float* lo, float* hiT, float* loT, int ld_out,
                     int d, bool identity, void* stream) {
  const int tiles = (d + 31) / 32;
  const int blocks = std::min(tiles * tiles, 148 * 8);
  split_planes_kernel<<<blocks, dim3(32, 8), 0, static_cast<cudaStream_t>(stream)>>>(
      x, ld_in, hi, lo, hiT, loT, ld_out, d, identity ? 1 : 0);
  return (int)cudaGetLastError();
}

int launch_axpby_f32(int d, const EpiParamsF32& ep, void* stream) {
  const size_t n = (size_t)d * d;
  int blocks = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
  axpby_f32_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(d, ep);
  return (int)cudaGetLastError();
}

#endif  // NSERIES_TF32_VARIANT

}  // namespace nseries
