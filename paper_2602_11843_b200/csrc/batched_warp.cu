// batched_warp.cu -- batched small-matrix path, fp32, d <= 32: a WARP GROUP PER MATRIX
// (config 4: 16384 independent 32 x 32 matrices).
//
// A persistent grid of warp groups (WPM = 1, 2 or 4 warps per matrix) walks the batch.  Each
// group owns (n_slots + 2) shared-memory slots of 32 x 32 fp32 (4 KiB, XOR-swizzled, no
// padding) and runs the whole compiled op list of the plan (mu_m + 2 products per radix-m
// update, the same fused epilogues as the large path) on its own matrix with only group-local
// barriers (__syncwarp / a named 32*WPM-thread barrier) between ops:
//
//   * the product X * Y (32 x 32 x 32) is computed ENTIRELY in registers: 2 x 4 mma.sync
//     m16n8k8 tf32 tiles (warp w of the group owns column tiles [w*4/WPM, (w+1)*4/WPM)),
//     3xTF32 split at fragment load (see split_tf32), hi*hi and the two
//     cross terms in separate accumulator chains (tensor-core accumulation truncates,
//     profiles/r01_tf32_accumulation_probe.txt);
//   * the epilogue out_j = alpha_j acc + sum_i beta_ji aux_i + gamma_j I runs on the
//     accumulator registers; because every operand has been read before any output is
//     written, outputs may overwrite values that die at this op (assign_slots_inplace),
//     which keeps the radix-9 live set at 5 slots;
//   * I as a GEMM operand (the paper's S_1 * T concatenation, PAPER.md:693-709 counting) is
//     synthesised in the fragment registers -- the product is executed, no slot is spent;
//   * the final S goes straight from the accumulators to global memory;
//   * A_{b+1} is prefetched with cp.async into the second A buffer while A_b is processed.
//
// K-permutation: a k-step of the MMA sums over its 8 k indices in any order, so lane (g,t) is
// given k = 8s+2t (fragment slot t) and 8s+2t+1 (slot t+4) in k-step s.  The A fragment of a
// row is then one 8-byte load -- the same access shape as the accumulator layout the epilogue
// reads and writes -- and the B fragment two 4-byte column loads.  Layout of a slot: 32 rows of
// four 8-float segments, segment' = segment ^ h(r) with h(r) = ((r ^ r>>2) & 1) | (r & 2); it
// makes the 8-byte row accesses (A fragments, epilogue) and the column loads (B fragments)
// bank-conflict free.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "internal.h"

namespace nseries {

namespace {

constexpr int kSlotF = 1024;   // floats per 32 x 32 slot

#if defined(NSERIES_BW_QSWZ)
// (SIMT control experiment) 4-float quads XOR-swizzled by row (r & 7): a warp's row-quad loads
// of 8 rows hit 32 distinct banks, but the epilogue's pair accesses become 2-way conflicted
__device__ __forceinline__ int swz(int r, int c) { return r * 32 + (((c >> 2) ^ (r & 7)) << 2) + (c & 3); }
#else
__device__ __forceinline__ int swz(int r, int c) {
  const int h = ((r ^ (r >> 2)) & 1) | (r & 2);
  return r * 32 + (((c >> 3) ^ h) << 3) + (c & 7);
}
#endif

// packed fp32x2 arithmetic (FADD2 / FMUL2 / FFMA2 on sm_100a), IEEE round-to-nearest
__device__ __forceinline__ unsigned long long pk(float x, float y) {
  return ((unsigned long long)__float_as_uint(y) << 32) | __float_as_uint(x);
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long c;
  asm("add.rn.f32x2 %0, %1, %2;\n" : "=l"(c) : "l"(a), "l"(b));
  return c;
}
__device__ __forceinline__ unsigned long long mul2(unsigned long long a, unsigned long long b) {
  unsigned long long c;
  asm("mul.rn.f32x2 %0, %1, %2;\n" : "=l"(c) : "l"(a), "l"(b));
  return c;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;\n" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// 3xTF32 split (reading R14): hi = tf32 round-to-nearest-even of x (cvt.rn.tf32.f32 is ONE
// F2FP.TF32 instruction; the round-1 bit-pattern rna split took two and is kept as the
// NSERIES_BW_SPLIT_BITS variant: 281 -> 258 us per config-4 batch, same error,
// profiles/r02_batched_f2fp_split.txt); lo = x - hi is
// exact in fp32 and is passed as is -- the tensor core reads the top 19 bits of a .tf32 operand,
// i.e. truncates lo, an error below 2^-11 |lo| <= 2^-22 |x| (same order as the dropped lo*lo).
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
#if defined(NSERIES_BW_NOSPLIT)   // timing experiment only (wrong numerics): no split instructions
  hi = lo = __float_as_uint(x);
  return;
#endif
#if defined(NSERIES_BW_SPLIT_BITS)
  hi = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
#else
  // round to nearest EVEN: one F2FP.TF32.F32 on sm_100a (cvt.rna is emulated by 4 instructions)
  asm("cvt.rn.tf32.f32 %0, %1;\n" : "=r"(hi) : "f"(x));
#endif
  lo = __float_as_uint(x - __uint_as_float(hi));
}

__device__ __forceinline__ void mma_tf32(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// first product of a chain: C = 0 (no accumulator zeroing instructions)
__device__ __forceinline__ void mma_tf32_z(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                           uint32_t a3, uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%10,%10,%10};\n"
      : "=f"(c[0]), "=f"(c[1]), "=f"(c[2]), "=f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(0.f));
}

__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async4(float* dst, const float* src, int bytes) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// A_b (d x d row-major, contiguous) -> swizzled 32 x 32 slot, zero padded; the group's
// 32*WPM lanes share the copy (glane = lane index within the group).
template <int WPM>
__device__ __forceinline__ void load_matrix_async(float* dst, const float* src, int d, bool vec, int glane) {
  if (vec) {   // d == 32 and 16-byte aligned: 256 chunks of 16 bytes
#pragma unroll
    for (int i = 0; i < 8 / WPM; ++i) {
      const int q = glane + 32 * WPM * i, r = q >> 3, c4 = q & 7;
      cp_async16(dst + swz(r, c4 * 4), src + q * 4);
    }
  } else {
    for (int i = 0; i < 32 / WPM; ++i) {
      const int idx = glane + 32 * WPM * i, r = idx >> 5, c = idx & 31;
      const bool in = r < d && c < d;
      cp_async4(dst + swz(r, c), in ? src + r * d + c : src, in ? 4 : 0);   // 0 bytes = zero fill
    }
  }
}

template <int WPM>
__device__ __forceinline__ void group_sync(int group) {
  if (WPM == 1) __syncwarp();
  else asm volatile("bar.sync %0, %1;\n" ::"r"(1 + group), "n"(32 * WPM) : "memory");   // <= 15 groups
}

// Decoded op in shared memory: slot codes resolved to float offsets from the group's slot base
// (two copies of the op list, one per A double-buffer phase, so no per-op address arithmetic).
struct __align__(16) DevOp {
  uint16_t x, y, aux[kMaxAux], out[kMaxOut];   // float offsets; out = kNoOff if not kept
  uint8_t kind, epi, gmask, pad;                // kind: 0 axpby, 1 gemm, 2 gemm X = I, 3 gemm Y = I
  float alpha[kMaxOut], beta[kMaxOut][kMaxAux], gamma[kMaxOut];
};
constexpr uint16_t kNoOff = 0xffff;

#ifdef NSERIES_BW_TIMING   // harness-only (tools/bw_probe.cu): per-phase clocks summed over warps
__device__ unsigned long long g_bwt[4];   // mainloop, barrier 1, epilogue, barrier 2
#define BW_T(i) const long long bwt##i = clock64()
#define BW_TACC tacc[0] += bwt1 - bwt0; tacc[1] += bwt2 - bwt1; tacc[2] += bwt3 - bwt2; tacc[3] += bwt4 - bwt3
#define BW_TPARAM , long long (&tacc)[4]
#define BW_TARG , tacc
#else
#define BW_T(i) ((void)0)
#define BW_TACC ((void)0)
#define BW_TPARAM
#define BW_TARG
#endif

// Row-block order: warp w of a 2-warp group walks its two m16 row blocks in the order
// mb = lm ^ w (lm = 0, 1), so the tiles holding diagonal elements are (lm = 0, j = hh) for both
// warps -- a compile-time fact in the epilogue (WPM = 1: j = 2 lm + hh with lm = mb).  WPM = 4
// keeps mb = lm and tests the diagonal at run time.  (Natural row order with a run-time
// mb == w predicate measured slower: 254 -> 260 us, profiles/r02_batched_diag_ab.txt.)
template <int WPM>
__device__ __forceinline__ int row_swap(int wig) { return WPM == 2 ? wig : 0; }
template <int WPM>
__device__ __forceinline__ bool diag_tile(int lm, int j, int hh, int nb0) {
  if (WPM == 2) return lm == 0 && j == hh;
  if (WPM == 1) return j == 2 * lm + hh;
  return nb0 + j == 2 * lm + hh;
}

// This warp's part of X * Y into registers: rows 0..31 (2 m16 tiles, local index lm = mb ^ msw)
// x column tiles nb0 .. nb0+NBW-1 (n8 tiles).  XI / YI: operand is the identity (synthesised,
// zero outside the d x d block); its tf32 lo part is exactly zero, so that cross product is not
// issued (the product is still the full 3xTF32 product: the skipped term is 0).
__device__ __forceinline__ void add_acc(float (&b)[4], const float (&t)[4]) {   // b += t, IEEE RN
  const unsigned long long p01 = add2(pk(b[0], b[1]), pk(t[0], t[1]));
  const unsigned long long p23 = add2(pk(b[2], b[3]), pk(t[2], t[3]));
  b[0] = __uint_as_float((uint32_t)p01);
  b[1] = __uint_as_float((uint32_t)(p01 >> 32));
  b[2] = __uint_as_float((uint32_t)p23);
  b[3] = __uint_as_float((uint32_t)(p23 >> 32));
}

#if defined(NSERIES_BW_FFMA)
// CONTROL VARIANT (harness-only, tools/variants): the same fragment outputs computed with SIMT
// fp32 FMAs (packed FFMA2, one fp32 product instead of three tf32 ones): the lane's 4 rows x
// 2 column pairs form a 4x4 outer-product block; X quads by LDS.128, Y pairs by LDS.64.
template <int NBW, bool XI, bool YI>
__device__ __forceinline__ void warp_mma(const float* X, const float* Y, int d, int g, int t, int nb0, int msw,
                                         float (&big)[2][NBW][4], float (&sml)[2][NBW][4]) {
#pragma unroll
  for (int lm = 0; lm < 2; ++lm)
#pragma unroll
    for (int j = 0; j < NBW; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) sml[lm][j][e] = 0.f;
  if (XI || YI) {   // I * Y = Y, X * I = X at the fragment positions (zero outside d x d)
    const float* V = XI ? Y : X;
#pragma unroll
    for (int lm = 0; lm < 2; ++lm)
#pragma unroll
      for (int j = 0; j < NBW; ++j)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const float2 v = *reinterpret_cast<const float2*>(V + 512 * (lm ^ msw) + swz(8 * hh + g, 8 * (nb0 + j) + 2 * t));
          big[lm][j][2 * hh] = v.x;
          big[lm][j][2 * hh + 1] = v.y;
        }
    return;
  }
  unsigned long long acc[2][NBW][2];
#pragma unroll
  for (int lm = 0; lm < 2; ++lm)
#pragma unroll
    for (int j = 0; j < NBW; ++j) acc[lm][j][0] = acc[lm][j][1] = 0ull;
#ifndef NSERIES_BW_FFMA_UNROLL
#define NSERIES_BW_FFMA_UNROLL 2
#endif
  constexpr int kFfmaUnroll = NSERIES_BW_FFMA_UNROLL;   // (pragma arguments are not macro-expanded)
#pragma unroll kFfmaUnroll
  for (int q = 0; q < 8; ++q) {   // k = 4q .. 4q+3
    float4 xq[2][2];
#pragma unroll
    for (int lm = 0; lm < 2; ++lm)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
        xq[lm][hh] = *reinterpret_cast<const float4*>(X + 512 * (lm ^ msw) + swz(8 * hh + g, 4 * q));
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      unsigned long long yp[NBW];
#pragma unroll
      for (int j = 0; j < NBW; ++j) yp[j] = *reinterpret_cast<const unsigned long long*>(Y + swz(4 * q + kk, 8 * (nb0 + j) + 2 * t));
#pragma unroll
      for (int lm = 0; lm < 2; ++lm)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const float xv = kk == 0 ? xq[lm][hh].x : kk == 1 ? xq[lm][hh].y : kk == 2 ? xq[lm][hh].z : xq[lm][hh].w;
#pragma unroll
          for (int j = 0; j < NBW; ++j) acc[lm][j][hh] = fma2(pk(xv, xv), yp[j], acc[lm][j][hh]);
        }
    }
  }
#pragma unroll
  for (int lm = 0; lm < 2; ++lm)
#pragma unroll
    for (int j = 0; j < NBW; ++j)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        big[lm][j][2 * hh] = __uint_as_float((uint32_t)acc[lm][j][hh]);
        big[lm][j][2 * hh + 1] = __uint_as_float((uint32_t)(acc[lm][j][hh] >> 32));
      }
}
#else
template <int NBW, bool XI, bool YI>
__device__ __forceinline__ void warp_mma(const float* X, const float* Y, int d, int g, int t, int nb0, int msw,
                                         float (&big)[2][NBW][4], float (&sml)[2][NBW][4]) {
#if !defined(NSERIES_BW_CHAIN_BIG)
  float tk[2][NBW][4];   // hi*hi of the previous k-step, added one k-step late
#endif
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int k0 = 8 * s + 2 * t;   // this lane's k pair in k-step s: k0 (slot t), k0+1 (slot t+4)
    float2 xa[2][2];                // [lm][hh]: X[16 (lm ^ msw) + 8 hh + g][k0 .. k0+1]
    float yb[NBW][2];               // [j][e]:  Y[k0 + e][8 (nb0 + j) + g]
#pragma unroll
    for (int lm = 0; lm < 2; ++lm)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int r = 16 * (lm ^ msw) + 8 * hh + g;
        if (XI) xa[lm][hh] = make_float2((r == k0 && r < d) ? 1.f : 0.f, (r == k0 + 1 && r < d) ? 1.f : 0.f);
        else xa[lm][hh] = *reinterpret_cast<const float2*>(X + 512 * (lm ^ msw) + swz(8 * hh + g, k0));
      }
#pragma unroll
    for (int j = 0; j < NBW; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * (nb0 + j) + g;
        if (YI) yb[j][e] = (k0 + e == c && c < d) ? 1.f : 0.f;
        else yb[j][e] = Y[swz(k0 + e, c)];
      }
    uint32_t ah[2][2][2], al[2][2][2], bh[NBW][2], bl[NBW][2];
#pragma unroll
    for (int lm = 0; lm < 2; ++lm)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        if (XI) {   // 0 / 1 are exact tf32 values
          ah[lm][hh][0] = __float_as_uint(xa[lm][hh].x);
          ah[lm][hh][1] = __float_as_uint(xa[lm][hh].y);
        } else {
          split_tf32(xa[lm][hh].x, ah[lm][hh][0], al[lm][hh][0]);
          split_tf32(xa[lm][hh].y, ah[lm][hh][1], al[lm][hh][1]);
        }
      }
#pragma unroll
    for (int j = 0; j < NBW; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (YI) bh[j][e] = __float_as_uint(yb[j][e]);
        else split_tf32(yb[j][e], bh[j][e], bl[j][e]);
      }
    // issue order: the three products of a k-step run over all tiles before an accumulator is
    // reused; fragment a = {(g, t), (g+8, t), (g, t+4), (g+8, t+4)}, b = {t, t+4}
    if (!XI) {
#pragma unroll
      for (int lm = 0; lm < 2; ++lm)
#pragma unroll
        for (int j = 0; j < NBW; ++j) {
          if (s == 0) mma_tf32_z(sml[lm][j], al[lm][0][0], al[lm][1][0], al[lm][0][1], al[lm][1][1], bh[j][0], bh[j][1]);
          else mma_tf32(sml[lm][j], al[lm][0][0], al[lm][1][0], al[lm][0][1], al[lm][1][1], bh[j][0], bh[j][1]);
        }
    }
#pragma unroll
    for (int lm = 0; lm < 2; ++lm)
#pragma unroll
      for (int j = 0; j < NBW; ++j) {
#if defined(NSERIES_BW_CHAIN_BIG)
        if (s == 0) mma_tf32_z(big[lm][j], ah[lm][0][0], ah[lm][1][0], ah[lm][0][1], ah[lm][1][1], bh[j][0], bh[j][1]);
        else mma_tf32(big[lm][j], ah[lm][0][0], ah[lm][1][0], ah[lm][0][1], ah[lm][1][1], bh[j][0], bh[j][1]);
#else
        // hi*hi of each k-step from a zero accumulator, summed in fp32 registers with IEEE
        // round-to-nearest adds: a chained tensor-core accumulator truncates at every k-step
        // (profiles/r01_tf32_accumulation_probe.txt), which biases the dominant term; the
        // cross terms (2^-11 smaller) stay chained
        if (s == 0) {
          mma_tf32_z(big[lm][j], ah[lm][0][0], ah[lm][1][0], ah[lm][0][1], ah[lm][1][1], bh[j][0], bh[j][1]);
        } else {
          // the k-step's hi*hi sum is added one k-step later, so the FADD2 does not wait on the
          // HMMA just issued (same summation order ((s0 + s1) + s2) + s3, bit-identical results;
          // 258 -> 254 us per config-4 batch, profiles/r02_batched_lag_add.txt)
          if (s >= 2) add_acc(big[lm][j], tk[lm][j]);
          mma_tf32_z(tk[lm][j], ah[lm][0][0], ah[lm][1][0], ah[lm][0][1], ah[lm][1][1], bh[j][0], bh[j][1]);
          if (s == 3) add_acc(big[lm][j], tk[lm][j]);
        }
#endif
      }
    if (!YI) {
#pragma unroll
      for (int lm = 0; lm < 2; ++lm)
#pragma unroll
        for (int j = 0; j < NBW; ++j) {
          if (XI && s == 0) mma_tf32_z(sml[lm][j], ah[lm][0][0], ah[lm][1][0], ah[lm][0][1], ah[lm][1][1], bl[j][0], bl[j][1]);
          else mma_tf32(sml[lm][j], ah[lm][0][0], ah[lm][1][0], ah[lm][0][1], ah[lm][1][1], bl[j][0], bl[j][1]);
        }
    }
  }
}

#endif   // NSERIES_BW_FFMA

// Epilogue out_j = alpha_j acc + sum_i beta_ji aux_i + gamma_j I on the accumulator registers.
// Outputs go to their shared-memory slots; with FIN (the op producing the final S, once per
// matrix) outputs flagged in gmask also go to global memory (8-byte stores when vec_out) and
// NSERIES_CHECK_FINITE counts their NaN/Inf entries.  Pairs of columns (2t, 2t+1) are
// processed as packed fp32x2.  gamma_j I is added on the diagonal tiles only (diag_tile);
// diagonal positions of the zero padding beyond d get it too: values stay block-diagonal
// (the padding block carries the scalar series at 0), and nothing beyond d is stored or read
// into the d x d block.
typedef unsigned long long u64;
template <int WPM, int NBW, int NA, int NO, bool FIN>
__device__ __forceinline__ void warp_epilogue(const DevOp& op, float* ws, float* Sg, int d, bool vec_out, int g,
                                              int t, int nb0, int msw, const float (&big)[2][NBW][4],
                                              const float (&sml)[2][NBW][4], int* nonfinite) {
  const float* auxp[NA > 0 ? NA : 1];
  float* outp[NO];
  u64 alpha[NO], beta[NO][NA > 0 ? NA : 1];
  float gamma[NO];
  bool to_slot[NO], to_g[NO];
  const bool dg0 = (g == 2 * t), dg1 = (g == 2 * t + 1);
#pragma unroll
  for (int x = 0; x < NA; ++x) auxp[x] = ws + op.aux[x];
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    to_slot[o] = !FIN || op.out[o] != kNoOff;
    to_g[o] = FIN && (op.gmask & (1 << o));
    outp[o] = ws + (to_slot[o] ? op.out[o] : 0);
    alpha[o] = pk(op.alpha[o], op.alpha[o]);
    gamma[o] = op.gamma[o];
#pragma unroll
    for (int x = 0; x < NA; ++x) beta[o][x] = pk(op.beta[o][x], op.beta[o][x]);
  }
  int nonfin = 0;
  // Batches of 2*NBW column pairs: every aux load of a batch is issued before its first store
  // (an output may overwrite an aux slot in place, so the compiler cannot reorder them itself).
#pragma unroll
  for (int lm = 0; lm < 2; ++lm) {
    const int rb = 16 * (lm ^ msw);
    u64 av[NBW][2][NA > 0 ? NA : 1];
#pragma unroll
    for (int j = 0; j < NBW; ++j)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
#pragma unroll
        for (int x = 0; x < NA; ++x)
          av[j][hh][x] = *reinterpret_cast<const u64*>(auxp[x] + 32 * rb + swz(8 * hh + g, 8 * (nb0 + j) + 2 * t));
#pragma unroll
    for (int j = 0; j < NBW; ++j)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int r = rb + 8 * hh + g, c = 8 * (nb0 + j) + 2 * t;
        const int off = 32 * rb + swz(8 * hh + g, c);
        const u64 acc = add2(pk(big[lm][j][2 * hh], big[lm][j][2 * hh + 1]),
                             pk(sml[lm][j][2 * hh], sml[lm][j][2 * hh + 1]));
        const bool diag = diag_tile<WPM>(lm, j, hh, nb0);
#pragma unroll
        for (int o = 0; o < NO; ++o) {
          u64 v = mul2(alpha[o], acc);
#pragma unroll
          for (int x = 0; x < NA; ++x) v = fma2(beta[o][x], av[j][hh][x], v);
          if (diag) v = add2(v, pk(dg0 ? gamma[o] : 0.f, dg1 ? gamma[o] : 0.f));
          if (to_slot[o]) *reinterpret_cast<u64*>(outp[o] + off) = v;
          if (FIN && to_g[o]) {
            const float v0 = __uint_as_float((uint32_t)v), v1 = __uint_as_float((uint32_t)(v >> 32));
            if (nonfinite)
              nonfin += ((r < d && c < d && !isfinite(v0)) ? 1 : 0) + ((r < d && c + 1 < d && !isfinite(v1)) ? 1 : 0);
            if (vec_out) {
              *reinterpret_cast<float2*>(Sg + r * 32 + c) = make_float2(v0, v1);
            } else if (r < d) {
              if (c < d) Sg[r * d + c] = v0;
              if (c + 1 < d) Sg[r * d + c + 1] = v1;
            }
          }
        }
      }
  }
  if (FIN && nonfinite) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nonfin += __shfl_xor_sync(0xffffffffu, nonfin, o);
    if (((threadIdx.x & 31) == 0) && nonfin) atomicAdd(nonfinite, nonfin);
  }
}

// One fused op for the group's matrix (this warp's column tiles).
template <int WPM>
__device__ __forceinline__ void warp_op(const DevOp& op, float* ws, float* Sg, int d, bool vec_out, int g, int t,
                                        int nb0, int msw, int group, int* nonfinite BW_TPARAM) {
  constexpr int NBW = 4 / WPM;
  float big[2][NBW][4], sml[2][NBW][4];
  const int kind = op.kind;
  BW_T(0);
  if (kind == 1) warp_mma<NBW, false, false>(ws + op.x, ws + op.y, d, g, t, nb0, msw, big, sml);
  else if (kind == 2) warp_mma<NBW, true, false>(ws, ws + op.y, d, g, t, nb0, msw, big, sml);
  else if (kind == 3) warp_mma<NBW, false, true>(ws + op.x, ws, d, g, t, nb0, msw, big, sml);
  else {   // axpby op (rare: elided binary plans, k = 1): acc = 0.  The zeros are volatile
           // moves so ptxas cannot hoist 16 CS2R above the kind branch into every product.
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int j = 0; j < NBW; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          asm volatile("mov.b32 %0, 0;\n" : "=f"(big[mb][j][e]));
          asm volatile("mov.b32 %0, 0;\n" : "=f"(sml[mb][j][e]));
        }
  }
#ifdef NSERIES_BW_TIMING
  {   // wait for the accumulators so the mainloop time includes the last HMMAs
    float z = 0.f;
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int j = 0; j < NBW; ++j) z += big[mb][j][0] + sml[mb][j][0];
    if (z == 1.2345e-30f) Sg[0] = z;
  }
#endif
  BW_T(1);
  NSERIES_SHAKE_POINT(8 * kind + 1);
  group_sync<WPM>(group);   // every operand read of the group precedes any output write (in-place slots)
  NSERIES_SHAKE_POINT(8 * kind + 2);
  BW_T(2);
#if defined(NSERIES_BW_PROBE) && NSERIES_BW_PROBE == 1   // tools/bw_probe.cu: mainloop only
  {
    float sum = 0.f;
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int j = 0; j < NBW; ++j) sum += big[mb][j][0] + sml[mb][j][3];
    if (sum == 1.2345f) Sg[0] = sum;
    group_sync<WPM>(group);
    return;
  }
#endif
  const int sel = op.epi + (op.gmask ? 16 : 0);
  switch (sel) {
#define NSERIES_EPI(NA, NO)                                                                          \
  case NA * 4 + NO:                                                                                  \
    warp_epilogue<WPM, NBW, NA, NO, false>(op, ws, Sg, d, vec_out, g, t, nb0, msw, big, sml, nonfinite); \
    break;
#define NSERIES_FIN(NA, NO)                                                                          \
  case 16 + NA * 4 + NO:                                                                             \
    warp_epilogue<WPM, NBW, NA, NO, true>(op, ws, Sg, d, vec_out, g, t, nb0, msw, big, sml, nonfinite);  \
    break;
    NSERIES_EPI(0, 1) NSERIES_EPI(0, 2) NSERIES_EPI(0, 3)
    NSERIES_EPI(1, 1) NSERIES_EPI(1, 2) NSERIES_EPI(1, 3)
    NSERIES_EPI(2, 1) NSERIES_EPI(2, 2) NSERIES_EPI(2, 3)
    NSERIES_EPI(3, 1) NSERIES_EPI(3, 2) NSERIES_EPI(3, 3)
    // the op producing the final S has at most 2 aux / 2 outputs in every compiled plan
    // (build_warp_program refuses others; the 3-aux / 3-output final variants would spill)
    NSERIES_FIN(0, 1) NSERIES_FIN(0, 2) NSERIES_FIN(1, 1) NSERIES_FIN(1, 2) NSERIES_FIN(2, 1) NSERIES_FIN(2, 2)
#undef NSERIES_FIN
#undef NSERIES_EPI
    default: break;
  }
  BW_T(3);
  NSERIES_SHAKE_POINT(8 * kind + 3);
  group_sync<WPM>(group);
  BW_T(4);
  BW_TACC;
}

// One CTA per SM holding up to 8 groups (one copy of the decoded op list per CTA); register
// budgets: WPM 1 -> 255, 2 -> 128, 4 -> 64 per thread.
template <int WPM>
#ifndef NSERIES_BW_GROUPS
#define NSERIES_BW_GROUPS 8   // warp groups (matrices) per CTA = per SM; the register budget follows
#endif                        // (measured: 6 groups / 170 regs 255.6 us, 7 / 146 295 us, 8 / 128 254 us)
__global__ void __launch_bounds__(32 * NSERIES_BW_GROUPS * WPM, 1)
batched_warp_f32_kernel(const float* __restrict__ A, int64_t strideA, const float* const* __restrict__ A_ptrs,
                        float* __restrict__ S, int64_t strideS, float* const* __restrict__ S_ptrs, int batch,
                        int d, const __grid_constant__ WarpProgram prog, int* __restrict__ nonfinite) {
  extern __shared__ __align__(16) float smem_f[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int group = warp / WPM, wig = warp % WPM, groups = (blockDim.x >> 5) / WPM;
  const int g = lane >> 2, t = lane & 3, glane = wig * 32 + lane, nb0 = wig * (4 / WPM);
  const int msw = row_swap<WPM>(wig);
  // decoded op list, two copies (A in buffer 0 / buffer 1), ahead of the groups' slots
  DevOp* sops = reinterpret_cast<DevOp*>(smem_f);
  for (int i = threadIdx.x; i < 2 * prog.n_ops; i += blockDim.x) {
    const int ph = i / prog.n_ops;
    const WarpOp& w = prog.ops[i % prog.n_ops];
    const int a_off = (prog.n_slots + ph) * kSlotF;
    auto off = [&](int code) -> uint16_t {
      return code >= 0 ? (uint16_t)(code * kSlotF) : (code == kWSlotA ? (uint16_t)a_off : kNoOff);
    };
    DevOp o;
    o.x = off(w.X);
    o.y = off(w.Y);
#pragma unroll
    for (int x = 0; x < kMaxAux; ++x) o.aux[x] = off(w.aux[x]);
#pragma unroll
    for (int j = 0; j < kMaxOut; ++j) o.out[j] = off(w.out[j]);
    o.kind = !w.gemm ? 0 : (w.X == kWSlotI ? 2 : (w.Y == kWSlotI ? 3 : 1));
    o.epi = (uint8_t)(w.n_aux * 4 + w.n_out);
    o.gmask = (uint8_t)w.gmask;
    o.pad = 0;
#pragma unroll
    for (int j = 0; j < kMaxOut; ++j) {
      o.alpha[j] = w.alpha[j];
      o.gamma[j] = w.gamma[j];
#pragma unroll
      for (int x = 0; x < kMaxAux; ++x) o.beta[j][x] = w.beta[j][x];
    }
    sops[i] = o;
  }
  __syncthreads();
  float* ws = smem_f + 2 * prog.n_ops * (sizeof(DevOp) / sizeof(float)) + (size_t)group * (prog.n_slots + 2) * kSlotF;
  float* abuf0 = ws + prog.n_slots * kSlotF;
  const int gg = blockIdx.x * groups + group, ng = gridDim.x * groups;
  auto srcp = [&](int b) -> const float* { return A_ptrs ? A_ptrs[b] : A + (int64_t)b * strideA; };
  auto vec_ok = [&](const void* p) { return d == 32 && ((uintptr_t)p & 15) == 0; };
  int cur = 0;
#ifdef NSERIES_BW_TIMING
  long long tacc[4] = {0, 0, 0, 0};
#endif
#ifdef NSERIES_BW_PROBE
  if (prog.probe_delay_ns && blockIdx.x * 2 >= gridDim.x) __nanosleep(prog.probe_delay_ns);
#endif
  if (gg < batch) {
    const float* p = srcp(gg);
    load_matrix_async<WPM>(abuf0, p, d, vec_ok(p), glane);
  }
  cp_async_commit();
  for (int b = gg; b < batch; b += ng) {
    const int bn = b + ng;
    NSERIES_SHAKE_POINT(100 + (b & 7));
    if (bn < batch) {
      const float* p = srcp(bn);
      load_matrix_async<WPM>(abuf0 + (cur ^ 1) * kSlotF, p, d, vec_ok(p), glane);
    }
    cp_async_commit();
    cp_async_wait<1>();
    NSERIES_SHAKE_POINT(110 + (b & 7));
    group_sync<WPM>(group);
    float* Sg = S_ptrs ? S_ptrs[b] : S + (int64_t)b * strideS;
    const bool vec_out = d == 32 && ((uintptr_t)Sg & 7) == 0;
    const DevOp* ops = sops + cur * prog.n_ops;
    for (int o = 0; o < prog.n_ops; ++o)
      warp_op<WPM>(ops[o], ws, Sg, d, vec_out, g, t, nb0, msw, group, nonfinite BW_TARG);
    cur ^= 1;
  }
  cp_async_wait<0>();
#ifdef NSERIES_BW_TIMING
  if (lane == 0)
    for (int i = 0; i < 4; ++i) atomicAdd(&g_bwt[i], (unsigned long long)tacc[i]);
#endif
}

template <int WPM>
int launch_wpm(const void* A, int64_t strideA, const void* const* A_ptrs, void* S, int64_t strideS,
               void* const* S_ptrs, int batch, int d, const WarpProgram& prog, cudaStream_t stream,
               int* nonfinite) {
  const size_t per_group = (size_t)(prog.n_slots + 2) * kSlotF * sizeof(float);
  const size_t prog_bytes = 2 * (size_t)prog.n_ops * sizeof(DevOp);
  const int groups = (int)std::min<size_t>(NSERIES_BW_GROUPS, (227 * 1024 - prog_bytes) / per_group);
  if (groups < 1 || prog.n_slots + 2 > 60) return -1;   // uint16 float offsets
  const size_t smem = prog_bytes + groups * per_group;
  auto kern = batched_warp_f32_kernel<WPM>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, groups * WPM * 32, smem);
  if (per_sm < 1) return -1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::max(1, std::min((batch + groups - 1) / groups, sms * per_sm));
  kern<<<grid, groups * WPM * 32, smem, stream>>>(
      static_cast<const float*>(A), strideA, reinterpret_cast<const float* const*>(A_ptrs),
      static_cast<float*>(S), strideS, reinterpret_cast<float* const*>(S_ptrs), batch, d, prog, nonfinite);
  return (int)cudaGetLastError();
}

}  // namespace

nseries_status build_warp_program(const Program& P, WarpProgram* out, bool inplace) {
  if ((int)P.ops.size() > kMaxBatchedOps) return NSERIES_ERR_UNSUPPORTED_SIZE;
  const std::vector<int> last_use = value_last_use(P);
  std::vector<bool> needs(P.n_values, false);
  for (int v = 0; v < P.n_values; ++v)
    needs[v] = P.val_kind[v] == V_TEMP || ((v == P.final_S || v == P.final_R) && last_use[v] >= 0);
  std::vector<int> wslot;
  WarpProgram& wp = *out;
  wp = WarpProgram{};
  wp.n_slots = assign_slots_inplace(P, needs, &wslot, inplace);
  wp.n_ops = (int)P.ops.size();
  auto code = [&](int v) -> int {
    if (P.val_kind[v] == V_USER_A) return kWSlotA;
    if (P.val_kind[v] == V_IDENT) return kWSlotI;
    return wslot[v] >= 0 ? wslot[v] : kWSlotNone;
  };
  for (int i = 0; i < wp.n_ops; ++i) {
    const Op& op = P.ops[i];
    WarpOp& w = wp.ops[i];
    w.gemm = op.gemm ? 1 : 0;
    w.X = op.gemm ? (int8_t)code(op.X) : 0;
    w.Y = op.gemm ? (int8_t)code(op.Y) : 0;
    if (op.gemm && w.X == kWSlotI && w.Y == kWSlotI) return NSERIES_ERR_INVALID_ARG;
    w.n_aux = (int8_t)op.n_aux;
    w.n_out = (int8_t)op.n_out;
    w.gmask = 0;
    w.rmask = 0;
    for (int a = 0; a < kMaxAux; ++a) {
      w.aux[a] = a < op.n_aux ? (int8_t)code(op.aux[a]) : 0;
      if (a < op.n_aux && w.aux[a] == kWSlotI) return NSERIES_ERR_INVALID_ARG;   // I is gamma
    }
    for (int j = 0; j < kMaxOut; ++j) {
      w.out[j] = j < op.n_out ? (int8_t)code(op.out[j]) : kWSlotNone;
      if (j < op.n_out && op.out[j] == P.final_S) w.gmask |= (int8_t)(1 << j);
      if (j < op.n_out && op.out[j] == P.final_R) w.rmask |= (int8_t)(1 << j);
      if (j < op.n_out && w.out[j] == kWSlotNone && !((w.gmask | w.rmask) & (1 << j)))
        return NSERIES_ERR_INVALID_ARG;
      w.alpha[j] = (float)op.alpha[j];
      w.gamma[j] = (float)op.gamma[j];
      w.dalpha[j] = op.alpha[j];
      w.dgamma[j] = op.gamma[j];
      for (int a = 0; a < kMaxAux; ++a) {
        w.beta[j][a] = (float)op.beta[j][a];
        w.dbeta[j][a] = op.beta[j][a];
      }
    }
  }
  for (int i = 0; i < wp.n_ops; ++i)   // final-S epilogues are instantiated up to 2 aux / 2 outputs
    if (wp.ops[i].gmask && (wp.ops[i].n_aux > 2 || wp.ops[i].n_out > 2)) return NSERIES_ERR_UNSUPPORTED_SIZE;
  return NSERIES_OK;
}

int launch_batched_warp_f32(const void* A, int64_t strideA, const void* const* A_ptrs, void* S,
                            int64_t strideS, void* const* S_ptrs, int batch, int d,
                            const WarpProgram& prog, void* stream, int* nonfinite) {
  if (d > 32) return -1;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const char* env = getenv("NSERIES_BATCHED_WPM");   // tuning knob (1, 2 or 4 warps per matrix)
  const int wpm = env ? atoi(env) : 2;
  if (wpm == 1) return launch_wpm<1>(A, strideA, A_ptrs, S, strideS, S_ptrs, batch, d, prog, s, nonfinite);
  if (wpm == 4) return launch_wpm<4>(A, strideA, A_ptrs, S, strideS, S_ptrs, batch, d, prog, s, nonfinite);
  return launch_wpm<2>(A, strideA, A_ptrs, S, strideS, S_ptrs, batch, d, prog, s, nonfinite);
}

}  // namespace nseries
