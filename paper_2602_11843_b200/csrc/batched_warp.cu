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

__device__ __forceinline__ int swz(int r, int c) {
  const int h = ((r ^ (r >> 2)) & 1) | (r & 2);
  return r * 32 + (((c >> 3) ^ h) << 3) + (c & 7);
}

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

// This warp's part of X * Y into registers: rows 0..31 (2 m16 tiles) x column tiles
// nb0 .. nb0+NBW-1 (n8 tiles).  XI / YI: operand is the identity (synthesised, zero outside
// the d x d block).
template <int NBW, bool XI, bool YI>
__device__ __forceinline__ void warp_mma(const float* X, const float* Y, int d, int g, int t, int nb0,
                                         float (&big)[2][NBW][4], float (&sml)[2][NBW][4]) {
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int k0 = 8 * s + 2 * t;   // this lane's k pair in k-step s: k0 (slot t), k0+1 (slot t+4)
    float2 xa[2][2];                // [mb][hh]: X[16 mb + 8 hh + g][k0 .. k0+1]
    float yb[NBW][2];               // [j][e]:  Y[k0 + e][8 (nb0 + j) + g]
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int r = 16 * mb + 8 * hh + g;
        if (XI) xa[mb][hh] = make_float2((r == k0 && r < d) ? 1.f : 0.f, (r == k0 + 1 && r < d) ? 1.f : 0.f);
        else xa[mb][hh] = *reinterpret_cast<const float2*>(X + swz(r, k0));
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
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        split_tf32(xa[mb][hh].x, ah[mb][hh][0], al[mb][hh][0]);
        split_tf32(xa[mb][hh].y, ah[mb][hh][1], al[mb][hh][1]);
      }
#pragma unroll
    for (int j = 0; j < NBW; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) split_tf32(yb[j][e], bh[j][e], bl[j][e]);
    // issue order: the three products of a k-step run over all tiles before an accumulator is
    // reused; fragment a = {(g, t), (g+8, t), (g, t+4), (g+8, t+4)}, b = {t, t+4}
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int j = 0; j < NBW; ++j) {
        if (s == 0) mma_tf32_z(sml[mb][j], al[mb][0][0], al[mb][1][0], al[mb][0][1], al[mb][1][1], bh[j][0], bh[j][1]);
        else mma_tf32(sml[mb][j], al[mb][0][0], al[mb][1][0], al[mb][0][1], al[mb][1][1], bh[j][0], bh[j][1]);
      }
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int j = 0; j < NBW; ++j) {
#if defined(NSERIES_BW_CHAIN_BIG)
        if (s == 0) mma_tf32_z(big[mb][j], ah[mb][0][0], ah[mb][1][0], ah[mb][0][1], ah[mb][1][1], bh[j][0], bh[j][1]);
        else mma_tf32(big[mb][j], ah[mb][0][0], ah[mb][1][0], ah[mb][0][1], ah[mb][1][1], bh[j][0], bh[j][1]);
#else
        // hi*hi of each k-step from a zero accumulator, summed in fp32 registers with IEEE
        // round-to-nearest adds: a chained tensor-core accumulator truncates at every k-step
        // (profiles/r01_tf32_accumulation_probe.txt), which biases the dominant term; the
        // cross terms (2^-11 smaller) stay chained
        if (s == 0) {
          mma_tf32_z(big[mb][j], ah[mb][0][0], ah[mb][1][0], ah[mb][0][1], ah[mb][1][1], bh[j][0], bh[j][1]);
        } else {
          float tk[4];
          mma_tf32_z(tk, ah[mb][0][0], ah[mb][1][0], ah[mb][0][1], ah[mb][1][1], bh[j][0], bh[j][1]);
          const unsigned long long p01 = add2(pk(big[mb][j][0], big[mb][j][1]), pk(tk[0], tk[1]));
          const unsigned long long p23 = add2(pk(big[mb][j][2], big[mb][j][3]), pk(tk[2], tk[3]));
          big[mb][j][0] = __uint_as_float((uint32_t)p01);
          big[mb][j][1] = __uint_as_float((uint32_t)(p01 >> 32));
          big[mb][j][2] = __uint_as_float((uint32_t)p23);
          big[mb][j][3] = __uint_as_float((uint32_t)(p23 >> 32));
        }
#endif
      }
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int j = 0; j < NBW; ++j)
        mma_tf32(sml[mb][j], ah[mb][0][0], ah[mb][1][0], ah[mb][0][1], ah[mb][1][1], bl[j][0], bl[j][1]);
  }
}

// Epilogue out_j = alpha_j acc + sum_i beta_ji aux_i + gamma_j I on the accumulator registers,
// outputs to shared-memory slots (every op but the one producing the final S).  Pairs of
// columns (2t, 2t+1) are processed as packed fp32x2.
typedef unsigned long long u64;
template <int NBW, int NA, int NO>
__device__ __forceinline__ void warp_epilogue(const DevOp& op, float* ws, int d, int g, int t,
                                              int nb0, const float (&big)[2][NBW][4],
                                              const float (&sml)[2][NBW][4]) {
  const float* auxp[NA > 0 ? NA : 1];
  float* outp[NO];
  u64 alpha[NO], beta[NO][NA > 0 ? NA : 1];
  float gamma[NO];
#pragma unroll
  for (int x = 0; x < NA; ++x) auxp[x] = ws + op.aux[x];
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    outp[o] = ws + op.out[o];
    alpha[o] = pk(op.alpha[o], op.alpha[o]);
    gamma[o] = op.gamma[o];
#pragma unroll
    for (int x = 0; x < NA; ++x) beta[o][x] = pk(op.beta[o][x], op.beta[o][x]);
  }
  // diagonal elements of this lane: tiles (mb, nb, hh) with nb == 2 mb + hh, row g, cols 2t, 2t+1
  const bool dg0 = (g == 2 * t), dg1 = (g == 2 * t + 1);
  // Batches of 2*NBW column pairs: every aux load of a batch is issued before its first store
  // (an output may overwrite an aux slot in place, so the compiler cannot reorder them itself).
#pragma unroll
  for (int mb = 0; mb < 2; ++mb) {
    u64 av[NBW][2][NA > 0 ? NA : 1];
#pragma unroll
    for (int j = 0; j < NBW; ++j)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
#pragma unroll
        for (int x = 0; x < NA; ++x)
          av[j][hh][x] = *reinterpret_cast<const u64*>(auxp[x] + swz(16 * mb + 8 * hh + g, 8 * (nb0 + j) + 2 * t));
#pragma unroll
    for (int j = 0; j < NBW; ++j)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int nb = nb0 + j;
        const int r = 16 * mb + 8 * hh + g, c = 8 * nb + 2 * t;
        const int off = swz(r, c);
        const u64 acc = add2(pk(big[mb][j][2 * hh], big[mb][j][2 * hh + 1]),
                             pk(sml[mb][j][2 * hh], sml[mb][j][2 * hh + 1]));
        const bool diag = (nb == 2 * mb + hh) && r < d;   // only these tiles hold diagonal elements
#pragma unroll
        for (int o = 0; o < NO; ++o) {
          u64 v = mul2(alpha[o], acc);
#pragma unroll
          for (int x = 0; x < NA; ++x) v = fma2(beta[o][x], av[j][hh][x], v);
          if (diag) v = add2(v, pk(dg0 ? gamma[o] : 0.f, dg1 ? gamma[o] : 0.f));
          *reinterpret_cast<u64*>(outp[o] + off) = v;
        }
      }
  }
}

// Generic epilogue for the op producing the final S (once per matrix): outputs with gmask go to
// global memory (and to their slot if they are read later).
template <int NBW>
__device__ __forceinline__ void warp_epilogue_final(const DevOp& op, float* ws, float* Sg, int d,
                                                    bool vec_out, int g, int t, int nb0,
                                                    const float (&big)[2][NBW][4], const float (&sml)[2][NBW][4],
                                                    int* nonfinite) {
  int nonfin = 0;   // NSERIES_CHECK_FINITE: NaN/Inf entries of the final S
#pragma unroll
  for (int mb = 0; mb < 2; ++mb)
#pragma unroll
    for (int j = 0; j < NBW; ++j)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int r = 16 * mb + 8 * hh + g, c = 8 * (nb0 + j) + 2 * t;
        const int off = swz(r, c);
        const float acc0 = big[mb][j][2 * hh] + sml[mb][j][2 * hh];
        const float acc1 = big[mb][j][2 * hh + 1] + sml[mb][j][2 * hh + 1];
        float2 av[kMaxAux];
#pragma unroll
        for (int x = 0; x < kMaxAux; ++x)
          av[x] = x < (op.epi >> 2) ? *reinterpret_cast<const float2*>(ws + op.aux[x] + off) : make_float2(0.f, 0.f);
#pragma unroll
        for (int o = 0; o < kMaxOut; ++o) {
          if (o >= (op.epi & 3)) break;
          float v0 = op.alpha[o] * acc0, v1 = op.alpha[o] * acc1;
#pragma unroll
          for (int x = 0; x < kMaxAux; ++x) {   // beta = 0 beyond n_aux
            v0 = fmaf(op.beta[o][x], av[x].x, v0);
            v1 = fmaf(op.beta[o][x], av[x].y, v1);
          }
          if (r == c && r < d) v0 += op.gamma[o];
          if (r == c + 1 && r < d) v1 += op.gamma[o];
          if (op.out[o] != kNoOff) *reinterpret_cast<float2*>(ws + op.out[o] + off) = make_float2(v0, v1);
          if (op.gmask & (1 << o)) {
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
  if (nonfinite) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nonfin += __shfl_xor_sync(0xffffffffu, nonfin, o);
    if (((threadIdx.x & 31) == 0) && nonfin) atomicAdd(nonfinite, nonfin);
  }
}

// One fused op for the group's matrix (this warp's column tiles).
template <int WPM>
__device__ __forceinline__ void warp_op(const DevOp& op, float* ws, float* Sg, int d, bool vec_out, int g, int t,
                                        int nb0, int group, int* nonfinite) {
  constexpr int NBW = 4 / WPM;
  float big[2][NBW][4], sml[2][NBW][4];
  const int kind = op.kind;
  if (kind == 1) warp_mma<NBW, false, false>(ws + op.x, ws + op.y, d, g, t, nb0, big, sml);
  else if (kind == 2) warp_mma<NBW, true, false>(ws, ws + op.y, d, g, t, nb0, big, sml);
  else if (kind == 3) warp_mma<NBW, false, true>(ws + op.x, ws, d, g, t, nb0, big, sml);
  else {
#pragma unroll
    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
      for (int j = 0; j < NBW; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) big[mb][j][e] = sml[mb][j][e] = 0.f;
  }
  NSERIES_SHAKE_POINT(8 * kind + 1);
  group_sync<WPM>(group);   // every operand read of the group precedes any output write (in-place slots)
  NSERIES_SHAKE_POINT(8 * kind + 2);
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
  if (op.gmask) {
    warp_epilogue_final<NBW>(op, ws, Sg, d, vec_out, g, t, nb0, big, sml, nonfinite);
  } else switch (op.epi) {
#define NSERIES_EPI(NA, NO) \
  case NA * 4 + NO: warp_epilogue<NBW, NA, NO>(op, ws, d, g, t, nb0, big, sml); break;
    NSERIES_EPI(0, 1) NSERIES_EPI(0, 2) NSERIES_EPI(0, 3)
    NSERIES_EPI(1, 1) NSERIES_EPI(1, 2) NSERIES_EPI(1, 3)
    NSERIES_EPI(2, 1) NSERIES_EPI(2, 2) NSERIES_EPI(2, 3)
    NSERIES_EPI(3, 1) NSERIES_EPI(3, 2) NSERIES_EPI(3, 3)
#undef NSERIES_EPI
    default: break;
  }
  NSERIES_SHAKE_POINT(8 * kind + 3);
  group_sync<WPM>(group);
}

// One CTA per SM holding up to 8 groups (one copy of the decoded op list per CTA); register
// budgets: WPM 1 -> 255, 2 -> 128, 4 -> 64 per thread.
template <int WPM>
__global__ void __launch_bounds__(256 * WPM, 1)
batched_warp_f32_kernel(const float* __restrict__ A, int64_t strideA, const float* const* __restrict__ A_ptrs,
                        float* __restrict__ S, int64_t strideS, float* const* __restrict__ S_ptrs, int batch,
                        int d, const __grid_constant__ WarpProgram prog, int* __restrict__ nonfinite) {
  extern __shared__ __align__(16) float smem_f[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int group = warp / WPM, wig = warp % WPM, groups = (blockDim.x >> 5) / WPM;
  const int g = lane >> 2, t = lane & 3, glane = wig * 32 + lane, nb0 = wig * (4 / WPM);
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
    for (int o = 0; o < prog.n_ops; ++o) warp_op<WPM>(ops[o], ws, Sg, d, vec_out, g, t, nb0, group, nonfinite);
    cur ^= 1;
  }
  cp_async_wait<0>();
}

template <int WPM>
int launch_wpm(const void* A, int64_t strideA, const void* const* A_ptrs, void* S, int64_t strideS,
               void* const* S_ptrs, int batch, int d, const WarpProgram& prog, cudaStream_t stream,
               int* nonfinite) {
  const size_t per_group = (size_t)(prog.n_slots + 2) * kSlotF * sizeof(float);
  const size_t prog_bytes = 2 * (size_t)prog.n_ops * sizeof(DevOp);
  const int groups = (int)std::min<size_t>(8, (227 * 1024 - prog_bytes) / per_group);
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
