// batched.cu -- batched small-matrix path.
//
// Many independent d x d matrices (d <= 64 fp32, d <= 32 fp64).  ONE launch evaluates the
// whole compiled plan for every matrix: a CTA loads A_b into shared memory once, runs every
// op of the plan (the same fused op list as the large path: mu_m + 2 products per radix-m
// step) on shared-memory slots with warp-level tensor-core MMAs, and stores S_b once.  HBM
// traffic is therefore the algorithmic minimum, 2 d^2 elements per matrix.
//
//   fp32: mma.sync m16n8k8 .tf32 with a 3xTF32 split done in registers at fragment load
//         (hi = cvt.rn.tf32(x), lo = cvt.rn.tf32(x - hi); acc += lo*hi + hi*lo + hi*hi),
//         fp32 accumulation (reading R14).
//   fp64: mma.sync m8n8k4 .f64 (DMMA).
// Matrices are zero-padded to DP (multiple of 16) inside shared memory; gamma*I is applied
// only inside the d x d block so the padding stays exactly zero (block-diagonal argument).
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

namespace nseries {

namespace {

__device__ __forceinline__ uint32_t tf32_rn(float x) {   // one F2FP.TF32 (round to nearest even)
  uint32_t r;
  asm("cvt.rn.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = tf32_rn(x);
  lo = tf32_rn(x - __uint_as_float(hi));
}

__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__device__ __forceinline__ void mma_f64(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

template <typename T, int DP>
struct Smem {
  static constexpr int kLd = DP + 4;            // row stride (elements)
  static constexpr int kSlot = DP * kLd;        // elements per slot
};

constexpr int kThreads = 128;

// ---- one fused op on shared-memory slots: out_j = alpha_j X Y + sum beta_ji aux_i + gamma_j I
// Each warp computes a 16x16 output block (one m16 row block, two n8 blocks) so the split A
// fragment serves two MMA triples.  Tensor-core accumulation truncates toward zero
// (profiles/r01_tf32_accumulation_probe.txt): the hi*hi products and the two cross terms run in
// separate accumulator chains (mode 1 there, bias halved) and are added once at the end.
template <int DP>
__device__ void op_f32(const BatchedOp& op, float* slots, int d) {
  using SM = Smem<float, DP>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  constexpr int MB = DP / 16, NP = DP / 16;     // row blocks x column-pair blocks
  const float* X = slots + op.X * SM::kSlot;
  const float* Y = slots + op.Y * SM::kSlot;
  for (int blk = warp; blk < MB * NP; blk += kThreads / 32) {
    const int mb = blk / NP, np = blk % NP;
    float big[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    float small[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    if (op.gemm) {
#pragma unroll
      for (int kb = 0; kb < DP / 8; ++kb) {
        const int r0 = mb * 16 + g, c0 = kb * 8 + t;
        const float af[4] = {X[r0 * SM::kLd + c0], X[(r0 + 8) * SM::kLd + c0], X[r0 * SM::kLd + c0 + 4],
                             X[(r0 + 8) * SM::kLd + c0 + 4]};
        uint32_t ah[4], al[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) split_tf32(af[i], ah[i], al[i]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int nc = (np * 2 + h) * 8 + g;
          const float bf[2] = {Y[(kb * 8 + t) * SM::kLd + nc], Y[(kb * 8 + t + 4) * SM::kLd + nc]};
          uint32_t bh[2], bl[2];
#pragma unroll
          for (int i = 0; i < 2; ++i) split_tf32(bf[i], bh[i], bl[i]);
          mma_tf32(small[h], al, bh);
          mma_tf32(small[h], ah, bl);
          // hi*hi of each k-step from a zero accumulator, summed with IEEE adds (a chained
          // tensor-core accumulator truncates at every k-step; same as batched_warp.cu)
          float tk[4] = {0.f, 0.f, 0.f, 0.f};
          mma_tf32(tk, ah, bh);
#pragma unroll
          for (int e = 0; e < 4; ++e) big[h][e] += tk[e];
        }
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float acc = big[h][e] + small[h][e];
        const int r = mb * 16 + g + ((e & 2) ? 8 : 0), c = (np * 2 + h) * 8 + 2 * t + (e & 1);
        const bool inside = r < d && c < d;
        float av[kMaxAux];
#pragma unroll
        for (int x = 0; x < kMaxAux; ++x)
          if (x < op.n_aux) av[x] = slots[op.aux[x] * SM::kSlot + r * SM::kLd + c];
#pragma unroll
        for (int o = 0; o < kMaxOut; ++o) {
          if (o >= op.n_out) break;
          float v = op.falpha[o] * acc;
#pragma unroll
          for (int x = 0; x < kMaxAux; ++x)
            if (x < op.n_aux) v = fmaf(op.fbeta[o][x], av[x], v);
          if (r == c && inside) v += op.fgamma[o];
          slots[op.out[o] * SM::kSlot + r * SM::kLd + c] = inside ? v : 0.f;
        }
      }
    }
  }
}

template <int DP>
__device__ void op_f64(const BatchedOp& op, double* slots, int d) {
  using SM = Smem<double, DP>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  constexpr int MB = DP / 8, NB = DP / 8;
  const double* X = slots + op.X * SM::kSlot;
  const double* Y = slots + op.Y * SM::kSlot;
  for (int blk = warp; blk < MB * NB; blk += kThreads / 32) {
    const int mb = blk / NB, nb = blk % NB;
    double acc[2] = {0.0, 0.0};
    if (op.gemm) {
#pragma unroll
      for (int kb = 0; kb < DP / 4; ++kb)
        mma_f64(acc, X[(mb * 8 + g) * SM::kLd + kb * 4 + t], Y[(kb * 4 + t) * SM::kLd + nb * 8 + g]);
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int r = mb * 8 + g, c = nb * 8 + 2 * t + e;
      const bool inside = r < d && c < d;
      double av[kMaxAux];
#pragma unroll
      for (int x = 0; x < kMaxAux; ++x)
        if (x < op.n_aux) av[x] = slots[op.aux[x] * SM::kSlot + r * SM::kLd + c];
#pragma unroll
      for (int o = 0; o < kMaxOut; ++o) {
        if (o >= op.n_out) break;
        double v = op.alpha[o] * acc[e];
#pragma unroll
        for (int x = 0; x < kMaxAux; ++x)
          if (x < op.n_aux) v += op.beta[o][x] * av[x];
        if (r == c && inside) v += op.gamma[o];
        slots[op.out[o] * SM::kSlot + r * SM::kLd + c] = inside ? v : 0.0;
      }
    }
  }
}

template <typename T, int DP>
__global__ void __launch_bounds__(kThreads)
batched_kernel(const T* __restrict__ A, int64_t strideA, const T* const* __restrict__ A_ptrs,
               T* __restrict__ S, int64_t strideS, T* const* __restrict__ S_ptrs, int batch, int d,
               const __grid_constant__ BatchedProgram prog) {
  using SM = Smem<T, DP>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* slots = reinterpret_cast<T*>(smem_raw);
  const int tid = threadIdx.x;
  // zero every slot once: padding rows/cols of each slot stay zero afterwards
  for (int i = tid; i < prog.n_slots * SM::kSlot; i += kThreads) slots[i] = T(0);
  if (prog.ident_slot >= 0)
    for (int i = tid; i < d; i += kThreads) slots[prog.ident_slot * SM::kSlot + i * SM::kLd + i] = T(1);
  __syncthreads();
  for (int b = blockIdx.x; b < batch; b += gridDim.x) {
    const T* Ab = A_ptrs ? A_ptrs[b] : A + (int64_t)b * strideA;
    T* Sb = S_ptrs ? S_ptrs[b] : S + (int64_t)b * strideS;
    T* sa = slots + prog.a_slot * SM::kSlot;
    for (int i = tid; i < d * d; i += kThreads) sa[(i / d) * SM::kLd + (i % d)] = Ab[i];
    __syncthreads();
    for (int o = 0; o < prog.n_ops; ++o) {
      if constexpr (sizeof(T) == 4) op_f32<DP>(prog.ops[o], reinterpret_cast<float*>(slots), d);
      else op_f64<DP>(prog.ops[o], reinterpret_cast<double*>(slots), d);
      __syncthreads();
    }
    const T* ss = slots + prog.s_slot * SM::kSlot;
    for (int i = tid; i < d * d; i += kThreads) Sb[i] = ss[(i / d) * SM::kLd + (i % d)];
    __syncthreads();
  }
}

template <typename T, int DP>
int launch_dp(const void* A, int64_t strideA, const void* const* A_ptrs, void* S, int64_t strideS,
              void* const* S_ptrs, int batch, int d, const BatchedProgram& prog, cudaStream_t s) {
  using SM = Smem<T, DP>;
  const size_t smem = (size_t)prog.n_slots * SM::kSlot * sizeof(T);
  if (smem > 227 * 1024) return -1;
  auto kern = batched_kernel<T, DP>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  if (per_sm < 1) return -1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int grid = std::min(batch, sms * per_sm);
  kern<<<grid, kThreads, smem, s>>>(static_cast<const T*>(A), strideA,
                                    reinterpret_cast<const T* const*>(A_ptrs), static_cast<T*>(S),
                                    strideS, reinterpret_cast<T* const*>(S_ptrs), batch, d, prog);
  return (int)cudaGetLastError();
}

}  // namespace

int launch_batched(nseries_dtype dt, const void* A, int64_t strideA, const void* const* A_ptrs,
                   void* S, int64_t strideS, void* const* S_ptrs, int batch, int d,
                   const BatchedProgram& prog, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dt == NSERIES_F32) {
    if (d <= 16) return launch_dp<float, 16>(A, strideA, A_ptrs, S, strideS, S_ptrs, batch, d, prog, s);
    if (d <= 32) return launch_dp<float, 32>(A, strideA, A_ptrs, S, strideS, S_ptrs, batch, d, prog, s);
    if (d <= 64) return launch_dp<float, 64>(A, strideA, A_ptrs, S, strideS, S_ptrs, batch, d, prog, s);
    return -1;
  }
  if (d <= 16) return launch_dp<double, 16>(A, strideA, A_ptrs, S, strideS, S_ptrs, batch, d, prog, s);
  if (d <= 32) return launch_dp<double, 32>(A, strideA, A_ptrs, S, strideS, S_ptrs, batch, d, prog, s);
  return -1;
}

}  // namespace nseries
