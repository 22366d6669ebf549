// plan_small.cu -- whole-plan single-CTA kernel for small single-matrix evaluations (fp64,
// d <= 64; config 1 of BASELINE.json is d = 64).
//
// At d <= 64 one product is 0.26 MFLOP (~2 us on one SM), far below the launch + tail cost of
// one grid launch per GEMM (~19 us measured per op with the tiled engine).  This kernel runs
// the ENTIRE compiled op list in one launch on one CTA: every op stages X and Y (d x d) from L2
// into shared memory with cp.async, 8 warps compute the d x d product on DMMA (m8n8k4 f64), and
// the fused epilogue writes its outputs back to global memory (L2-resident at this size).  The
// CTA barrier between ops orders the global writes of op i before the reads of op i+1.
// Products are exactly the plan's (mu_m + 2 per step), counted per op as in the tiled path.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "internal.h"

namespace nseries {
namespace {

constexpr int kSmallThreads = 256;
constexpr int kLd = 68;   // padded row (doubles): conflict-free 64-bit fragment loads

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp8(double* smem, const double* g, bool ok) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(g), "r"(ok ? 8 : 0));
}

__global__ void __launch_bounds__(kSmallThreads, 1)
plan_small_f64_kernel(int d, const __grid_constant__ SmallProgram prog) {
  extern __shared__ __align__(16) double sm[];
  double* sX = sm;
  double* sY = sm + 64 * kLd;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  // 8 warps tile the 64 x 64 output as 4 (rows) x 2 (cols) warp tiles of 16 x 32
  const int wm0 = (warp >> 1) * 16, wn0 = (warp & 1) * 32;
  for (int o = 0; o < prog.n_ops; ++o) {
    const SmallOp& op = prog.ops[o];
    double acc[2][4][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    if (op.gemm) {
      for (int i = tid; i < 64 * 64; i += kSmallThreads) {
        const int r = i >> 6, c = i & 63;
        const bool ok = r < d && c < d;
        cp8(sX + r * kLd + c, ok ? op.X + (size_t)r * d + c : op.X, ok);
        cp8(sY + r * kLd + c, ok ? op.Y + (size_t)r * d + c : op.Y, ok);
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
      __syncthreads();
      const int kmax = (d + 3) & ~3;
      for (int k = 0; k < kmax; k += 4) {
        double af[2], bf[4];
#pragma unroll
        for (int i = 0; i < 2; ++i) af[i] = sX[(wm0 + i * 8 + g) * kLd + k + t];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = sY[(k + t) * kLd + wn0 + j * 8 + g];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma884(acc[i][j], af[i], bf[j]);
      }
    }
    // fused epilogue (same algebra as the tiled engine)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int row = wm0 + i * 8 + g;
      if (row >= d) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = wn0 + j * 8 + 2 * t + e;
          if (col >= d) continue;
          const size_t off = (size_t)row * d + col;
          double av[kMaxAux];
#pragma unroll
          for (int x = 0; x < kMaxAux; ++x)
            if (x < op.n_aux) av[x] = op.aux[x][off];
#pragma unroll
          for (int q = 0; q < kMaxOut; ++q) {
            if (q >= op.n_out) break;
            double v = op.alpha[q] * acc[i][j][e];
#pragma unroll
            for (int x = 0; x < kMaxAux; ++x)
              if (x < op.n_aux) v += op.beta[q][x] * av[x];
            if (row == col) v += op.gamma[q];
            op.out[q][off] = v;
          }
        }
      }
    }
    __syncthreads();   // this op's outputs (global, L2) are visible to the next op's loads
  }
}

}  // namespace

int launch_plan_small_f64(int d, const SmallProgram& prog, void* stream) {
  if (d > 64 || prog.n_ops > kMaxSmallOps) return -1;
  const size_t smem = 2 * 64 * kLd * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(plan_small_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    attr = true;
  }
  plan_small_f64_kernel<<<1, kSmallThreads, smem, static_cast<cudaStream_t>(stream)>>>(d, prog);
  return (int)cudaGetLastError();
}

}  // namespace nseries

// ---------------------------------------------------------------------------------------------
// plan_smem_f64_kernel -- the same single-CTA whole-plan launch with EVERY value resident in
// shared memory (d <= 64 fp64, config 1): no per-op global round trip.  Values live in 64x64
// fp64 slots (32 KiB, unpadded, XOR-swizzled in 4-double groups: column c of row r is stored at
// c ^ 4((r & 3) ^ 2(r & 1)), which keeps the DMMA A/B fragment loads and the epilogue's 16-byte
// accesses bank-conflict free).  Slot assignment is in place (assign_slots_inplace): every
// operand of an op is read before a CTA barrier, then the epilogue may overwrite values that die
// at this op.  I as an operand (the paper's S_1 * T) is synthesised in the fragment registers;
// the final S (and R) are written from the accumulators straight to global memory.
namespace nseries {
namespace {

constexpr int kSlotD = 64 * 64;   // doubles per slot

__device__ __forceinline__ int swz64(int r, int c) {
  return r * 64 + (c ^ (4 * ((r & 3) ^ ((r & 1) << 1))));
}

// NW warps tile the 64 x 64 output as 4 (rows, 16 each) x NW/4 (cols, NJ n8 tiles each)
template <int NJ, bool XI, bool YI>
__device__ __forceinline__ void smem_mma(const double* X, const double* Y, int d, int g, int t, int wm0, int wn0,
                                         double (&acc)[2][NJ][2]) {
#pragma unroll 4
  for (int k = 0; k < 64; k += 4) {
    double af[2], bf[NJ];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int r = wm0 + i * 8 + g;
      af[i] = XI ? ((r == k + t && r < d) ? 1.0 : 0.0) : X[swz64(r, k + t)];
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int c = wn0 + j * 8 + g;
      bf[j] = YI ? ((c == k + t && c < d) ? 1.0 : 0.0) : Y[swz64(k + t, c)];
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) dmma884(acc[i][j], af[i], bf[j]);
  }
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1)
plan_smem_f64_kernel(int d, const double* __restrict__ A, double* __restrict__ S, double* __restrict__ R,
                     const __grid_constant__ WarpProgram prog) {
  constexpr int NT = NW * 32, NJ = 8 / (NW / 4);
  extern __shared__ __align__(16) double smd[];
  double* const sA = smd + prog.n_slots * kSlotD;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm0 = (warp & 3) * 16, wn0 = (warp >> 2) * (8 * NJ);
  // A -> its slot (zero padded to 64 x 64)
  for (int i = tid; i < kSlotD; i += NT) {
    const int r = i >> 6, c = i & 63;
    const bool ok = r < d && c < d;
    cp8(sA + swz64(r, c), ok ? A + (size_t)r * d + c : A, ok);
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  auto slot = [&](int code) -> double* { return code == kWSlotA ? sA : smd + (code > 0 ? code : 0) * kSlotD; };
  for (int o = 0; o < prog.n_ops; ++o) {
    const WarpOp& op = prog.ops[o];
    double acc[2][NJ][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    if (op.gemm) {
      if (op.X == kWSlotI) smem_mma<NJ, true, false>(nullptr, slot(op.Y), d, g, t, wm0, wn0, acc);
      else if (op.Y == kWSlotI) smem_mma<NJ, false, true>(slot(op.X), nullptr, d, g, t, wm0, wn0, acc);
      else smem_mma<NJ, false, false>(slot(op.X), slot(op.Y), d, g, t, wm0, wn0, acc);
    }
    __syncthreads();   // every operand read precedes any output write (in-place slots)
    const double* auxp[kMaxAux];
#pragma unroll
    for (int x = 0; x < kMaxAux; ++x) auxp[x] = slot(x < op.n_aux ? op.aux[x] : 0);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int row = wm0 + i * 8 + g;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int col = wn0 + j * 8 + 2 * t;
        const int off = swz64(row, col);   // (col, col + 1) stay adjacent under the swizzle
        double2 av[kMaxAux];
#pragma unroll
        for (int x = 0; x < kMaxAux; ++x)
          av[x] = x < op.n_aux ? *reinterpret_cast<const double2*>(auxp[x] + off) : make_double2(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < kMaxOut; ++q) {
          if (q >= op.n_out) break;
          double v0 = op.dalpha[q] * acc[i][j][0], v1 = op.dalpha[q] * acc[i][j][1];
#pragma unroll
          for (int x = 0; x < kMaxAux; ++x) {   // dbeta = 0 beyond n_aux
            v0 = fma(op.dbeta[q][x], av[x].x, v0);
            v1 = fma(op.dbeta[q][x], av[x].y, v1);
          }
          if (row == col && row < d) v0 += op.dgamma[q];
          if (row == col + 1 && row < d) v1 += op.dgamma[q];
          if (op.out[q] >= 0) *reinterpret_cast<double2*>(smd + op.out[q] * kSlotD + off) = make_double2(v0, v1);
          double* gdst = (op.gmask & (1 << q)) ? S : ((op.rmask & (1 << q)) ? R : nullptr);
          if (gdst && row < d) {
            if (col < d) gdst[(size_t)row * d + col] = v0;
            if (col + 1 < d) gdst[(size_t)row * d + col + 1] = v1;
          }
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace

int launch_plan_smem_f64(int d, const WarpProgram& prog, const double* A, double* S, double* R, void* stream) {
  if (d > 64) return -1;
  const size_t smem = (size_t)(prog.n_slots + 1) * kSlotD * sizeof(double);
  if (smem > 227 * 1024) return -1;
  static const int nw = std::getenv("NSERIES_SMALL_WARPS") ? std::atoi(std::getenv("NSERIES_SMALL_WARPS")) : 16;
  auto launch = [&](auto kern, int threads) -> int {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    kern<<<1, threads, smem, static_cast<cudaStream_t>(stream)>>>(d, A, S, R, prog);
    return (int)cudaGetLastError();
  };
  if (nw == 8) return launch(plan_smem_f64_kernel<8>, 256);
  if (nw == 32) return launch(plan_smem_f64_kernel<32>, 1024);
  return launch(plan_smem_f64_kernel<16>, 512);
}

}  // namespace nseries
