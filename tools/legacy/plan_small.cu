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
#include <algorithm>
#include <vector>

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
  if (int e = smem_attr_once<plan_small_f64_kernel>((int)smem)) return e;
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

// ---------------------------------------------------------------------------------------------
// plan_cluster_f64_kernel -- d <= 64 fp64 single matrix on a CLUSTER of 4 CTAs (4 SMs).  CTA c
// owns rows [16c, 16c+16) of every value (its slots hold only that row block, swizzled as
// above).  A product out = X Y needs X's local rows and ALL rows of Y: the 48 remote rows are
// read through distributed shared memory (ld from the peer CTA's slot, mapa-mapped pointers).
// The epilogue writes only local rows (plus this CTA's rows of the final S / R to HBM), and a
// cluster barrier after every op makes them visible to the peers' next reads.  Slots are
// assigned without in-place reuse (a peer may still be reading an operand row while this CTA
// writes its outputs), so one barrier per op suffices.
#include <cooperative_groups.h>
namespace nseries {
namespace {

constexpr int kClusterCtas = 8, kRowsPerCta = 64 / kClusterCtas;     // default cluster: 8 x 8 rows (25 us vs 29 at 4, 36 at 2)
#ifdef NSERIES_SMALL_PROFILE
__device__ long long g_small_prof[256];
#endif
constexpr int kCSlotD = kRowsPerCta * 64;                               // doubles per slot block

// op decoded once per CTA into shared memory (resolved slot offsets; LDS instead of indexed
// constant-bank loads on the per-op critical path)
struct __align__(16) ClusterOp {
  double alpha[kMaxOut], beta[kMaxOut][kMaxAux], gamma[kMaxOut];
  int x, y, kind, n_aux, n_out, gmask, rmask, pad;   // kind: 0 axpby, 1 gemm, 2 X = I, 3 Y = I
  int aux[kMaxAux], out[kMaxOut];                      // offsets (doubles); out < 0: not kept
  int push, csync, wait_bar, tx;   // push bit q: output q replicated; wait_bar: op whose pushes to await
                                   // first (-1: none); tx: bytes this CTA receives from this op's pushes
};

template <int NC>   // CTAs per cluster; each owns RPC = 64 / NC rows of every value
__global__ void __cluster_dims__(NC, 1, 1) __launch_bounds__(256, 1)
plan_cluster_f64_kernel(int d, const double* __restrict__ A, double* __restrict__ S, double* __restrict__ R,
                        const __grid_constant__ WarpProgram prog) {
  constexpr int RPC = 64 / NC, MB = RPC / 8, kLSlotD = RPC * 64, kRSlotD = 64 * 64;
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double smc[];
  const int rank = (int)cluster.block_rank();
  const int r0 = rank * RPC;
  const int n_ops = prog.n_ops;
  // layout: [row-block slots: n_slots x RPC x 64] [replicated slots: n_rep x 64 x 64] [A: 64 x 64]
  const int rep_base = prog.n_slots * kLSlotD;
  const int a_base = rep_base + prog.n_rep * kRSlotD;
  ClusterOp* const sops = reinterpret_cast<ClusterOp*>(smc + a_base + kRSlotD);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wn0 = warp * 8;            // 8 warps x 8 output columns; each warp all local rows
  // own-row base of a value (row-block slot, or this CTA's rows inside a replicated slot / A)
  auto own_of = [&](int code) -> int {
    if (code == kWSlotA) return a_base + r0 * 64;
    if (code >= kWSlotRep) return rep_base + (code - kWSlotRep) * kRSlotD + r0 * 64;
    return (code > 0 ? code : 0) * kLSlotD;
  };
  // full (all 64 rows) base of a replicated value (right operands)
  auto full_of = [&](int code) -> int {
    if (code == kWSlotA) return a_base;
    return rep_base + (code >= kWSlotRep ? code - kWSlotRep : 0) * kRSlotD;
  };
  for (int i = tid; i < n_ops; i += 256) {
    const WarpOp& w = prog.ops[i];
    ClusterOp c;
    c.kind = !w.gemm ? 0 : (w.X == kWSlotI ? 2 : (w.Y == kWSlotI ? 3 : 1));
    c.x = own_of(w.X);
    c.y = full_of(w.Y);
    c.n_aux = w.n_aux;
    c.n_out = w.n_out;
    c.gmask = w.gmask;
    c.rmask = w.rmask;
    c.pad = 0;
    for (int x = 0; x < kMaxAux; ++x) c.aux[x] = own_of(x < w.n_aux ? w.aux[x] : 0);
    c.push = 0;
    c.csync = w.csync;
    c.wait_bar = -1;
    for (int q = 0; q < kMaxOut; ++q) {
      const bool keep = q < w.n_out && w.out[q] != kWSlotNone;
      c.out[q] = keep ? own_of(w.out[q]) : -1;
      if (keep && w.out[q] >= kWSlotRep) c.push |= 1 << q;
      c.alpha[q] = w.dalpha[q];
      c.gamma[q] = w.dgamma[q];
      for (int x = 0; x < kMaxAux; ++x) c.beta[q][x] = w.dbeta[q][x];
    }
    c.tx = (NC - 1) * kLSlotD * 8 * __popc(c.push);
    sops[i] = c;
  }
  __syncthreads();   // every op decoded (threads 0..n_ops-1) before thread 0 reads push / tx
  uint64_t* const bars = reinterpret_cast<uint64_t*>(sops + n_ops);   // one mbarrier per op
  if (tid == 0) {
    int last = -1;
    for (int i = 0; i < n_ops; ++i) {
      sops[i].wait_bar = last;          // pushes of the previous pushing op must have landed
      if (sops[i].push) last = i;
      const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bars + i));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(b) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(sops[i].tx) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // A: every CTA holds all 64 rows (A is read as a right operand), zero padded
  for (int i = tid; i < kRSlotD; i += 256) {
    const int r = i >> 6, c = i & 63;
    const bool ok = r < d && c < d;
    cp8(smc + a_base + swz64(r, c), ok ? A + (size_t)r * d + c : A, ok);
  }
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  // shared::cluster address of this CTA's slot area in every peer (pushes go to the same offset)
  uint32_t peer[NC];
  {
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(smc));
#pragma unroll
    for (int c = 0; c < NC; ++c) asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(peer[c]) : "r"(base), "r"(c));
  }
  const uint32_t bar_off = static_cast<uint32_t>(reinterpret_cast<char*>(bars) - reinterpret_cast<char*>(smc));
  auto wait_bar = [&](int b) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bars + b));
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(a) : "memory");
  };
  cluster.sync();
#ifdef NSERIES_SMALL_PROFILE
  long long tp0 = clock64();
  if (tid == 0 && rank == 0) g_small_prof[0] = tp0;
#endif
  for (int o = 0; o < n_ops; ++o) {
    const ClusterOp& op = sops[o];
    // the replicated rows this op reads were pushed by earlier ops: wait for the latest pushing
    // op's bytes (earlier ones were awaited at their turn); the CTA barrier orders this op's
    // local writes after every warp's reads of the previous ops
    if (op.wait_bar >= 0 && (o == 0 || sops[o - 1].wait_bar != op.wait_bar)) wait_bar(op.wait_bar);
    __syncthreads();
    // KS independent partial accumulators per row block (k-steps s with s % KS == p)
    constexpr int KS = 4;
    double part[MB][KS][2];
#pragma unroll
    for (int i = 0; i < MB; ++i)
#pragma unroll
      for (int p = 0; p < KS; ++p) part[i][p][0] = part[i][p][1] = 0.0;
    const int kind = op.kind;
    if (kind != 0) {
      const bool xi = kind == 2, yi = kind == 3;
      const int xo = op.x, yo = op.y;
      const int col = wn0 + g;
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        const int k = 4 * s + t;
        // right operand: the local replica holds all 64 rows
        const double b = yi ? ((k == col && col < d) ? 1.0 : 0.0) : smc[yo + swz64(k, col)];
#pragma unroll
        for (int i = 0; i < MB; ++i) {
          const int rl = i * 8 + g;
          const double a = xi ? ((r0 + rl == k && r0 + rl < d) ? 1.0 : 0.0) : smc[xo + swz64(rl, k)];
          dmma884(part[i][s % KS], a, b);
        }
      }
    }
    double acc[MB][2];
#pragma unroll
    for (int i = 0; i < MB; ++i)
#pragma unroll
      for (int e = 0; e < 2; ++e) acc[i][e] = (part[i][0][e] + part[i][1][e]) + (part[i][2][e] + part[i][3][e]);
#ifdef NSERIES_SMALL_PROFILE
    if (tid == 0 && rank == 0) g_small_prof[1 + 3 * o] = clock64() + (long long)(acc[0][0] * 0.0);
#endif
    // epilogue on local rows; outputs read later as right operands are pushed to every peer's
    // replica (same offset) with st.async, completing on the peer's mbarrier of this op.  Outputs
    // never alias this op's operands (slots are not reused in place); a replicated slot reused
    // after a peer read it is safe once that peer's later pushes arrived (build_cluster_program
    // marks csync where no such push lies in between)
    if (op.csync) cluster.sync();
    const int n_aux = op.n_aux, n_out = op.n_out;
    const uint32_t my_bar = bar_off + 8u * (uint32_t)o;
#pragma unroll
    for (int i = 0; i < MB; ++i) {
      const int rl = i * 8 + g, row = r0 + rl;
      const int colp = wn0 + 2 * t;
      const int off = swz64(rl, colp);
      double2 av[kMaxAux];
#pragma unroll
      for (int x = 0; x < kMaxAux; ++x)
        av[x] = x < n_aux ? *reinterpret_cast<const double2*>(smc + op.aux[x] + off) : make_double2(0.0, 0.0);
#pragma unroll
      for (int q = 0; q < kMaxOut; ++q) {
        if (q >= n_out) break;
        double v0 = op.alpha[q] * acc[i][0], v1 = op.alpha[q] * acc[i][1];
#pragma unroll
        for (int x = 0; x < kMaxAux; ++x) {
          v0 = fma(op.beta[q][x], av[x].x, v0);
          v1 = fma(op.beta[q][x], av[x].y, v1);
        }
        if (row == colp && row < d) v0 += op.gamma[q];
        if (row == colp + 1 && row < d) v1 += op.gamma[q];
        if (op.out[q] >= 0) {
          *reinterpret_cast<double2*>(smc + op.out[q] + off) = make_double2(v0, v1);
          if (op.push & (1 << q)) {
            const uint32_t lo = 8u * (uint32_t)(op.out[q] + off);
#pragma unroll
            for (int c = 0; c < NC; ++c)
              if (c != rank)
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n"
                             ::"r"(peer[c] + lo), "d"(v0), "d"(v1), "r"(peer[c] + my_bar) : "memory");
          }
        }
        double* gdst = (op.gmask & (1 << q)) ? S : ((op.rmask & (1 << q)) ? R : nullptr);
        if (gdst && row < d) {
          if (colp < d) gdst[(size_t)row * d + colp] = v0;
          if (colp + 1 < d) gdst[(size_t)row * d + colp + 1] = v1;
        }
      }
    }
#ifdef NSERIES_SMALL_PROFILE
    if (tid == 0 && rank == 0) g_small_prof[2 + 3 * o] = clock64();
#endif
#ifdef NSERIES_SMALL_PROFILE
    if (tid == 0 && rank == 0) g_small_prof[3 + 3 * o] = clock64();
#endif
  }
  // no CTA leaves while pushes into it are in flight (every byte addressed to it has landed once
  // its mbarriers completed; st.async carries register values: no closing cluster barrier)
  for (int o = 0; o < n_ops; ++o)
    if (sops[o].push) wait_bar(o);
}

template <int NC>
int launch_cluster_nc(int d, const WarpProgram& prog, const double* A, double* S, double* R, cudaStream_t stream) {
  constexpr int kLSlotD = (64 / NC) * 64;
  const size_t smem = ((size_t)prog.n_slots * kLSlotD + (size_t)(prog.n_rep + 1) * 4096) * sizeof(double) +
                      (size_t)prog.n_ops * (sizeof(ClusterOp) + sizeof(uint64_t));
  if (smem > 227 * 1024) return -1;
  cudaError_t e = cudaFuncSetAttribute(plan_cluster_f64_kernel<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  plan_cluster_f64_kernel<NC><<<NC, 256, smem, stream>>>(d, A, S, R, prog);
  return (int)cudaGetLastError();
}

}  // namespace

nseries_status build_cluster_program(const Program& P, WarpProgram* out) {
  if ((int)P.ops.size() > kMaxBatchedOps) return NSERIES_ERR_UNSUPPORTED_SIZE;
  const int nv = P.n_values;
  std::vector<int> last_use(nv, -1), producer(nv, -1);
  std::vector<char> rep(nv, 0);
  for (int i = 0; i < (int)P.ops.size(); ++i) {
    const Op& op = P.ops[i];
    if (op.gemm) { last_use[op.X] = i; last_use[op.Y] = i; rep[op.Y] = 1; }
    for (int a = 0; a < op.n_aux; ++a) last_use[op.aux[a]] = i;
    for (int j = 0; j < op.n_out; ++j) producer[op.out[j]] = i;
  }
  auto needs_slot = [&](int v) {
    return P.val_kind[v] == V_TEMP || ((v == P.final_S || v == P.final_R) && last_use[v] >= 0);
  };
  // two pools, slots freed after the outputs of the op reading them last are placed
  std::vector<int> slot(nv, -1), last_y_read(nv, -1);
  for (int i = 0; i < (int)P.ops.size(); ++i)
    if (P.ops[i].gemm) last_y_read[P.ops[i].Y] = i;
  std::vector<int> free_l, free_r, slot_read(128, -1);   // slot_read: last op reading the slot as Y
  std::vector<char> csync(P.ops.size(), 0);
  int n_l = 0, n_r = 0, last_push = -1;
  for (int i = 0; i < (int)P.ops.size(); ++i) {
    const Op& op = P.ops[i];
    bool pushes = false;
    for (int j = 0; j < op.n_out; ++j) {
      const int v = op.out[j];
      if (!needs_slot(v)) continue;
      std::vector<int>& fl = rep[v] ? free_r : free_l;
      int sidx;
      if (!fl.empty()) { sidx = fl.back(); fl.pop_back(); }
      else sidx = rep[v] ? n_r++ : n_l++;
      slot[v] = sidx;
      if (rep[v]) {
        // a peer may still read the previous occupant unless it pushed since (see the kernel)
        if (slot_read[sidx] >= 0 && last_push < slot_read[sidx]) csync[i] = 1;
        slot_read[sidx] = std::max(slot_read[sidx], last_y_read[v]);
        pushes = true;
      }
    }
    if (pushes) last_push = i;
    for (int v = 0; v < nv; ++v)
      if (slot[v] >= 0 && ((last_use[v] == i && producer[v] < i) || (producer[v] == i && last_use[v] < 0)))
        (rep[v] ? free_r : free_l).push_back(slot[v]);
  }
  if (n_l >= kWSlotRep || n_r > 127 - kWSlotRep) return NSERIES_ERR_UNSUPPORTED_SIZE;
  WarpProgram& wp = *out;
  wp = WarpProgram{};
  wp.n_slots = n_l;
  wp.n_rep = n_r;
  wp.n_ops = (int)P.ops.size();
  auto code = [&](int v) -> int {
    if (P.val_kind[v] == V_USER_A) return kWSlotA;
    if (P.val_kind[v] == V_IDENT) return kWSlotI;
    if (slot[v] < 0) return kWSlotNone;
    return rep[v] ? kWSlotRep + slot[v] : slot[v];
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
    w.csync = csync[i];
    w.rmask = 0;
    for (int a = 0; a < kMaxAux; ++a) w.aux[a] = a < op.n_aux ? (int8_t)code(op.aux[a]) : 0;
    for (int j = 0; j < kMaxOut; ++j) {
      w.out[j] = j < op.n_out ? (int8_t)code(op.out[j]) : kWSlotNone;
      if (j < op.n_out && op.out[j] == P.final_S) w.gmask |= (int8_t)(1 << j);
      if (j < op.n_out && op.out[j] == P.final_R) w.rmask |= (int8_t)(1 << j);
      w.dalpha[j] = op.alpha[j];
      w.dgamma[j] = op.gamma[j];
      for (int a = 0; a < kMaxAux; ++a) w.dbeta[j][a] = op.beta[j][a];
    }
  }
  return NSERIES_OK;
}

int launch_plan_cluster_f64(int d, const WarpProgram& prog, const double* A, double* S, double* R, void* stream) {
  if (d > 64) return -1;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  static const int nc = std::getenv("NSERIES_SMALL_CLUSTER") ? std::atoi(std::getenv("NSERIES_SMALL_CLUSTER")) : kClusterCtas;
  if (nc == 2) return launch_cluster_nc<2>(d, prog, A, S, R, s);
  if (nc == 4) return launch_cluster_nc<4>(d, prog, A, S, R, s);
  return launch_cluster_nc<8>(d, prog, A, S, R, s);
}

}  // namespace nseries
