// internal.h -- library-internal types shared by the plan compiler, the executor and the
// device engines.  Not part of the C ABI (see include/nseries.h).
#pragma once
#include <cstdint>
#include <string>
#include <atomic>
#ifdef __CUDACC__
#include <cuda_runtime.h>
#endif
#include <vector>

#include "../../include/nseries.h"

namespace nseries {

// ---------------------------------------------------------------- kernel circuits (host)
// Coefficients of the radix kernels as the library evaluates them (binary64).
struct Radix15Params {
  double L2[3], R2[3], L3[4], R3[4], L4[5], R4[5], gamma[4];
};
const Radix15Params& radix15_params();
constexpr int kMaxNaiveRadix = 32;   // naive radix-m splitting for 4 <= m <= 32, m != 5, 9, 15
int kernel_mu(int m);            // products of the kernel circuit, -1 if unsupported
bool kernel_exact(int m);
// monomial coefficients of the kernel polynomial (double), evaluated from the circuit
std::vector<double> kernel_poly(int m);

// ---------------------------------------------------------------- plan builder (host)
nseries_status build_plan(int64_t k, nseries_plan_kind kind, const int32_t* radices, int32_t n,
                          uint32_t flags, nseries_plan* out);
nseries_status finalize_plan(nseries_plan* plan, int64_t k, uint32_t flags);
int step_products(int step, bool first, bool last, uint32_t flags);

// ---------------------------------------------------------------- op list (host)
// Every GEMM op computes acc = X * Y (d x d x d) and an epilogue
//   out_j = alpha_j * acc + sum_i beta_ji * aux_i + gamma_j * I        (j < n_out <= 3)
// where aux_i are d x d matrices read at the accumulator tile's coordinates (i < n_aux <= 3).
// A degenerate "AXPBY" op (no product) evaluates the same epilogue with alpha = 0; it only
// occurs for k = 1 or fully elided binary plans.
constexpr int kMaxAux = 3;
constexpr int kMaxOut = 3;

enum ValKind : int { V_USER_A = 0, V_IDENT = 1, V_USER_S = 2, V_USER_R = 3, V_TEMP = 4 };

struct Op {
  bool gemm = true;
  int X = -1, Y = -1;            // value ids (operands)
  int n_aux = 0, n_out = 0;
  int aux[kMaxAux] = {-1, -1, -1};
  int out[kMaxOut] = {-1, -1, -1};
  double alpha[kMaxOut] = {0, 0, 0};
  double beta[kMaxOut][kMaxAux] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  double gamma[kMaxOut] = {0, 0, 0};
  int step = -1;                 // plan step this op belongs to
  const char* tag = "";
};

struct Program {
  std::vector<Op> ops;
  int n_values = 0;              // value ids 0..n_values-1
  std::vector<int> val_kind;     // ValKind per value
  std::vector<int> val_buf;      // workspace slot per V_TEMP value (-1 otherwise)
  int n_slots = 0;               // workspace d x d slots needed
  int final_S = -1, final_R = -1;
  bool needs_identity = false;   // the IDENT value is read from memory (paper counting)
  int products = 0;
  std::vector<int> step_S, step_B; // value ids of (S_n, B_n) after each plan step
};

// Compile a finalized plan into an op list with workspace slot assignment.
// want_R: route the final power/residual into the user's R_out buffer.
nseries_status compile_plan(const nseries_plan& plan, bool want_R, Program* prog);
// Slot assignment allowing an op's outputs to overwrite the operands/aux that die at that op
// (for executors that read all inputs of an op before writing; returns the slot count).
int assign_slots_inplace(const Program& P, const std::vector<bool>& needs_slot,
                         std::vector<int>* slot_of_value, bool inplace = true);
// last op index reading value v (operand or aux), -1 if never read
std::vector<int> value_last_use(const Program& P);

#ifdef __CUDACC__
// Opt a kernel into more than 48 KB of dynamic shared memory once per (kernel, device): the
// attribute is per device, so a process driving several GPUs sets it on each.
template <auto Kern>
inline int smem_attr_once(int bytes) {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return 0;
  const cudaError_t e = cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return (int)e;
  done.fetch_or(bit, std::memory_order_release);
  return 0;
}
#endif

// ---------------------------------------------------------------- device engines
constexpr int kMaxShards = 16;   // row blocks a directly-read right factor may span
struct EpiParams {
  int n_aux, n_out;
  const void* aux[kMaxAux];
  void* out[kMaxOut];
  double alpha[kMaxOut];
  double beta[kMaxOut][kMaxAux];
  double gamma[kMaxOut];
  double* sumsq = nullptr;       // optional: atomically accumulate sum of squares of out[sumsq_out]
  int sumsq_out = -1;
  int sym = 0;                   // symmetric mode: X, Y, aux and outputs are symmetric (polynomials
                                 // of a symmetric A); only tiles on/above the diagonal are computed
                                 // and each off-diagonal output tile is also stored transposed
  int rows = 0;                  // row-sharded chain: X, aux and outputs are `rows` x d row blocks
  int row0 = 0;                  // (0: rows = d) starting at global row row0 (I's diagonal offset)
  int* nonfinite = nullptr;      // NSERIES_CHECK_FINITE: count NaN/Inf entries of out[nf_out]
  int nf_out = -1;
  // NSERIES_SHARDED_DIRECT: the right factor Y is read in place from row blocks of yrows rows
  // (yrows > 0, a multiple of every BK, so a k-tile never straddles two blocks)
  int yrows = 0;
  const double* yblk[kMaxShards] = {};
};
// NSERIES_CHECK_FINITE on paths without a fused count: NaN/Inf entries of a (batch of) rows x d S
int launch_count_nonfinite(nseries_dtype dt, const void* S, int64_t stride, const void* const* S_ptrs, int batch,
                           int rows, int d, int* count, void* stream);

// Batched small-matrix path: the compiled op list with values mapped to shared-memory slots.
constexpr int kMaxBatchedOps = 48;
struct BatchedOp {
  int8_t gemm, X, Y, n_aux, n_out, aux[kMaxAux], out[kMaxOut];
  double alpha[kMaxOut];
  double beta[kMaxOut][kMaxAux];
  double gamma[kMaxOut];
  float falpha[kMaxOut];          // fp32 copies for the fp32 kernel (no per-element F2F)
  float fbeta[kMaxOut][kMaxAux];
  float fgamma[kMaxOut];
};
struct BatchedProgram {
  int n_ops, n_slots, a_slot, ident_slot, s_slot;
  BatchedOp ops[kMaxBatchedOps];
};
// returns 0 on success, -1 if the size is unsupported, else a cudaError_t
int launch_batched(nseries_dtype dt, const void* A, int64_t strideA, const void* const* A_ptrs,
                   void* S, int64_t strideS, void* const* S_ptrs, int batch, int d,
                   const BatchedProgram& prog, void* stream);

// Warp-per-matrix batched fp32 path (batched_warp.cu, d <= 32).  Slot codes: >= 0 warp
// shared-memory slot, kWSlotA the current A_b buffer, kWSlotI the identity (synthesised in
// fragment registers, operands only), kWSlotNone (output not kept in shared memory).
constexpr int kWSlotNone = -1, kWSlotA = -2, kWSlotI = -3;
constexpr int kWSlotRep = 64;   // cluster kernel: code kWSlotRep + i = replicated slot i
struct WarpOp {
  int8_t gemm, X, Y, n_aux, n_out, gmask;   // gmask bit j: output j is the final S (global)
  int8_t rmask;                             // rmask bit j: output j is the final R (global)
  int8_t aux[kMaxAux], out[kMaxOut];
  int8_t csync;                             // cluster kernel: full cluster barrier before the pushes
  float alpha[kMaxOut];
  float beta[kMaxOut][kMaxAux];
  float gamma[kMaxOut];
  double dalpha[kMaxOut];                   // binary64 copies (fp64 shared-memory plan kernel)
  double dbeta[kMaxOut][kMaxAux];
  double dgamma[kMaxOut];
};
struct WarpProgram {
  int n_ops, n_slots;
  unsigned probe_delay_ns;         // harness-only experiments (tools/bw_probe.cu); 0 in the library
  int n_rep;                       // cluster kernel: slots replicated in every CTA (codes >= kWSlotRep)
  WarpOp ops[kMaxBatchedOps];
};
// Map a compiled op list onto the warp kernel's slot codes (in-place slot assignment; the final
// S is stored from the accumulators, and kept in a slot only if a later op reads it).
nseries_status build_warp_program(const Program& P, WarpProgram* wp, bool inplace = true);
int launch_batched_warp_f32(const void* A, int64_t strideA, const void* const* A_ptrs, void* S,
                            int64_t strideS, void* const* S_ptrs, int batch, int d,
                            const WarpProgram& prog, void* stream, int* nonfinite = nullptr);

// fp32 engine (gemm_tf32.cu): operands as tf32 hi/lo planes with leading dimension ldp
// (multiple of 32): X role row-major (hi, lo), Y role transposed (hiT, loT); epilogue planes:
// x (fp32 value), hi, lo, hiT, loT (any may be null).
struct EpiParamsF32 {
  int n_aux, n_out;
  const float* aux[kMaxAux];
  int aux_ld[kMaxAux];
  float* out_x[kMaxOut];
  float* out_hi[kMaxOut];
  float* out_lo[kMaxOut];
  float* out_hiT[kMaxOut];      // transposed operand planes (B role)
  float* out_loT[kMaxOut];
  int out_ld[kMaxOut];          // leading dimension of out_x (operand planes use ldp)
  int ldp;
  int sym;                      // symmetric mode: upper-triangle 256x256 pair tiles only; every
                                // output's x / hi / lo planes are also stored mirrored (no
                                // transposed operand planes: Y^T = Y for symmetric values)
  double alpha[kMaxOut];          // binary64: the epilogue combines in double, rounds once
  double beta[kMaxOut][kMaxAux];
  double gamma[kMaxOut];
  // split-K of the last partial wave (set by launch_gemm_tf32x3 when sk_ws is given): pair tiles
  // >= sk_first are computed as sk_split K ranges; the last CTA of a tile to finish adds the
  // others' partial accumulators (sk_part) in K order and runs the epilogue
  int sk_first, sk_split;
  float* sk_part;
  unsigned* sk_cnt;               // per CTA tile: [arrivals, partials written]
};
// bytes of split-K workspace launch_gemm_tf32x3 may use at size d (0: never splits); the first
// 256 bytes hold counters that must be zero before the first launch (the kernel re-zeroes them)
size_t tf32_splitk_ws_bytes(int d);
// the 128x128-tile variant (gemm_tf32_b128.cu) for small grids; same contract
size_t tf32_splitk_ws_bytes_b128(int d);
int launch_gemm_tf32x3_b128(const float* Xh, const float* Xl, const float* Yh, const float* Yl, int d, int ldp,
                            const EpiParamsF32& ep, void* stream, void* sk_ws = nullptr);
constexpr int kTf32SmallGridMaxD = 1600;   // api.cu: d <= this (and not symmetric) uses the variant
int launch_gemm_tf32x3(const float* Xh, const float* Xl, const float* Yh, const float* Yl, int d, int ldp,
                       const EpiParamsF32& ep, void* stream, void* sk_ws = nullptr);
int launch_split_f32(const float* x, int ld_in, float* hi, float* lo, float* hiT, float* loT, int ld_out,
                     int d, bool identity, void* stream);
int launch_axpby_f32(int d, const EpiParamsF32& ep, void* stream);
inline int padded_ld(int d) { return (d + 31) / 32 * 32; }

// 2-D cluster kernel (plan_cluster2d.cu): CTA (r, c) of an RB x CB cluster owns the 64/RB x
// 64/CB block (r, c) of every product.  A value read as a LEFT factor lives in "row views"
// (the CTA's 64/RB rows, all 64 columns, replicated across its row group), one read as a RIGHT
// factor in "column views" (all rows, the CTA's 64/CB columns, replicated across its column
// group), an aux-only value in an own-block slot.  Slot indices per pool, -1 = none.
struct C2Op {
  int8_t kind, n_aux, n_out, gmask, rmask, csync;   // kind: 0 axpby, 1 gemm, 2 X = I, 3 Y = I
  int8_t aux_kind[kMaxAux];                         // 0 row view, 1 column view, 2 own block
  int16_t x, y;                                     // row-view slot of X, column-view slot of Y
  int16_t aux_slot[kMaxAux];
  int16_t out_row[kMaxOut], out_col[kMaxOut], out_own[kMaxOut];
  double alpha[kMaxOut];
  double beta[kMaxOut][kMaxAux];
  double gamma[kMaxOut];
};
struct C2Program {
  int n_ops, n_row, n_col, n_own;
  int a_row, a_col;                                 // slots A is loaded into (-1: not needed)
  C2Op ops[kMaxBatchedOps];
};
nseries_status build_cluster2d_program(const Program& P, C2Program* out);
// true if the whole program runs as one 4 x 2 cluster launch at this d (op count, shared memory)
bool cluster2d_fits(const Program& P, int d);
int launch_plan_cluster2d_f64(int d, const C2Program& prog, const double* A, double* S, double* R, void* stream);

// Race shaking (harness builds only, -DNSERIES_SHAKE=<seed>; tools/race_shake.py): a seeded
// pseudo-random __nanosleep of up to ~4 us at a quarter of the hand-synchronised protocol points
// (mbarrier waits, DSMEM pushes, TMA / MMA issue, drains, split-K counters, group barriers).  A
// missing wait or barrier shows up as a result that differs from the unshaken build.  Delays
// are per warp (all lanes sleep alike), so warp-synchronous instructions stay converged.
#ifdef __CUDACC__
#ifdef NSERIES_SHAKE
__device__ __forceinline__ void shake_point(unsigned site) {
  unsigned h = (blockIdx.x + 1u) * 0x9E3779B1u ^ ((threadIdx.x >> 5) + 1u) * 0x85EBCA77u ^
               (site + 1u) * 0xC2B2AE3Du ^ (unsigned)(NSERIES_SHAKE) * 0x27D4EB2Fu;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  if ((h & 3u) == 0u) __nanosleep(h >> 20);
}
#define NSERIES_SHAKE_POINT(site) shake_point(site)
#else
#define NSERIES_SHAKE_POINT(site) ((void)0)
#endif
#endif

// fp64: C-side launchers implemented in gemm_f64.cu.  Return cudaError_t as int.
int launch_gemm_f64(const double* X, const double* Y, int d, const EpiParams& ep, void* stream);
int launch_axpby_f64(int d, const EpiParams& ep, void* stream);
int launch_identity_f64(double* I, int d, void* stream);

}  // namespace nseries
