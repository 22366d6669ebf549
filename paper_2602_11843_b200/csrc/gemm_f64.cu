// gemm_f64.cu -- FP64 tensor-core GEMM with the fused multi-output epilogue (sm_100a).
//
// acc = X * Y (d x d x d, row-major, binary64) on the FP64 tensor pipe: sm_100a has no
// tcgen05 .kind::f64, so the FP64 tensor path is the warp-level mma.sync m8n8k4 f64
// (SASS DMMA.8x8x4).  Measured on this pool's B200 (profiles/peaks_r01_*):
// DMMA.8x8x4 register loop 37.16 TFLOP/s = 148 SM x 64 FMA/clk x 1.965 GHz, so the engine's
// job is to keep every SM sub-partition issuing one DMMA per 16 cycles.
//
// Design:
//   * CTA tile BM x BN x BK (128x128x32 / 3 stages for d >= 1536, 64x64x16 / 4 stages below),
//     warps tile the CTA as (BM/WM) x (BN/WN) with a WM x WN warp tile of m8n8 blocks
//     (accumulators in registers).
//   * STAGES-deep cp.async ring in shared memory; rows padded (+4 doubles) so every 64-bit
//     fragment load of a half-warp hits 32 distinct banks; register double-buffered fragments
//     (software pipeline) and one barrier per k-tile.
//   * Epilogue: out_j = alpha_j acc + sum_i beta_ji aux_i + gamma_j I for up to 3 aux and 3
//     outputs (every linear combination of the radix kernels).
//   * Grouped rasterisation of the tile grid so concurrently resident CTAs share X row panels
//     and Y column panels in L2.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdint>

#include "internal.h"

namespace nseries {
namespace {

__device__ __forceinline__ void dmma_m8n8k4(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16-byte async copy global->shared with zero fill when !valid.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(valid ? 16 : 0));
}
// same, issued only when `on` (straight-line code: no branch around the copy)
__device__ __forceinline__ void cp_async16_if(void* smem, const void* gmem, bool valid, bool on) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n @p cp.async.cg.shared.global [%0], [%1], 16, %2;\n}\n"
               ::"r"(smem_u32(smem)), "l"(gmem), "r"(valid ? 16 : 0), "r"((int)on));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
struct Cfg {
  static constexpr int kWarpsM = BM / WM, kWarpsN = BN / WN;
  static constexpr int kThreads = kWarpsM * kWarpsN * 32;
  static constexpr int kMI = WM / 8, kNI = WN / 8;
  static constexpr int kLdA = BK + 4;   // padded row (doubles) of the A tile [BM][BK]
  static constexpr int kLdB = BN + 4;   // padded row of the B tile [BK][BN]
  static constexpr int kStageA = BM * kLdA, kStageB = BK * kLdB;
  static constexpr size_t kSmem = (size_t)STAGES * (kStageA + kStageB) * sizeof(double);
  // 8 warps of 32x32 (64 accumulator registers): two CTAs per SM, 16 warps per SM
  static constexpr int kMinBlocks = (kThreads == 256 && WM == 32 && WN == 32) ? 2 : 1;
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool V2, bool SYM>
__global__ void __launch_bounds__(Cfg<BM, BN, BK, WM, WN, STAGES>::kThreads, Cfg<BM, BN, BK, WM, WN, STAGES>::kMinBlocks)
gemm_f64_kernel(const double* __restrict__ X, const double* __restrict__ Y, int d, EpiParams ep) {
  using C = Cfg<BM, BN, BK, WM, WN, STAGES>;
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * C::kStageA;

  // ---- grouped raster: GROUP tile-rows per band
#ifndef NSERIES_F64_GROUP
#define NSERIES_F64_GROUP 8
#endif
  constexpr int GROUP = NSERIES_F64_GROUP;
  const int M = ep.rows > 0 ? ep.rows : d;   // rows of X / aux / outputs (row-sharded chain)
  const int ntm = (M + BM - 1) / BM, ntn = (d + BN - 1) / BN;
  const int pid = blockIdx.x;
  int tm, tn;
  if constexpr (SYM) {
    // symmetric mode (BM == BN): the upper triangle tm <= tn, row after row
    int rem = pid, r = 0;
    while (rem >= ntn - r) { rem -= ntn - r; ++r; }
    tm = r;
    tn = r + rem;
  } else {
    const int band = GROUP * ntn;
    const int first_tm = (pid / band) * GROUP;
    const int gsz = min(ntm - first_tm, GROUP);
    tm = first_tm + (pid % band) % gsz;
    tn = (pid % band) / gsz;
  }
  const int m0 = tm * BM, n0 = tn * BN;
  // symmetric mode: an off-diagonal tile is also stored transposed; inside a diagonal tile the
  // strictly upper elements are stored at both positions and the strictly lower ones are not
  // stored at all, so every output is exactly symmetric
  const bool mirror = SYM && tm != tn;
  const bool diag_tile = SYM && tm == tn;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / C::kWarpsN) * WM, wn0 = (warp % C::kWarpsN) * WN;
  const int g = lane >> 2, t = lane & 3;

  // row k0 of the right factor: Y itself, or (NSERIES_SHARDED_DIRECT) inside the row block that
  // holds rows k0 .. k0+BK-1 (one integer division per k-tile)
  auto y_rows = [&](int k0) -> const double* {
    if (ep.yrows > 0) {
      const int sh = k0 / ep.yrows;
      return ep.yblk[sh] + (size_t)(k0 - sh * ep.yrows) * d;
    }
    return Y + (size_t)k0 * d;
  };
  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * BK;
    double* a = sA + stage * C::kStageA;
    double* b = sB + stage * C::kStageB;
    if constexpr (V2) {
      // A tile: BM rows x BK cols, 2 doubles per chunk
      constexpr int kChunksA = BM * BK / 2;
#pragma unroll
      for (int q = tid; q < kChunksA; q += C::kThreads) {
        int r = q / (BK / 2), c = (q % (BK / 2)) * 2;
        int gr = m0 + r, gc = k0 + c;
        bool ok = gr < M && gc < d;
        cp_async16(a + r * C::kLdA + c, ok ? X + (size_t)gr * d + gc : X, ok);
      }
      const double* Yk = y_rows(k0);   // row k0 of Y (in place: inside its row block)
      constexpr int kChunksB = BK * BN / 2;
#pragma unroll
      for (int q = tid; q < kChunksB; q += C::kThreads) {
        int r = q / (BN / 2), c = (q % (BN / 2)) * 2;
        int gr = k0 + r, gc = n0 + c;
        bool ok = gr < d && gc < d;
        cp_async16(b + r * C::kLdB + c, ok ? Yk + (size_t)r * d + gc : Yk, ok);
      }
    } else {
#pragma unroll 4
      for (int q = tid; q < BM * BK; q += C::kThreads) {
        int r = q / BK, c = q % BK;
        int gr = m0 + r, gc = k0 + c;
        bool ok = gr < M && gc < d;
        cp_async8(a + r * C::kLdA + c, ok ? X + (size_t)gr * d + gc : X, ok);
      }
      const double* Yk = y_rows(k0);
#pragma unroll 4
      for (int q = tid; q < BK * BN; q += C::kThreads) {
        int r = q / BN, c = q % BN;
        int gr = k0 + r, gc = n0 + c;
        bool ok = gr < d && gc < d;
        cp_async8(b + r * C::kLdB + c, ok ? Yk + (size_t)r * d + gc : Yk, ok);
      }
    }
  };

#ifndef NSERIES_F64_NO_SPREAD
  // The k-tile's copies spread over its k-steps (V2 only): part `k` of KK issues the chunks
  // it = k ITA / KK .. (k+1) ITA / KK - 1 of each thread, so the address arithmetic and the
  // LDGSTS issue between the DMMAs instead of in a block of their own at the top of the k-tile.
  // Per-thread invariants are hoisted where a thread's chunks share one column (kThreads a multiple
  // of the chunks per tile row): chunk `it` is then row r0 + it * rows-per-pass at a fixed column.
  constexpr int kCA = BK / 2, kCB = BN / 2;                       // 16-byte chunks per tile row
  // Measured (`profiles/r02_s7_f64_spread_loads.txt`): hoisting gains 1.7% on the 128x128 tiles and
  // loses on the 64x64 tiles at two CTAs per SM (d = 2048: 0.915 -> 0.817), so only the former use it.
#ifndef NSERIES_F64_HOIST64
#define NSERIES_F64_HOIST64 0   // harness: 1 = hoist A's, 2 = B's, 3 = both on the 64x64 tiles
#endif
#ifndef NSERIES_F64_HOIST96
#define NSERIES_F64_HOIST96 0   // harness: 1 = hoist A's on the 96x80 tiles (B's 40 chunks per row do not divide 256)
#endif
  constexpr int kHoistSel = (BM == 128 && BN == 128) ? 3 : (BM == 64 && BN == 64) ? NSERIES_F64_HOIST64
                            : (BM == 96 && BN == 80) ? NSERIES_F64_HOIST96 : 0;
  constexpr bool kHoist = kHoistSel != 0;
  constexpr bool kHoistA = (kHoistSel & 1) && C::kThreads % kCA == 0, kHoistB = (kHoistSel & 2) && C::kThreads % kCB == 0;
  constexpr int kRA = C::kThreads / kCA, kRB = C::kThreads / kCB;   // tile rows per pass
  const int a_r0 = tid / kCA, a_c = (tid % kCA) * 2, b_r0 = tid / kCB, b_c = (tid % kCB) * 2;
  const double* const pA = X + (size_t)(m0 + a_r0) * d + a_c;      // + k0 per k-tile, + it kRA d per chunk
  const int a_rows = M - m0 - a_r0;                                 // chunk `it` is inside A iff it kRA < a_rows
  const bool b_col_ok = n0 + b_c < d;
  const int sa_off = a_r0 * C::kLdA + a_c, sb_off = b_r0 * C::kLdB + b_c;
  auto load_stage_part = [&](int stage, int kt, const double* Ykt, int part, int parts, bool on) {
    const int k0 = kt * BK;
    const double* const Yk = kHoist ? Ykt : y_rows(on ? k0 : 0);
    double* a = sA + stage * C::kStageA;
    double* b = sB + stage * C::kStageB;
    constexpr int kChunksA = BM * BK / 2, kChunksB = BK * BN / 2;
    constexpr int ITA = (kChunksA + C::kThreads - 1) / C::kThreads;
    constexpr int ITB = (kChunksB + C::kThreads - 1) / C::kThreads;
    if constexpr (kHoistA) {
      const bool col_ok = k0 + a_c < d;
#pragma unroll
      for (int it = part * ITA / parts; it < (part + 1) * ITA / parts; ++it) {
        if (kChunksA % C::kThreads == 0 || tid + it * C::kThreads < kChunksA) {
          const bool ok = col_ok && it * kRA < a_rows;
          cp_async16_if(a + sa_off + it * kRA * C::kLdA, ok ? pA + (size_t)(it * kRA) * d + k0 : X, ok, on);
        }
      }
    } else {
#pragma unroll
      for (int it = part * ITA / parts; it < (part + 1) * ITA / parts; ++it) {
        const int q = tid + it * C::kThreads;
        if (kChunksA % C::kThreads == 0 || q < kChunksA) {
          int r = q / kCA, c = (q % kCA) * 2;
          int gr = m0 + r, gc = k0 + c;
          bool ok = gr < M && gc < d;
          cp_async16_if(a + r * C::kLdA + c, ok ? X + (size_t)gr * d + gc : X, ok, on);
        }
      }
    }
    if constexpr (kHoistB) {
      const double* const pB = Yk + (size_t)b_r0 * d + n0 + b_c;
#pragma unroll
      for (int it = part * ITB / parts; it < (part + 1) * ITB / parts; ++it) {
        if (kChunksB % C::kThreads == 0 || tid + it * C::kThreads < kChunksB) {
          const bool ok = b_col_ok && k0 + b_r0 + it * kRB < d;
          cp_async16_if(b + sb_off + it * kRB * C::kLdB, ok ? pB + (size_t)(it * kRB) * d : Yk, ok, on);
        }
      }
    } else {
#pragma unroll
      for (int it = part * ITB / parts; it < (part + 1) * ITB / parts; ++it) {
        const int q = tid + it * C::kThreads;
        if (kChunksB % C::kThreads == 0 || q < kChunksB) {
          int r = q / kCB, c = (q % kCB) * 2;
          int gr = k0 + r, gc = n0 + c;
          bool ok = gr < d && gc < d;
          cp_async16_if(b + r * C::kLdB + c, ok ? Yk + (size_t)r * d + gc : Yk, ok, on);
        }
      }
    }
  };
#endif

  double acc[C::kMI][C::kNI][2];
#pragma unroll
  for (int i = 0; i < C::kMI; ++i)
#pragma unroll
    for (int j = 0; j < C::kNI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int KT = (d + BK - 1) / BK;
  // programmatic dependent launch: everything above overlaps the tail of the previous GEMM of
  // the plan; its outputs (this GEMM's operands and aux values) are read only after the wait.
  // This CTA lets the next GEMM be scheduled right away (it waits for our completion itself).
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }
  cp_async_wait<STAGES - 2>();
  __syncthreads();

  // Software pipeline: fragments of k-step k+1 are loaded from shared memory while the DMMAs
  // of k-step k issue; the next tile's first fragments are loaded right after the single
  // per-tile barrier, so neither LDS latency nor the barrier drains the DMMA pipe.
  constexpr int KK = BK / 4;
  double af[2][C::kMI], bf[2][C::kNI];
  auto load_frags = [&](int buf, const double* a, const double* b, int kk) {
#pragma unroll
    for (int i = 0; i < C::kMI; ++i) af[buf][i] = a[(wm0 + i * 8 + g) * C::kLdA + kk + t];
#pragma unroll
    for (int j = 0; j < C::kNI; ++j) bf[buf][j] = b[(kk + t) * C::kLdB + wn0 + j * 8 + g];
  };
  load_frags(0, sA, sB, 0);

  for (int kt = 0; kt < KT; ++kt) {
    // stage (kt-1) % STAGES was fully consumed before the barrier of iteration kt-1
    const int nk = kt + STAGES - 1;
#ifndef NSERIES_F64_NO_SPREAD
    constexpr bool kSpread = V2;   // -DNSERIES_F64_NO_SPREAD: the copies in one block per k-tile (A/B harness)
#else
    constexpr bool kSpread = false, kHoist = false;
#endif
    // hoisted form: one row-block lookup per k-tile
    const double* const Ynk = (kSpread && kHoist) ? y_rows(nk < KT ? nk * BK : 0) : Y;
    if constexpr (!kSpread) {
      if (nk < KT) load_stage(nk % STAGES, nk);
      cp_async_commit();
    }
    const double* a = sA + (kt % STAGES) * C::kStageA;
    const double* b = sB + (kt % STAGES) * C::kStageB;
#pragma unroll
    for (int k = 0; k < KK; ++k) {
#ifndef NSERIES_F64_NO_SPREAD
      if constexpr (kSpread) {
        load_stage_part(nk % STAGES, nk, Ynk, k, KK, nk < KT);
        if (k == KK - 1) cp_async_commit();
      }
#endif
      if (k == KK - 1) {
        NSERIES_SHAKE_POINT(kt);
        cp_async_wait<STAGES - 2>();   // tile kt+1 has landed
        __syncthreads();
      }
      if (k + 1 < KK) {
        load_frags((k + 1) & 1, a, b, (k + 1) * 4);
      } else if (kt + 1 < KT) {
        load_frags((k + 1) & 1, sA + ((kt + 1) % STAGES) * C::kStageA,
                   sB + ((kt + 1) % STAGES) * C::kStageB, 0);
      }
#pragma unroll
      for (int i = 0; i < C::kMI; ++i)
#pragma unroll
        for (int j = 0; j < C::kNI; ++j) dmma_m8n8k4(acc[i][j], af[k & 1][i], bf[k & 1][j]);
    }
  }
  cp_async_wait<0>();

  // ---- fused epilogue: out_j = alpha_j acc + sum_i beta_ji aux_i + gamma_j I
  const int n_aux = ep.n_aux, n_out = ep.n_out;
  double ssq = 0.0;   // optional fused residual norm (sum of squares of out[sumsq_out])
  int nonfin = 0;     // optional NaN/Inf count of out[nf_out] (NSERIES_CHECK_FINITE)
#pragma unroll
  for (int i = 0; i < C::kMI; ++i) {
    const int row = m0 + wm0 + i * 8 + g;
    if (row >= M) continue;
    const int grow = row + ep.row0;   // global row (identity terms)
    // the row block's aux values are all loaded before its first store: one memory round trip
    // per row block instead of one per 8x8 block (an output may overwrite its own aux element
    // in place, which is why the compiler cannot hoist the loads itself)
    double2 avb[V2 ? C::kNI : 1][kMaxAux];
    if constexpr (V2) {
#pragma unroll
      for (int j = 0; j < C::kNI; ++j) {
        const int col = n0 + wn0 + j * 8 + 2 * t;
#pragma unroll
        for (int x = 0; x < kMaxAux; ++x)
          if (x < n_aux && col < d)
            avb[j][x] = *reinterpret_cast<const double2*>(static_cast<const double*>(ep.aux[x]) +
                                                          (size_t)row * d + col);
      }
    }
#pragma unroll
    for (int j = 0; j < C::kNI; ++j) {
      const int col = n0 + wn0 + j * 8 + 2 * t;
      if (col >= d) continue;
      const size_t off = (size_t)row * d + col;
      if constexpr (V2) {
        const double2 (&av)[kMaxAux] = avb[j];
#pragma unroll
        for (int o = 0; o < kMaxOut; ++o) {
          if (o >= n_out) break;
          double v0 = ep.alpha[o] * acc[i][j][0], v1 = ep.alpha[o] * acc[i][j][1];
#pragma unroll
          for (int x = 0; x < kMaxAux; ++x)
            if (x < n_aux) { v0 += ep.beta[o][x] * av[x].x; v1 += ep.beta[o][x] * av[x].y; }
          if (grow == col) v0 += ep.gamma[o];
          if (grow == col + 1) v1 += ep.gamma[o];
          double* const od = static_cast<double*>(ep.out[o]);
          if (o == ep.nf_out) nonfin += (isfinite(v0) ? 0 : 1) + (isfinite(v1) ? 0 : 1);
          if (!diag_tile) {
            if (o == ep.sumsq_out) ssq += (mirror ? 2.0 : 1.0) * (v0 * v0 + v1 * v1);
            *reinterpret_cast<double2*>(od + off) = make_double2(v0, v1);
            if (mirror) {
              od[(size_t)col * d + row] = v0;
              od[(size_t)(col + 1) * d + row] = v1;
            }
          } else {
            if (row <= col) {
              od[off] = v0;
              od[(size_t)col * d + row] = v0;
              if (o == ep.sumsq_out) ssq += (row == col ? 1.0 : 2.0) * v0 * v0;
            }
            if (row <= col + 1) {
              od[off + 1] = v1;
              od[(size_t)(col + 1) * d + row] = v1;
              if (o == ep.sumsq_out) ssq += (row == col + 1 ? 1.0 : 2.0) * v1 * v1;
            }
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (col + e >= d) continue;
          double av[kMaxAux];
#pragma unroll
          for (int x = 0; x < kMaxAux; ++x)
            if (x < n_aux) av[x] = static_cast<const double*>(ep.aux[x])[off + e];
#pragma unroll
          for (int o = 0; o < kMaxOut; ++o) {
            if (o >= n_out) break;
            double v = ep.alpha[o] * acc[i][j][e];
#pragma unroll
            for (int x = 0; x < kMaxAux; ++x)
              if (x < n_aux) v += ep.beta[o][x] * av[x];
            if (grow == col + e) v += ep.gamma[o];
            if (o == ep.nf_out) nonfin += isfinite(v) ? 0 : 1;
            if (diag_tile && row > col + e) continue;   // written by its mirror element
            const bool twice = mirror || (diag_tile && row < col + e);
            if (o == ep.sumsq_out) ssq += (twice ? 2.0 : 1.0) * v * v;
            static_cast<double*>(ep.out[o])[off + e] = v;
            if (twice) static_cast<double*>(ep.out[o])[(size_t)(col + e) * d + row] = v;
          }
        }
      }
    }
  }
  if (ep.sumsq) {
#pragma unroll
    for (int off2 = 16; off2 > 0; off2 >>= 1) ssq += __shfl_xor_sync(0xffffffffu, ssq, off2);
    if ((threadIdx.x & 31) == 0 && ssq != 0.0) atomicAdd(ep.sumsq, ssq);
  }
  if (ep.nonfinite) {
    // symmetric diagonal tiles count both mirror positions' values once each (a value computed
    // for row > col is discarded but equals its mirror), so the count is of computed values
#pragma unroll
    for (int off2 = 16; off2 > 0; off2 >>= 1) nonfin += __shfl_xor_sync(0xffffffffu, nonfin, off2);
    if ((threadIdx.x & 31) == 0 && nonfin) atomicAdd(ep.nonfinite, nonfin);
  }
}

// Degenerate epilogue without a product (k = 1 identity, elided k = 2 binary, R copy).
__global__ void axpby_f64_kernel(int d, EpiParams ep) {
  const size_t n = (size_t)(ep.rows > 0 ? ep.rows : d) * d;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < n;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int row = (int)(idx / d) + ep.row0, col = (int)(idx % d);
    for (int o = 0; o < ep.n_out; ++o) {
      double v = 0.0;
      for (int x = 0; x < ep.n_aux; ++x) v += ep.beta[o][x] * static_cast<const double*>(ep.aux[x])[idx];
      if (row == col) v += ep.gamma[o];
      static_cast<double*>(ep.out[o])[idx] = v;
      if (ep.sumsq && o == ep.sumsq_out) atomicAdd(ep.sumsq, v * v);
    }
  }
}

__global__ void identity_f64_kernel(double* I, int d) {
  const size_t n = (size_t)d * d;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < n;
       idx += (size_t)gridDim.x * blockDim.x)
    I[idx] = (idx / d == idx % d) ? 1.0 : 0.0;
}

// Launch with the programmatic-stream-serialization attribute (PDL): the kernel may start while
// the previous kernel on the stream drains; it synchronises with griddepcontrol.wait before
// touching that kernel's outputs.  NSERIES_PDL=0 launches without it (A/B harness).
template <typename Kern, typename... Args>
int launch_pdl(Kern kern, int grid, int threads, size_t smem, cudaStream_t s, Args... args) {
  static const bool pdl = !(std::getenv("NSERIES_PDL") && std::atoi(std::getenv("NSERIES_PDL")) == 0);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return (int)cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool V2, bool SYM>
int launch_cfg_t(const double* X, const double* Y, int d, const EpiParams& ep, cudaStream_t s) {
  using C = Cfg<BM, BN, BK, WM, WN, STAGES>;
  auto kern = gemm_f64_kernel<BM, BN, BK, WM, WN, STAGES, V2, SYM>;
  if (int e = smem_attr_once<gemm_f64_kernel<BM, BN, BK, WM, WN, STAGES, V2, SYM>>((int)C::kSmem)) return e;
  const int nt = (d + BM - 1) / BM;
  static_assert(!SYM || BM == BN, "symmetric mode assumes square tiles");
  const int M = ep.rows > 0 ? ep.rows : d;
  const int tiles = SYM ? nt * (nt + 1) / 2 : ((M + BM - 1) / BM) * ((d + BN - 1) / BN);
  return launch_pdl(kern, tiles, C::kThreads, C::kSmem, s, X, Y, d, ep);
}

// the symmetric variant is a separate instantiation: the general kernel is unchanged by it
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool V2>
int launch_cfg(const double* X, const double* Y, int d, const EpiParams& ep, cudaStream_t s) {
  return ep.sym ? launch_cfg_t<BM, BN, BK, WM, WN, STAGES, V2, true>(X, Y, d, ep, s)
                : launch_cfg_t<BM, BN, BK, WM, WN, STAGES, V2, false>(X, Y, d, ep, s);
}

}  // namespace

#ifndef NSERIES_F64_BK64
#define NSERIES_F64_BK64 16   // k-tile and stages of the 64x64 configuration
#define NSERIES_F64_ST64 4
#endif
constexpr int kBK64 = NSERIES_F64_BK64, kST64 = NSERIES_F64_ST64;

int launch_gemm_f64(const double* X, const double* Y, int d, const EpiParams& ep, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  bool v2 = (d % 2 == 0) && ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) % 16 == 0);
  for (int i = 0; i < ep.n_aux; ++i) v2 = v2 && reinterpret_cast<uintptr_t>(ep.aux[i]) % 16 == 0;
  for (int i = 0; i < ep.n_out; ++i) v2 = v2 && reinterpret_cast<uintptr_t>(ep.out[i]) % 16 == 0;
  if (ep.yrows > 0) {
    if (ep.sym || ep.yrows % 32 != 0 || (d + ep.yrows - 1) / ep.yrows > kMaxShards) return (int)cudaErrorInvalidValue;
    for (int i = 0; i < (d + ep.yrows - 1) / ep.yrows; ++i) v2 = v2 && reinterpret_cast<uintptr_t>(ep.yblk[i]) % 16 == 0;
  }
  // Tile choice: 32x32 for small whole matrices (below), else by modelled efficiency 128x128
  // (1 CTA/SM) vs 64x64 (2 CTAs/SM) over 148 SMs (NSERIES_F64_TILE = 1 / 3 / 4 forces one,
  // harness only).
  if (ep.sym && ep.rows > 0 && ep.rows != d) return (int)cudaErrorInvalidValue;
  const int M = ep.rows > 0 ? ep.rows : d;
  const double nb = std::ceil(d / 128.0), ns = std::ceil(d / 64.0);
  const double mb = std::ceil(M / 128.0), ms = std::ceil(M / 64.0);
  const double tb = ep.sym ? nb * (nb + 1) / 2 : mb * nb, ts = ep.sym ? ns * (ns + 1) / 2 : ms * ns;
  // Model fitted to tools/time_f64_tiles.py (fraction of the DMMA peak per tile config):
  // 128x128 tiles run one CTA per SM at ~0.935 with whole-wave quantisation; 64x64 tiles run
  // two CTAs per SM (~0.87 together, ~0.73 for a lone CTA) and, from two waves up, fill the
  // tail well enough that ~0.87 holds (d = 2048: 0.87 measured vs 0.79 for 128x128).
  double eb = 0.935 * tb / (std::ceil(tb / 148.0) * 148.0);
  double es;
  if (ts >= 2 * 296) es = 0.87;
  else if (ts > 148) es = (ts / 148.0) / (2.0 * std::ceil(ts / 296.0) / 0.87);
  else es = 0.73 * ts / 148.0;
  static const int force = std::getenv("NSERIES_F64_TILE") ? std::atoi(std::getenv("NSERIES_F64_TILE")) : 0;
  // 32x32 tiles (4 warps of 16x16, several CTAs per SM) win for whole matrices up to d ~ 1470
  // except where 64x64 tiles fill exactly one wave (d ~ 768: 144 tiles): measured
  // (`profiles/r01_f64_tile_choice.txt`) 0.27 -> 0.46 of peak at d = 500, 0.72 -> 0.75 at 1024
  // (row blocks of the sharded chain: same rule on the block's M x d area)
  bool small32 = !ep.sym && (double)M * d <= 1472.0 * 1472.0 && !(M == d && d > 704 && d <= 800);
  // Whole even-d matrices (the spread-copy kernels, session 7) choose by a model refitted to
  // `profiles/r02_s7_tile_model.txt`: 128x128 at (0.90 + 0.065 d/3072, capped 0.965) x whole-wave
  // fill; 64x64 as pairs of CTAs per SM -- an SM with c = ceil(tiles/148) tiles runs floor(c/2)
  // pairs at 0.92 and a last lone tile at 0.75 (within 0.03 of all 15 measured sizes; +0.025
  // from ~3.5 waves up, where dynamic scheduling smooths the tail); 32x32 at
  // min(0.73, 0.00116 d - 0.23) up to d = 1472.  Sharded row blocks, symmetric mode and odd d
  // keep the rules above.
  if (v2 && !ep.sym && M == d) {
    eb = std::min(0.965, 0.90 + 0.065 * d / 3072.0) * tb / (std::ceil(tb / 148.0) * 148.0);
    const double c = std::ceil(ts / 148.0);
    const double t = std::floor(c / 2.0) * (2.0 / 0.92) + (std::fmod(c, 2.0) > 0.5 ? 1.0 / 0.75 : 0.0);
    es = (ts / 148.0) / t + (ts >= 1000.0 ? 0.025 : 0.0);
    const double e32 = d <= 1472 ? std::min(0.73, 0.00116 * d - 0.23) : 0.0;
    small32 = e32 >= std::max(es, eb);
  }
#ifdef NSERIES_F64_TILE_EXPERIMENTS
  if (v2 && !ep.sym) {
    if (force == 10) return launch_cfg_t<128, 64, 16, 32, 32, 3, true, false>(X, Y, d, ep, s);
    if (force == 12) return launch_cfg_t<128, 128, 16, 32, 32, 4, true, false>(X, Y, d, ep, s);
    if (force == 13) return launch_cfg_t<64, 128, 16, 32, 32, 3, true, false>(X, Y, d, ep, s);
    if (force == 14) return launch_cfg_t<128, 128, 32, 32, 32, 3, true, false>(X, Y, d, ep, s);
    if (force == 15) return launch_cfg_t<128, 64, 32, 32, 32, 2, true, false>(X, Y, d, ep, s);
    if (force == 22) return launch_cfg_t<128, 128, 16, 64, 32, 6, true, false>(X, Y, d, ep, s);
    if (force == 16) return launch_cfg_t<96, 80, 32, 24, 40, 3, true, false>(X, Y, d, ep, s);
    if (force == 17) return launch_cfg_t<80, 96, 32, 40, 24, 3, true, false>(X, Y, d, ep, s);
    if (force == 19) return launch_cfg_t<96, 80, 32, 48, 40, 3, true, false>(X, Y, d, ep, s);
  }
#endif
  // One wave of 96x80 tiles (8 warps of 24x40, BK 16, 4 stages, one CTA per SM) where a whole
  // matrix cuts into <= 148 of them that fill >= 86% of the 148 SMs' tile area: d = 989..1040,
  // i.e. config 2 (d = 1024: 11 x 13 = 143 tiles, fill 0.92).  The 32x32 tiles need 1.4 waves
  // of 5 CTAs per SM there.  Measured (`profiles/r02_s7_cfg2_single_wave.txt`): plain product
  // 0.758 -> 0.785 of the DMMA peak, x9^3 1.142 -> 1.107 ms, bit-identical results (every tile
  // shape sums k in the same order).  NSERIES_F64_TILE = 20 forces it (harness only).
  const double t1 = std::ceil(M / 96.0) * std::ceil(d / 80.0);
  const bool wave1 = v2 && !ep.sym && M == d && t1 <= 148.0 && (double)M * d >= 0.86 * 148.0 * 96.0 * 80.0;
  if (force == 20 || (force == 0 && wave1)) {
    if (!v2 || ep.sym) return (int)cudaErrorInvalidValue;
    return launch_cfg_t<96, 80, 16, 24, 40, 4, true, false>(X, Y, d, ep, s);
  }
  if (force == 4 || (force == 0 && small32)) {
    if (ep.sym) return (int)cudaErrorInvalidValue;
    return v2 ? launch_cfg_t<32, 32, 16, 16, 16, 4, true, false>(X, Y, d, ep, s)
              : launch_cfg_t<32, 32, 16, 16, 16, 4, false, false>(X, Y, d, ep, s);
  }
  if (force == 1 || force == 2 || (force == 0 && eb >= es)) {
    // BK 16 / 4 stages since the copies are spread over the k-steps (session 7: x15^3 70.01 ->
    // 69.64 ms against BK 32 / 3 stages, 6 stages no better); NSERIES_F64_TILE = 2 forces the old shape
    if (force == 2)
      return v2 ? launch_cfg<128, 128, 32, 64, 32, 3, true>(X, Y, d, ep, s)
                : launch_cfg<128, 128, 32, 64, 32, 3, false>(X, Y, d, ep, s);
    return v2 ? launch_cfg<128, 128, 16, 64, 32, 4, true>(X, Y, d, ep, s)
              : launch_cfg<128, 128, 16, 64, 32, 4, false>(X, Y, d, ep, s);
  }
  return v2 ? launch_cfg<64, 64, kBK64, 32, 16, kST64, true>(X, Y, d, ep, s)
            : launch_cfg<64, 64, kBK64, 32, 16, kST64, false>(X, Y, d, ep, s);
}

int launch_axpby_f64(int d, const EpiParams& ep, void* stream) {
  const size_t n = (size_t)d * d;
  int blocks = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
  axpby_f64_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(d, ep);
  return (int)cudaGetLastError();
}

int launch_identity_f64(double* I, int d, void* stream) {
  const size_t n = (size_t)d * d;
  int blocks = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
  identity_f64_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(I, d);
  return (int)cudaGetLastError();
}

}  // namespace nseries
