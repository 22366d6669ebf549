// plan_cluster2d.cu -- whole-plan kernel for one small fp64 matrix (d <= 64, config 1 of
// BASELINE.json) on a 2-D cluster of CTAs.
//
// CTA (r, c) of an RB x CB cluster computes block (r, c) -- rows [r*RPC, +RPC), columns
// [c*CPC, +CPC) -- of every product of the compiled op list (the same fused
// ops as the tiled engine, mu_m + 2 products per radix-m step).  A product's block needs the
// left factor's rows r*RPC.. (all 64 columns) and the right factor's columns c*CPC.. (all 64
// rows), so each value lives where it is read:
//   * read as a left factor  -> "row view"   RPC x 64, replicated in the CTA's row group,
//   * read as a right factor -> "column view" 64 x CPC, replicated in its column group,
//   * read only as an epilogue term -> the CTA's own RPC x CPC block.
// The epilogue stores its block locally and pushes it with st.async into the row peers' row
// views (CB - 1 copies) and the column peers' column views (RB - 1 copies); each push completes
// on the receiver's mbarrier of that op, so a CTA starts op i once the bytes of the last pushing
// op have landed and the mainloop reads only local shared memory.  Against the 1-D row split
// (plan_small.cu, 7 copies of every right factor) this cuts the DSMEM traffic per value from 7
// to 1 (left) / 3 (right) block copies at RB x CB = 4 x 2.
//
// Slot reuse: a pushed slot may be rewritten only after every peer finished reading the old
// value; that holds once the same peer group has pushed again since the old value's last read
// (the pushes follow the pusher's mainloop).  build_cluster2d_program marks ops where no such
// push lies in between (`csync`: full cluster barrier before their pushes).
#include <memory>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "internal.h"

namespace nseries {
namespace {

#ifdef NSERIES_C2_PROFILE
__device__ long long g_c2_prof[256];   // harness-only (tools/c2_probe.cu): per-op phase clocks
#endif

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp8(double* smem, const double* g, bool ok) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(g), "r"(ok ? 8 : 0));
}
__device__ __forceinline__ void cp16(double* smem, const double* g, bool ok) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "r"(ok ? 16 : 0));
}

// row view (RPC x 64): fragment loads read rows g, columns 4s + t -> XOR-swizzle in 4s
__device__ __forceinline__ int swz_row(int r, int c) { return r * 64 + (c ^ (4 * ((r & 3) ^ ((r & 1) << 1)))); }
// column view / own block (rows x 32): fragment loads read rows 4s + t, columns 8j + g.  A
// double's bank pair is set by its column mod 16 (a 32-double row spans 64 banks), so the XOR
// moves the four rows of a k-step to the four 4-column groups: each half-warp hits 16 distinct
// bank pairs
__device__ __forceinline__ int swz_col(int r, int c) { return r * 32 + (c ^ (4 * (r & 3))); }

struct C2Dev {                      // an op with resolved shared-memory offsets (doubles)
  int kind, n_aux, n_out, gmask, rmask, csync, wait_bar, tx;
  int x, y;
  int aux_kind[kMaxAux], aux_off[kMaxAux];
  int out_row[kMaxOut], out_col[kMaxOut], out_own[kMaxOut];
  int push_row, push_col, pad[2];
  double alpha[kMaxOut], beta[kMaxOut][kMaxAux], gamma[kMaxOut];
};

template <int RB, int CB>
__global__ void __cluster_dims__(RB * CB, 1, 1) __launch_bounds__(256, 1)
plan_cluster2d_f64_kernel(int d, const double* __restrict__ A, double* __restrict__ S, double* __restrict__ R,
                          const __grid_constant__ C2Program prog) {
  constexpr int NC = RB * CB, RPC = 64 / RB, CPC = 64 / CB;
  constexpr int kRowD = RPC * 64, kColD = 64 * CPC, kOwnD = RPC * CPC;
  static_assert(RPC == 16 && CPC == 32, "8 warps tile a 16 x 32 block with m8n8 tiles");
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double smc[];
  const int rank = (int)cluster.block_rank();
  const int rb = rank / CB, cb = rank % CB;
  const int r0 = rb * RPC, c0 = cb * CPC;
  const int n_ops = prog.n_ops;
  const int col_base = prog.n_row * kRowD, own_base = col_base + prog.n_col * kColD;
  const int ops_base = own_base + prog.n_own * kOwnD;
  C2Dev* const sops = reinterpret_cast<C2Dev*>(smc + ops_base);
  uint64_t* const bars = reinterpret_cast<uint64_t*>(sops + n_ops);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int mt = warp >> 2, nt = warp & 3;          // this warp's 8 x 8 tile of the 16 x 32 block
  auto row_off = [&](int slot) { return slot * kRowD; };
  auto col_off = [&](int slot) { return col_base + slot * kColD; };
  // A into its row view (this CTA's rows, all columns) and column view (all rows, its columns),
  // issued before the op decode so the memory latency overlaps it; column pairs move as one
  // 16-byte copy when d is even (both swizzles keep (2c, 2c+1) adjacent)
  {
    const bool v16 = (d % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
    if (prog.a_row >= 0)
      for (int i = tid; i < kRowD / 2; i += 256) {
        const int rl = i >> 5, c = 2 * (i & 31), r = r0 + rl;
        double* dst = smc + row_off(prog.a_row) + swz_row(rl, c);
        if (v16) {
          const bool ok = r < d && c < d;
          cp16(dst, ok ? A + (size_t)r * d + c : A, ok);
        } else {   // out-of-range elements are zero-filled from a valid dummy address
          const bool ok0 = r < d && c < d, ok1 = r < d && c + 1 < d;
          cp8(dst, ok0 ? A + (size_t)r * d + c : A, ok0);
          cp8(dst + 1, ok1 ? A + (size_t)r * d + c + 1 : A, ok1);
        }
      }
    if (prog.a_col >= 0)
      for (int i = tid; i < kColD / 2; i += 256) {
        const int r = i / (CPC / 2), cl = 2 * (i % (CPC / 2)), c = c0 + cl;
        double* dst = smc + col_off(prog.a_col) + swz_col(r, cl);
        if (v16) {
          const bool ok = r < d && c < d;
          cp16(dst, ok ? A + (size_t)r * d + c : A, ok);
        } else {   // out-of-range elements are zero-filled from a valid dummy address
          const bool ok0 = r < d && c < d, ok1 = r < d && c + 1 < d;
          cp8(dst, ok0 ? A + (size_t)r * d + c : A, ok0);
          cp8(dst + 1, ok1 ? A + (size_t)r * d + c + 1 : A, ok1);
        }
      }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  for (int i = tid; i < n_ops; i += 256) {
    const C2Op& w = prog.ops[i];
    C2Dev o;
    o.kind = w.kind;
    o.n_aux = w.n_aux;
    o.n_out = w.n_out;
    o.gmask = w.gmask;
    o.rmask = w.rmask;
    o.csync = w.csync;
    o.wait_bar = -1;
    o.x = w.x >= 0 ? row_off(w.x) : 0;
    o.y = w.y >= 0 ? col_off(w.y) : 0;
    for (int a = 0; a < kMaxAux; ++a) {
      o.aux_kind[a] = w.aux_kind[a];
      const int sl = a < w.n_aux ? w.aux_slot[a] : 0;
      o.aux_off[a] = w.aux_kind[a] == 0 ? row_off(sl) : (w.aux_kind[a] == 1 ? col_off(sl) : own_base + sl * kOwnD);
    }
    int nr = 0, ncl = 0;
    for (int q = 0; q < kMaxOut; ++q) {
      const bool on = q < w.n_out;
      o.out_row[q] = on && w.out_row[q] >= 0 ? row_off(w.out_row[q]) : -1;
      o.out_col[q] = on && w.out_col[q] >= 0 ? col_off(w.out_col[q]) : -1;
      o.out_own[q] = on && w.out_own[q] >= 0 ? own_base + w.out_own[q] * kOwnD : -1;
      nr += o.out_row[q] >= 0;
      ncl += o.out_col[q] >= 0;
      o.alpha[q] = w.alpha[q];
      o.gamma[q] = w.gamma[q];
      for (int a = 0; a < kMaxAux; ++a) o.beta[q][a] = w.beta[q][a];
    }
    o.push_row = CB > 1 && nr > 0;
    o.push_col = RB > 1 && ncl > 0;
    o.tx = (nr * (CB - 1) + ncl * (RB - 1)) * kOwnD * 8;   // bytes this CTA receives from the op
    sops[i] = o;
  }
  __syncthreads();
  if (tid == 0) {
    int last = -1;
    for (int i = 0; i < n_ops; ++i) {
      sops[i].wait_bar = last;
      if (sops[i].tx) last = i;
      const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bars + i));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(b) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(sops[i].tx) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");   // A (issued first, below)
  uint32_t rpeer[CB], cpeer[RB];            // shared::cluster base of the row / column peers
  {
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(smc));
#pragma unroll
    for (int q = 0; q < CB; ++q)
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rpeer[q]) : "r"(base), "r"(rb * CB + q));
#pragma unroll
    for (int q = 0; q < RB; ++q)
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(cpeer[q]) : "r"(base), "r"(q * CB + cb));
  }
  const uint32_t bar_off = static_cast<uint32_t>(reinterpret_cast<char*>(bars) - reinterpret_cast<char*>(smc));
  auto wait_bar = [&](int b) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bars + b));
    uint32_t done = 0;
#ifdef NSERIES_SHAKE
    // harness builds: bounded, so a protocol bug traps instead of hanging the GPU (the bound
    // costs ~2 us per x9^2 eval at d = 64 -- 16.5 -> 18.5 us -- so the library spins freely)
    for (uint32_t i = 0; !done; ++i) {
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(a) : "memory");
      if (i > (1u << 26)) __trap();
    }
#else
    while (!done)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(a) : "memory");
#endif
  };
  cluster.sync();
  const int rl = 8 * mt + g;                 // this lane's block row (epilogue) / A-fragment row
  const int cl = 8 * nt + 2 * t;             // this lane's block column pair (epilogue)
  const int grow = r0 + rl;
#ifdef NSERIES_C2_PROFILE
  if (tid == 0 && rank == 0) g_c2_prof[0] = clock64();
#endif
  for (int o = 0; o < n_ops; ++o) {
    const C2Dev& op = sops[o];
    NSERIES_SHAKE_POINT(64 * o + 0);
    if (op.wait_bar >= 0 && (o == 0 || sops[o - 1].wait_bar != op.wait_bar)) wait_bar(op.wait_bar);
    __syncthreads();
#ifdef NSERIES_C2_PROFILE
    if (tid == 0 && rank == 0) g_c2_prof[1 + 3 * o] = clock64();
#endif
    constexpr int KS = 8;                    // independent partial accumulators (DMMA latency)
    double part[KS][2];
#pragma unroll
    for (int p = 0; p < KS; ++p) part[p][0] = part[p][1] = 0.0;
    if (op.kind != 0) {
      const bool xi = op.kind == 2, yi = op.kind == 3;
      const double* X = smc + op.x;
      const double* Y = smc + op.y;
      const int bcol = 8 * nt + g;           // B-fragment column (block-local)
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        const int k = 4 * s + t;
        const double a = xi ? ((grow == k && grow < d) ? 1.0 : 0.0) : X[swz_row(rl, k)];
        const double b = yi ? ((k == c0 + bcol && k < d) ? 1.0 : 0.0) : Y[swz_col(k, bcol)];
        dmma884(part[s % KS], a, b);
      }
    }
    double acc[2];
#pragma unroll
    for (int e = 0; e < 2; ++e)
      acc[e] = ((part[0][e] + part[1][e]) + (part[2][e] + part[3][e])) +
               ((part[4][e] + part[5][e]) + (part[6][e] + part[7][e]));
#ifdef NSERIES_C2_PROFILE
    if (tid == 0 && rank == 0) g_c2_prof[2 + 3 * o] = clock64() + (long long)(acc[0] * 0.0);
#endif
    NSERIES_SHAKE_POINT(64 * o + 1);
    if (op.csync) cluster.sync();
    NSERIES_SHAKE_POINT(64 * o + 2);
    const uint32_t my_bar = bar_off + 8u * (uint32_t)o;
    double2 av[kMaxAux];
#pragma unroll
    for (int x = 0; x < kMaxAux; ++x) {
      if (x < op.n_aux) {
        const int k = op.aux_kind[x];
        const int off = k == 0 ? swz_row(rl, c0 + cl) : (k == 1 ? swz_col(grow, cl) : swz_col(rl, cl));
        av[x] = *reinterpret_cast<const double2*>(smc + op.aux_off[x] + off);
      } else {
        av[x] = make_double2(0.0, 0.0);
      }
    }
    const int gcol = c0 + cl;
#pragma unroll
    for (int q = 0; q < kMaxOut; ++q) {
      if (q >= op.n_out) break;
      double v0 = op.alpha[q] * acc[0], v1 = op.alpha[q] * acc[1];
#pragma unroll
      for (int x = 0; x < kMaxAux; ++x) {
        v0 = fma(op.beta[q][x], av[x].x, v0);
        v1 = fma(op.beta[q][x], av[x].y, v1);
      }
      if (grow == gcol && grow < d) v0 += op.gamma[q];
      if (grow == gcol + 1 && grow < d) v1 += op.gamma[q];
      if (op.out_row[q] >= 0) {
        const int off = op.out_row[q] + swz_row(rl, gcol);
        *reinterpret_cast<double2*>(smc + off) = make_double2(v0, v1);
        NSERIES_SHAKE_POINT(64 * o + 3 + q);
#pragma unroll
        for (int cc = 0; cc < CB; ++cc)
          if (cc != cb) {
            const uint32_t pr = rpeer[cc];
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n"
                         ::"r"(pr + 8u * (uint32_t)off), "d"(v0), "d"(v1), "r"(pr + my_bar) : "memory");
          }
      }
      if (op.out_col[q] >= 0) {
        const int off = op.out_col[q] + swz_col(grow, cl);
        *reinterpret_cast<double2*>(smc + off) = make_double2(v0, v1);
        NSERIES_SHAKE_POINT(64 * o + 8 + q);
#pragma unroll
        for (int rr = 0; rr < RB; ++rr)
          if (rr != rb) {
            const uint32_t pr = cpeer[rr];
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n"
                         ::"r"(pr + 8u * (uint32_t)off), "d"(v0), "d"(v1), "r"(pr + my_bar) : "memory");
          }
      }
      if (op.out_own[q] >= 0)
        *reinterpret_cast<double2*>(smc + op.out_own[q] + swz_col(rl, cl)) = make_double2(v0, v1);
      double* gdst = (op.gmask & (1 << q)) ? S : ((op.rmask & (1 << q)) ? R : nullptr);
      if (gdst && grow < d) {
        if (gcol < d) gdst[(size_t)grow * d + gcol] = v0;
        if (gcol + 1 < d) gdst[(size_t)grow * d + gcol + 1] = v1;
      }
    }
#ifdef NSERIES_C2_PROFILE
    if (tid == 0 && rank == 0) g_c2_prof[3 + 3 * o] = clock64();
#endif
  }
  // no CTA leaves while pushes into it are in flight: every byte addressed to this CTA has
  // landed once all its mbarriers completed, and nothing else touches a peer's shared memory
  // (st.async carries register values), so no closing cluster barrier is needed
  NSERIES_SHAKE_POINT(64 * n_ops + 63);
  for (int o = 0; o < n_ops; ++o)
    if (sops[o].tx) wait_bar(o);
#ifdef NSERIES_C2_END_SYNC
  cluster.sync();
#endif
}

template <int RB, int CB>
size_t c2_smem_bytes(const C2Program& prog) {
  constexpr int RPC = 64 / RB, CPC = 64 / CB;
  return ((size_t)prog.n_row * RPC * 64 + (size_t)prog.n_col * 64 * CPC + (size_t)prog.n_own * RPC * CPC) *
             sizeof(double) +
         (size_t)prog.n_ops * (sizeof(C2Dev) + sizeof(uint64_t));
}

template <int RB, int CB>
int launch_c2(int d, const C2Program& prog, const double* A, double* S, double* R, cudaStream_t stream) {
  const size_t smem = c2_smem_bytes<RB, CB>(prog);
  if (smem > 227 * 1024) return -1;
  cudaError_t e = cudaFuncSetAttribute(plan_cluster2d_f64_kernel<RB, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return (int)e;
  plan_cluster2d_f64_kernel<RB, CB><<<RB * CB, 256, smem, stream>>>(d, A, S, R, prog);
  return (int)cudaGetLastError();
}

}  // namespace

nseries_status build_cluster2d_program(const Program& P, C2Program* out) {
  const int n_ops = (int)P.ops.size();
  if (n_ops > kMaxBatchedOps) return NSERIES_ERR_UNSUPPORTED_SIZE;
  const int nv = P.n_values;
  std::vector<char> xrole(nv, 0), yrole(nv, 0), auxu(nv, 0);
  std::vector<int> last_use(nv, -1), producer(nv, -1), last_x(nv, -1), last_y(nv, -1);
  for (int i = 0; i < n_ops; ++i) {
    const Op& op = P.ops[i];
    if (op.gemm) {
      if (op.X == op.Y && P.val_kind[op.X] == V_IDENT) return NSERIES_ERR_INVALID_ARG;
      if (P.val_kind[op.X] != V_IDENT) { xrole[op.X] = 1; last_x[op.X] = i; last_use[op.X] = i; }
      if (P.val_kind[op.Y] != V_IDENT) { yrole[op.Y] = 1; last_y[op.Y] = i; last_use[op.Y] = i; }
    }
    for (int a = 0; a < op.n_aux; ++a) { auxu[op.aux[a]] = 1; last_use[op.aux[a]] = i; }
    for (int j = 0; j < op.n_out; ++j) producer[op.out[j]] = i;
  }
  auto stored = [&](int v) {
    return P.val_kind[v] == V_TEMP || ((v == P.final_S || v == P.final_R) && last_use[v] >= 0);
  };
  std::vector<int> rs(nv, -1), cs(nv, -1), os(nv, -1);
  std::vector<int> free_r, free_c, free_o, rread(128, -1), cread(128, -1);
  int n_r = 0, n_c = 0, n_o = 0;
  auto take = [](std::vector<int>& fl, int& n) {
    if (!fl.empty()) { const int s = fl.back(); fl.pop_back(); return s; }
    return n++;
  };
  C2Program& pr = *out;
  pr = C2Program{};
  pr.a_row = pr.a_col = -1;
  for (int v = 0; v < nv; ++v)
    if (P.val_kind[v] == V_USER_A) {   // A: loaded once, never freed
      if (xrole[v] || auxu[v]) rs[v] = pr.a_row = take(free_r, n_r);
      if (yrole[v]) cs[v] = pr.a_col = take(free_c, n_c);
    }
  int last_rpush = -1, last_cpush = -1;
  std::vector<char> csync(n_ops, 0);
  for (int i = 0; i < n_ops; ++i) {
    const Op& op = P.ops[i];
    bool rp = false, cp = false;
    for (int j = 0; j < op.n_out; ++j) {
      const int v = op.out[j];
      if (!stored(v)) continue;
      if (xrole[v]) {
        const int s = take(free_r, n_r);
        rs[v] = s;
        if (s < 128) {
          if (rread[s] >= 0 && last_rpush < rread[s]) csync[i] = 1;   // a row peer may still read it
          rread[s] = last_x[v];
        }
        rp = true;
      }
      if (yrole[v]) {
        const int s = take(free_c, n_c);
        cs[v] = s;
        if (s < 128) {
          if (cread[s] >= 0 && last_cpush < cread[s]) csync[i] = 1;
          cread[s] = last_y[v];
        }
        cp = true;
      }
      if (!xrole[v] && !yrole[v] && auxu[v]) os[v] = take(free_o, n_o);
    }
    if (rp) last_rpush = i;
    if (cp) last_cpush = i;
    // free what dies here (after this op's outputs are placed: no in-place reuse)
    for (int v = 0; v < nv; ++v) {
      if (P.val_kind[v] == V_USER_A) continue;
      const bool dies = (last_use[v] == i && producer[v] < i) || (producer[v] == i && last_use[v] < 0);
      if (!dies) continue;
      if (rs[v] >= 0) free_r.push_back(rs[v]);
      if (cs[v] >= 0) free_c.push_back(cs[v]);
      if (os[v] >= 0) free_o.push_back(os[v]);
    }
  }
  if (n_r > 127 || n_c > 127 || n_o > 127) return NSERIES_ERR_UNSUPPORTED_SIZE;
  pr.n_ops = n_ops;
  pr.n_row = n_r;
  pr.n_col = n_c;
  pr.n_own = n_o;
  for (int i = 0; i < n_ops; ++i) {
    const Op& op = P.ops[i];
    C2Op& w = pr.ops[i];
    w.kind = !op.gemm ? 0 : (P.val_kind[op.X] == V_IDENT ? 2 : (P.val_kind[op.Y] == V_IDENT ? 3 : 1));
    w.x = op.gemm && w.kind != 2 ? (int16_t)rs[op.X] : (int16_t)-1;
    w.y = op.gemm && w.kind != 3 ? (int16_t)cs[op.Y] : (int16_t)-1;
    if (op.gemm && ((w.kind != 2 && w.x < 0) || (w.kind != 3 && w.y < 0))) return NSERIES_ERR_INVALID_ARG;
    w.n_aux = (int8_t)op.n_aux;
    w.n_out = (int8_t)op.n_out;
    w.csync = csync[i];
    w.gmask = w.rmask = 0;
    for (int a = 0; a < kMaxAux; ++a) {
      w.aux_kind[a] = 0;
      w.aux_slot[a] = 0;
      if (a >= op.n_aux) continue;
      const int v = op.aux[a];
      if (rs[v] >= 0) { w.aux_kind[a] = 0; w.aux_slot[a] = (int16_t)rs[v]; }
      else if (cs[v] >= 0) { w.aux_kind[a] = 1; w.aux_slot[a] = (int16_t)cs[v]; }
      else if (os[v] >= 0) { w.aux_kind[a] = 2; w.aux_slot[a] = (int16_t)os[v]; }
      else return NSERIES_ERR_INVALID_ARG;
    }
    for (int j = 0; j < kMaxOut; ++j) {
      const bool on = j < op.n_out;
      const int v = on ? op.out[j] : -1;
      w.out_row[j] = on ? (int16_t)rs[v] : (int16_t)-1;
      w.out_col[j] = on ? (int16_t)cs[v] : (int16_t)-1;
      w.out_own[j] = on ? (int16_t)os[v] : (int16_t)-1;
      if (on && v == P.final_S) w.gmask |= (int8_t)(1 << j);
      if (on && v == P.final_R) w.rmask |= (int8_t)(1 << j);
      w.alpha[j] = op.alpha[j];
      w.gamma[j] = op.gamma[j];
      for (int a = 0; a < kMaxAux; ++a) w.beta[j][a] = op.beta[j][a];
    }
  }
  return NSERIES_OK;
}

bool cluster2d_fits(const Program& P, int d) {
  if (d > 64 || (int)P.ops.size() > kMaxBatchedOps) return false;
  auto c2 = std::make_unique<C2Program>();
  if (build_cluster2d_program(P, c2.get()) != NSERIES_OK) return false;
  return c2_smem_bytes<4, 2>(*c2) <= 227 * 1024;
}

int launch_plan_cluster2d_f64(int d, const C2Program& prog, const double* A, double* S, double* R, void* stream) {
  if (d > 64) return -1;
  return launch_c2<4, 2>(d, prog, A, S, R, static_cast<cudaStream_t>(stream));
}

}  // namespace nseries
