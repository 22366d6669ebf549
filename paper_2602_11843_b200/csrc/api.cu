// api.cu -- C ABI (include/nseries.h): handle, workspace, plan compilation cache and the
// stream executor that launches one fused GEMM kernel per op.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "internal.h"

using namespace nseries;

struct nseries_ctx {
  int device = 0;
  nseries_status sticky = NSERIES_OK;
  // workspace: slots of d x d elements
  void* ws = nullptr;
  size_t ws_bytes = 0;
  // identity matrix (paper counting multiplies by S_1 = I)
  void* ident = nullptr;
  size_t ident_bytes = 0;
  int ident_d = 0;
  nseries_dtype ident_dt = NSERIES_F64;
  // host-API staging
  void* stage = nullptr;
  size_t stage_bytes = 0;
  // compiled programs keyed by plan bytes + want_R
  std::map<std::string, Program> programs;
  nseries_stats stats{};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // nseries_eval_host: the executor records ev_S right after the op that writes the final S,
  // so the device->host copy of S overlaps the plan's trailing product (the final power)
  bool want_ev_S = false;
  cudaEvent_t ev_S = nullptr;
  cudaStream_t copy_stream = nullptr;
  // CUDA-graph cache: one executable graph per (program, d, dtype, buffer pointers)
  cudaStream_t cap_stream = nullptr;
  struct CachedGraph { cudaGraphExec_t exec; int launches; bool nf_fused; };
  std::map<std::string, CachedGraph> graphs;
  // small fp64 single matrices (d <= 64): 0 = one launch of the 4 x 2 cluster kernel when the
  // plan fits (default), 1 = tiled engine (NSERIES_SMALL_MODE, for tests)
  int small_mode = 0;
  // fp32 engine split-K workspace (tail-wave partial accumulators + per-tile counters)
  void* sk_ws = nullptr;
  size_t sk_bytes = 0;
  // row-sharded chain (nseries_eval_sharded): NCCL communicator and the three d x d gather
  // buffers (gathered A, two gathered right operands)
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  void* full = nullptr;
  size_t full_bytes = 0;
  // NSERIES_HOST_ASYNC: two device staging sets, a copy-in stream and per-set events
  void* astage[2] = {nullptr, nullptr};
  size_t astage_bytes = 0;
  int aset = 0;
  cudaStream_t h2d_stream = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_evaldone[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  cudaStream_t last_eval_stream = nullptr;
  cudaStream_t gather_stream = nullptr;      // prefetching gathers run here
  // NSERIES_SHARDED_DIRECT across processes: this rank's arena (plain cudaMalloc, exported by
  // CUDA IPC) holding the row blocks of every value, the peers' arenas mapped over NVLink
  // (index = rank; own entry = arena), and a 1-int buffer the per-op barrier all-reduces
  void* arena = nullptr;
  size_t arena_bytes = 0;
  std::vector<void*> peer_arena;
  int* bar_dev = nullptr;
  cudaEvent_t ev_bar = nullptr;
  cudaEvent_t ev_gready = nullptr, ev_gdone[3] = {nullptr, nullptr, nullptr};
  // NSERIES_CHECK_FINITE: device counter of NaN/Inf entries of S and its pinned host copy;
  // nf_active is set while an eval with the flag enqueues its ops (engines that count in
  // their final epilogue take it and set nf_fused)
  int* nf_dev = nullptr;
  int* nf_host = nullptr;
  int* nf_active = nullptr;
  bool nf_fused = false;
  // NSERIES_SYNC_STATS: one event per plan-step boundary (eager launches)
  std::vector<cudaEvent_t> ev_step;
  bool step_timing = false;
  bool eager = false;   // ops launched directly (not captured): NVTX range per plan step
  // stream-ordered buffer lifetime: recorded after every enqueued evaluation (grow_buffer)
  cudaEvent_t ev_use = nullptr;
  bool use_recorded = false;
  void* ssq = nullptr;   // nseries_solve's per-step residual-norm accumulators
  size_t ssq_bytes = 0;
  int steps_marked = 0;
};

namespace {

nseries_status cuda_fail(nseries_ctx* h, cudaError_t e) {
  if (e == cudaSuccess) return NSERIES_OK;
  if (h) h->sticky = NSERIES_ERR_CUDA;
  std::fprintf(stderr, "[nseries] CUDA error: %s\n", cudaGetErrorString(e));
  return NSERIES_ERR_CUDA;
}

size_t elem_size(nseries_dtype dt) { return dt == NSERIES_F64 ? sizeof(double) : sizeof(float); }

// Handle buffers (workspace, split-K area, identity, gather buffers, staging) are allocated and
// retired in stream order (cudaMallocAsync / cudaFreeAsync on the calling stream): a growing
// buffer's old allocation is freed after the last work that used it -- the stream waits for
// h->ev_use, recorded after every enqueued evaluation -- with no device-wide synchronisation.
void mark_use(nseries_ctx* h, cudaStream_t s) {
  if (!h->ev_use && cudaEventCreateWithFlags(&h->ev_use, cudaEventDisableTiming) != cudaSuccess) return;
  cudaEventRecord(h->ev_use, s);
  h->use_recorded = true;
}
nseries_status grow_buffer(nseries_ctx* h, void** buf, size_t* cur, size_t bytes, cudaStream_t s) {
  if (bytes <= *cur) return NSERIES_OK;
  if (*buf) {
    cudaError_t e = h->use_recorded ? cudaStreamWaitEvent(s, h->ev_use, 0) : cudaSuccess;
    if (e == cudaSuccess) e = cudaFreeAsync(*buf, s);
    if (e != cudaSuccess) return cuda_fail(h, e);
    *buf = nullptr;
    *cur = 0;
  }
  if (cudaMallocAsync(buf, bytes, s) != cudaSuccess) {
    cudaGetLastError();
    *buf = nullptr;
    return NSERIES_ERR_OOM;
  }
  *cur = bytes;
  return NSERIES_OK;
}

nseries_status ensure_ws(nseries_ctx* h, size_t bytes, cudaStream_t s) {
  return grow_buffer(h, &h->ws, &h->ws_bytes, bytes, s);
}

// split-K workspace of the fp32 engine at size d (counters zeroed; the kernel re-zeroes them)
// largest d for the small-grid fp32 variant (NSERIES_TF32_SMALL_MAXD overrides, harness only)
int tf32_small_maxd() {
  static const int v = std::getenv("NSERIES_TF32_SMALL_MAXD") ? std::atoi(std::getenv("NSERIES_TF32_SMALL_MAXD"))
                                                              : kTf32SmallGridMaxD;
  return v;
}

nseries_status ensure_splitk(nseries_ctx* h, int d, cudaStream_t s) {
  const size_t bytes = std::max(tf32_splitk_ws_bytes(d), tf32_splitk_ws_bytes_b128(d));
  if (bytes == 0 || bytes <= h->sk_bytes) return NSERIES_OK;
  nseries_status st = grow_buffer(h, &h->sk_ws, &h->sk_bytes, bytes, s);
  if (st != NSERIES_OK) return st;
  return cuda_fail(h, cudaMemsetAsync(h->sk_ws, 0, bytes, s));   // counters start at zero
}

// NSERIES_CHECK_FINITE: zeroed device counter on the stream (allocated once per handle)
nseries_status begin_check(nseries_ctx* h, cudaStream_t s) {
  if (!h->nf_dev) {
    if (cudaMalloc(&h->nf_dev, sizeof(int)) != cudaSuccess) { cudaGetLastError(); return NSERIES_ERR_OOM; }
    if (cudaMallocHost(&h->nf_host, sizeof(int)) != cudaSuccess) { cudaGetLastError(); return NSERIES_ERR_OOM; }
  }
  return cuda_fail(h, cudaMemsetAsync(h->nf_dev, 0, sizeof(int), s));
}
// read the count back (synchronizes the stream); NONFINITE if any entry was NaN / Inf
nseries_status finish_check(nseries_ctx* h, cudaStream_t s) {
  cudaError_t e = cudaMemcpyAsync(h->nf_host, h->nf_dev, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(h, e);
  h->stats.nonfinite = *h->nf_host;
  return *h->nf_host > 0 ? NSERIES_ERR_NONFINITE : NSERIES_OK;
}
// the paper's product count of a plan (Table 2 counting, no elision)
int paper_products(const nseries_plan& p) {
  int c = 0;
  for (int i = 0; i < p.n_steps; ++i) c += step_products(p.step[i], i == 0, i + 1 == p.n_steps, 0u);
  return c;
}

nseries_status ensure_identity(nseries_ctx* h, int d, nseries_dtype dt, cudaStream_t s) {
  if (h->ident && h->ident_d == d && h->ident_dt == dt) return NSERIES_OK;
  const size_t bytes = dt == NSERIES_F64 ? (size_t)d * d * sizeof(double)
                                          : 2 * (size_t)d * padded_ld(d) * sizeof(float);
  h->ident_bytes = 0;                              // contents change: always re-allocate / rewrite
  nseries_status gst = grow_buffer(h, &h->ident, &h->ident_bytes, bytes, s);
  if (gst != NSERIES_OK) return gst;
  h->ident_d = d;
  h->ident_dt = dt;
  int rc;
  if (dt == NSERIES_F64) {
    rc = launch_identity_f64(static_cast<double*>(h->ident), d, s);
  } else {
    float* hi = static_cast<float*>(h->ident);
    float* lo = hi + (size_t)d * padded_ld(d);
    cudaMemsetAsync(h->ident, 0, bytes, s);
    rc = launch_split_f32(nullptr, 0, hi, lo, nullptr, nullptr, padded_ld(d), d, true, s);
  }
  return cuda_fail(h, (cudaError_t)rc);
}

std::string plan_key(const nseries_plan& p, bool want_R) {
  std::string k(reinterpret_cast<const char*>(&p), sizeof(p));
  k.push_back(want_R ? 'R' : '-');
  return k;
}

nseries_status resolve_plan(const nseries_plan* plan, int64_t k, uint32_t flags, nseries_plan* out) {
  if (!plan) return build_plan(k, NSERIES_PLAN_AUTO, nullptr, 0, flags, out);
  *out = *plan;
  if (out->k != k) return NSERIES_ERR_PLAN_K_MISMATCH;
  return finalize_plan(out, k, plan->flags | (flags & (NSERIES_ALLOW_APPROX)));
}

// fp32: every value has up to five planes -- x (fp32 value: aux reads, returned S/R), hi/lo
// (tf32 operand planes for the left GEMM role, row-major) and hiT/loT (right role,
// transposed: the tcgen05 B operand must be K-major for .kind::tf32).  Planes are d x ldp.
// Slot i < n_slots holds temp value i's planes; slots n_slots..+2 hold the operand planes of
// the user's A, S and R buffers (their x planes are the user buffers, ld = d).
constexpr int kF32Planes = 5;
// NSERIES_SYNC_STATS: record the event of plan step op.step before the first op of the step,
// and an NVTX range per plan step (eager launches only: a captured graph replays without host
// code, so graph evals carry one range around the whole call)
void mark_step(nseries_ctx* h, const Program& P, int i, int i_end, cudaStream_t s) {
  (void)i_end;
  const int st = P.ops[i].step;
  if (i > 0 && P.ops[i - 1].step == st) return;
  if (h->step_timing && st >= 0 && st < (int)h->ev_step.size()) {
    cudaEventRecord(h->ev_step[st], s);
    ++h->steps_marked;
  }
  if (h->eager) {
    char name[64];
    std::snprintf(name, sizeof(name), "nseries step %d (%s)", st, P.ops[i].tag);
    nvtxRangePushA(name);
  }
}
void end_step(nseries_ctx* h, const Program& P, int i, int i_end) {
  const int st = P.ops[i].step;
  if (h->eager && (i + 1 == i_end || P.ops[i + 1].step != st)) nvtxRangePop();
}

// record h->ev_S if op i writes the final S (eval_host overlaps the copy-out of S with the rest)
void mark_final_S(nseries_ctx* h, const Program& P, int i, cudaStream_t s) {
  if (!h->want_ev_S) return;
  const Op& op = P.ops[i];
  for (int j = 0; j < op.n_out; ++j)
    if (op.out[j] == P.final_S) cudaEventRecordWithFlags(h->ev_S, s, cudaEventRecordExternal);
}

size_t f32_ws_bytes(const Program& P, int d) {
  return (size_t)(P.n_slots + 3) * kF32Planes * d * padded_ld(d) * sizeof(float);
}

nseries_status run_program_f32(nseries_ctx* h, const Program& P, const float* A, float* S, float* R,
                               int d, cudaStream_t s, int* launches, bool sym = false) {
  const int ldp = padded_ld(d);
  const size_t plane = (size_t)d * ldp;
  float* ws = static_cast<float*>(h->ws);
  // --- operand roles: X.Y = Y.X (all values are polynomials in A), so each GEMM may put
  // either factor on the left; pick the order that needs the fewest new plane layouts.
  std::vector<int> role(P.n_values, 0);          // bit 0: left (row planes), bit 1: right (T)
  std::vector<std::pair<int, int>> lr(P.ops.size(), {-1, -1});
  const int ident = 1;
  role[ident] = 3;
  for (size_t i = 0; i < P.ops.size(); ++i) {
    const Op& op = P.ops[i];
    if (!op.gemm) continue;
    auto cost = [&](int l, int r) { return ((role[l] & 1) ? 0 : 1) + ((role[r] & 2) ? 0 : 1); };
    int l = op.X, r = op.Y;
    if (cost(op.Y, op.X) < cost(op.X, op.Y)) std::swap(l, r);
    role[l] |= 1;
    role[r] |= sym ? 1 : 2;   // symmetric values: the right factor reads the row-major planes
    lr[i] = {l, r};
  }
  auto slot_of = [&](int v) -> int {
    switch (P.val_kind[v]) {
      case V_USER_A: return P.n_slots;
      case V_USER_S: return P.n_slots + 1;
      case V_USER_R: return P.n_slots + 2;
      case V_TEMP: return P.val_buf[v];
      default: return -1;
    }
  };
  auto planes = [&](int v) -> float* { return ws + (size_t)slot_of(v) * kF32Planes * plane; };
  auto xplane = [&](int v, int* ld) -> float* {
    switch (P.val_kind[v]) {
      case V_USER_A: *ld = d; return const_cast<float*>(A);
      case V_USER_S: *ld = d; return S;
      case V_USER_R: *ld = d; return R;
      case V_TEMP: *ld = ldp; return planes(v);
      default: *ld = ldp; return nullptr;
    }
  };
  float* id_hi = static_cast<float*>(h->ident);
  float* id_lo = id_hi + plane;
  auto hi = [&](int v) { return P.val_kind[v] == V_IDENT ? id_hi : planes(v) + plane; };
  auto lo = [&](int v) { return P.val_kind[v] == V_IDENT ? id_lo : planes(v) + 2 * plane; };
  auto hiT = [&](int v) { return P.val_kind[v] == V_IDENT ? id_hi : planes(v) + (sym ? 1 : 3) * plane; };
  auto loT = [&](int v) { return P.val_kind[v] == V_IDENT ? id_lo : planes(v) + (sym ? 2 : 4) * plane; };
  int nl = 0;
  const int vA = 0;
  if (role[vA]) {   // one-off split of the user's A into the engine's operand planes
    int rc = launch_split_f32(A, d, (role[vA] & 1) ? hi(vA) : nullptr, (role[vA] & 1) ? lo(vA) : nullptr,
                              (role[vA] & 2) ? hiT(vA) : nullptr, (role[vA] & 2) ? loT(vA) : nullptr,
                              ldp, d, false, s);
    if (rc) return cuda_fail(h, (cudaError_t)rc);
    ++nl;
  }
  std::vector<char> needx(P.n_values, 0);
  for (const Op& op : P.ops)
    for (int i = 0; i < op.n_aux; ++i) needx[op.aux[i]] = 1;
  if (P.final_S >= 0) needx[P.final_S] = 1;
  if (P.final_R >= 0) needx[P.final_R] = 1;
  for (size_t i = 0; i < P.ops.size(); ++i) {
    const Op& op = P.ops[i];
    EpiParamsF32 ep{};
    ep.n_aux = op.n_aux;
    ep.n_out = op.n_out;
    ep.ldp = ldp;
    ep.sym = (sym && op.gemm) ? 1 : 0;
    for (int a = 0; a < op.n_aux; ++a) ep.aux[a] = xplane(op.aux[a], &ep.aux_ld[a]);
    for (int j = 0; j < op.n_out; ++j) {
      const int v = op.out[j];
      int ld = ldp;
      float* x = xplane(v, &ld);
      ep.out_x[j] = (needx[v] || !role[v]) ? x : nullptr;
      ep.out_hi[j] = (role[v] & 1) ? hi(v) : nullptr;
      ep.out_lo[j] = (role[v] & 1) ? lo(v) : nullptr;
      ep.out_hiT[j] = (role[v] & 2) ? hiT(v) : nullptr;
      ep.out_loT[j] = (role[v] & 2) ? loT(v) : nullptr;
      ep.out_ld[j] = ld;
      ep.alpha[j] = op.alpha[j];
      ep.gamma[j] = op.gamma[j];
      for (int a = 0; a < kMaxAux; ++a) ep.beta[j][a] = op.beta[j][a];
    }
    mark_step(h, P, (int)i, (int)P.ops.size(), s);
    int rc;
    if (op.gemm) {
      const int l = lr[i].first, r = lr[i].second;
      rc = (!sym && d <= tf32_small_maxd())
               ? launch_gemm_tf32x3_b128(hi(l), lo(l), hiT(r), loT(r), d, ldp, ep, s, h->sk_ws)
               : launch_gemm_tf32x3(hi(l), lo(l), hiT(r), loT(r), d, ldp, ep, s, h->sk_ws);
    } else {
      rc = launch_axpby_f32(d, ep, s);
    }
    if (rc != 0) return cuda_fail(h, (cudaError_t)rc);
    mark_final_S(h, P, (int)i, s);
    end_step(h, P, (int)i, (int)P.ops.size());
    ++nl;
  }
  *launches = nl;
  return NSERIES_OK;
}

// Execute ops [i0, i1) of a compiled fp64 program on the stream; sumsq_op / sumsq_ptr add the
// fused sum-of-squares reduction of output sumsq_out of op sumsq_op.
nseries_status run_program_range(nseries_ctx* h, const Program& P, const void* A, void* S, void* R,
                                 int d, cudaStream_t s, int i0, int i1, int* launches,
                                 int sumsq_op = -1, int sumsq_out = -1, double* sumsq_ptr = nullptr,
                                 bool sym = false) {
  const size_t slot = (size_t)d * d * sizeof(double);
  auto ptr = [&](int v) -> void* {
    switch (P.val_kind[v]) {
      case V_USER_A: return const_cast<void*>(A);
      case V_IDENT: return h->ident;
      case V_USER_S: return S;
      case V_USER_R: return R;
      default: return static_cast<char*>(h->ws) + (size_t)P.val_buf[v] * slot;
    }
  };
  int nl = 0;
  for (int i = i0; i < i1; ++i) {
    const Op& op = P.ops[i];
    EpiParams ep{};
    ep.n_aux = op.n_aux;
    ep.n_out = op.n_out;
    for (int a = 0; a < op.n_aux; ++a) ep.aux[a] = ptr(op.aux[a]);
    for (int j = 0; j < op.n_out; ++j) {
      ep.out[j] = ptr(op.out[j]);
      ep.alpha[j] = op.alpha[j];
      ep.gamma[j] = op.gamma[j];
      for (int a = 0; a < kMaxAux; ++a) ep.beta[j][a] = op.beta[j][a];
    }
    if (i == sumsq_op) {
      ep.sumsq = sumsq_ptr;
      ep.sumsq_out = sumsq_out;
    }
    if (h->nf_active && op.gemm)   // NSERIES_CHECK_FINITE counted in the epilogue writing S
      for (int j = 0; j < op.n_out; ++j)
        if (op.out[j] == P.final_S) {
          ep.nonfinite = h->nf_active;
          ep.nf_out = j;
          h->nf_fused = true;
        }
    ep.sym = sym ? 1 : 0;
    mark_step(h, P, i, i1, s);
    const int rc = op.gemm ? launch_gemm_f64(static_cast<const double*>(ptr(op.X)),
                                             static_cast<const double*>(ptr(op.Y)), d, ep, s)
                           : launch_axpby_f64(d, ep, s);
    if (rc != 0) return cuda_fail(h, (cudaError_t)rc);
    mark_final_S(h, P, i, s);
    end_step(h, P, i, i1);
    ++nl;
  }
  *launches = nl;
  return NSERIES_OK;
}

// Execute a compiled program on the stream.  fp64 with d <= 64: the whole op list runs in one
// launch of the 4 x 2 cluster kernel (plan_cluster2d.cu) when its live set fits shared memory;
// otherwise (and with NSERIES_SMALL_MODE=1) one tiled GEMM launch per op.
nseries_status run_program(nseries_ctx* h, const Program& P, const void* A, void* S, void* R,
                           int d, nseries_dtype dt, cudaStream_t s, int* launches, bool sym = false) {
  if (dt != NSERIES_F64) return NSERIES_ERR_INVALID_ARG;
  if (h->small_mode == 0 && cluster2d_fits(P, d)) {
    // 4 x 2 cluster, each CTA a 16 x 32 block of every product (row / column views, DSMEM pushes)
    auto c2 = std::make_unique<C2Program>();   // ~8 KB: heap, copied into the launch parameters
    if (build_cluster2d_program(P, c2.get()) == NSERIES_OK) {
      const int rc = launch_plan_cluster2d_f64(d, *c2, static_cast<const double*>(A), static_cast<double*>(S),
                                               static_cast<double*>(R), s);
      if (rc == 0) {
        if (h->want_ev_S) cudaEventRecordWithFlags(h->ev_S, s, cudaEventRecordExternal);
        *launches = 1;
        return NSERIES_OK;
      }
      if (rc != -1) return cuda_fail(h, (cudaError_t)rc);
    }
  }
  return run_program_range(h, P, A, S, R, d, s, 0, (int)P.ops.size(), launches, -1, -1, nullptr, sym);
}

}  // namespace

namespace {

// ---------------------------------------------------------------- NCCL (opened at run time)
// The library does not link NCCL: libnccl.so.2 is dlopen'ed on first use (the copy torch has
// loaded if there is one, else the system library), so single-GPU use needs no NCCL at all.
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclBroadcast) broadcast = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
};
NcclApi load_nccl() {
  NcclApi api;
  {
    void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (lib) {
      api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(lib, "ncclGetUniqueId"));
      api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(lib, "ncclCommInitRank"));
      api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(lib, "ncclCommDestroy"));
      api.broadcast = reinterpret_cast<decltype(api.broadcast)>(dlsym(lib, "ncclBroadcast"));
      api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(lib, "ncclGroupStart"));
      api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(lib, "ncclGroupEnd"));
      api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(lib, "ncclGetErrorString"));
      api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(lib, "ncclAllReduce"));
      api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.broadcast && api.group_start &&
               api.group_end && api.error_string && api.all_reduce;
    }
  }
  return api;
}
const NcclApi& nccl() {
  static const NcclApi api = load_nccl();   // thread-safe one-time initialisation
  return api;
}

nseries_status nccl_fail(nseries_ctx* h, ncclResult_t r) {
  if (r == ncclSuccess) return NSERIES_OK;
  std::fprintf(stderr, "[nseries] NCCL error: %s\n", nccl().error_string ? nccl().error_string(r) : "?");
  if (h) h->sticky = NSERIES_ERR_CUDA;
  return NSERIES_ERR_CUDA;
}

void shard_range(int d, int n, int s, int* row0, int* rows) {
  const int q = d / n, r = d % n;
  *row0 = s * q + (s < r ? s : r);
  *rows = q + (s < r ? 1 : 0);
}

// Row-sharded executor (NEXT-3).  Values live as row blocks; before each product the right
// factor is gathered into a full d x d buffer (allgather-v over NCCL, or device copies when
// every shard is local), then every local row block runs the fused-epilogue DMMA GEMM on
// (rows x d) x (d x d) with its identity terms offset by the block's first row.
nseries_status run_sharded(nseries_ctx* h, const Program& P, const double* const* A_sh, double* const* S_sh,
                           double* const* R_sh, int n_local, int first, int nshards, int d, cudaStream_t s,
                           bool want_direct, int* launches, int* gathers, int* prefetched) {
  // over NCCL whenever the handle's communicator matches the shard map (with one rank the
  // broadcasts are all local: the single-GPU test of the collective path); else device copies
  const bool remote = h->comm && nshards == h->nranks * n_local && first == h->rank * n_local;
  int rows_max = 0;
  std::vector<int> row0(nshards), rows(nshards);
  for (int i = 0; i < nshards; ++i) {
    shard_range(d, nshards, i, &row0[i], &rows[i]);
    rows_max = std::max(rows_max, rows[i]);
  }
  const size_t slot = (size_t)rows_max * d;                 // doubles per row-block slot
  const size_t dd = (size_t)d * d;
  double* ws = static_cast<double*>(h->ws);
  double* const A_full = static_cast<double*>(h->full);
  double* const G[2] = {A_full + dd, A_full + 2 * dd};
  double* const ident = static_cast<double*>(h->ident);
  // NSERIES_SHARDED_DIRECT: a product reads its right factor in place from the factor's row
  // blocks (the GEMM's k-tile loads pick the block; no gather, no full copy) when every block
  // is addressable here and the blocks are uniform.  Single process: all shards local.  Across
  // processes (direct_mr): every value's blocks live in the ranks' arenas at the same offsets
  // (per local shard: n_slots value slots + a copy of A), the peers' arenas are mapped over
  // NVLink (nseries_peer_import), and an all-reduce of one int after every op is the barrier
  // that orders a rank's writes before the peers' reads (and the reads before the next write).
  const bool uniform = nshards <= kMaxShards && d % nshards == 0 && (d / nshards) % 32 == 0;
  const int slots_per = P.n_slots + 1;
  const size_t arena_need = (size_t)n_local * slots_per * ((size_t)rows_max * d) * sizeof(double);
  const bool direct_mr = want_direct && remote && uniform && h->arena && h->bar_dev &&
                         (int)h->peer_arena.size() == h->nranks && h->arena_bytes >= arena_need;
  const bool direct = (want_direct && !remote && n_local == nshards && uniform) || direct_mr;
  double* const arena = static_cast<double*>(h->arena);
  // block of value v in the arena based at `base` (local shard index jl of its owner)
  auto arena_blk = [&](double* base, int v, int jl) -> double* {
    const int slot_idx = P.val_kind[v] == V_USER_A ? P.n_slots : P.val_buf[v];
    return base + ((size_t)jl * slots_per + slot_idx) * slot;
  };
  auto addressable = [&](int v) {
    if (!direct) return false;
    const int kd = P.val_kind[v];
    if (kd == V_USER_R && R_sh == nullptr) return false;
    if (direct_mr && (kd == V_USER_S || kd == V_USER_R)) return h->nranks == 1;   // peers' user blocks: gathered
    return true;
  };
  // row block j (local index) of value v
  auto blk = [&](int v, int j) -> double* {
    const int g = first + j;
    if (direct_mr && (P.val_kind[v] == V_USER_A || P.val_kind[v] == V_TEMP)) return arena_blk(arena, v, j);
    switch (P.val_kind[v]) {
      case V_USER_A: return const_cast<double*>(A_sh[j]);
      case V_IDENT: return ident + (size_t)row0[g] * d;
      case V_USER_S: return S_sh[j];
      case V_USER_R: return R_sh ? R_sh[j] : nullptr;
      default: return ws + ((size_t)j * P.n_slots + P.val_buf[v]) * slot;
    }
  };
  int ng = 0, nl = 0, npf = 0;
  // Every gather -- on the critical path or prefetched -- runs on ONE stream (h->gather_stream),
  // so the NCCL collectives of the communicator are issued and executed in the same order on
  // every rank (program order of the op list): no two NCCL calls on one communicator are ever
  // in flight on different streams.  Ordering with the compute stream s is by events only:
  // the gather stream waits for everything issued on s so far (the producer of the value and
  // every earlier reader of the destination buffer), s waits for the gather's completion event
  // before the first reader.
  if (!h->gather_stream && cudaStreamCreateWithFlags(&h->gather_stream, cudaStreamNonBlocking) != cudaSuccess)
    return cuda_fail(h, cudaGetLastError());
  if (!h->ev_gready) {
    cudaError_t e = cudaEventCreateWithFlags(&h->ev_gready, cudaEventDisableTiming);
    for (int b = 0; b < 3 && e == cudaSuccess; ++b) e = cudaEventCreateWithFlags(&h->ev_gdone[b], cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(h, e);
  }
  cudaStream_t const gs = h->gather_stream;
  // gather value v into dst on the gather stream; completion recorded on ev_gdone[b]
  auto gather = [&](int v, double* dst, int b) -> nseries_status {
    ++ng;
    cudaError_t e = cudaEventRecord(h->ev_gready, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(gs, h->ev_gready, 0);
    if (e != cudaSuccess) return cuda_fail(h, e);
    if (!remote) {
      for (int j = 0; j < n_local; ++j) {
        const int g = first + j;
        e = cudaMemcpyAsync(dst + (size_t)row0[g] * d, blk(v, j), (size_t)rows[g] * d * sizeof(double),
                            cudaMemcpyDeviceToDevice, gs);
        if (e != cudaSuccess) return cuda_fail(h, e);
      }
    } else {
      // allgather-v: every shard broadcast from its owner into its rows of the full buffer
      const NcclApi& nc = nccl();
      ncclResult_t r = nc.group_start();
      for (int g = 0; g < nshards && r == ncclSuccess; ++g) {
        const int owner = g / n_local;
        double* rows_dst = dst + (size_t)row0[g] * d;
        const void* src = owner == h->rank ? blk(v, g - first) : rows_dst;
        r = nc.broadcast(src, rows_dst, (size_t)rows[g] * d, ncclFloat64, owner, h->comm, gs);
      }
      const ncclResult_t r2 = nc.group_end();
      nseries_status st = nccl_fail(h, r != ncclSuccess ? r : r2);
      if (st != NSERIES_OK) return st;
    }
    return cuda_fail(h, cudaEventRecord(h->ev_gdone[b], gs));
  };
  // block of value v owned by shard g, wherever it lives (direct modes): this process's block,
  // or -- direct_mr -- the same arena offset in the owner's mapped arena
  auto any_blk = [&](int v, int g) -> const double* {
    const int owner = g / n_local, jl = g - owner * n_local;
    if (!direct_mr || owner == h->rank) return blk(v, g - first);
    if (P.val_kind[v] == V_IDENT) return ident + (size_t)row0[g] * d;
    return arena_blk(static_cast<double*>(h->peer_arena[owner]), v, jl);
  };
  // cross-rank barrier of direct_mr: a one-int all-reduce on the gather stream (the only
  // stream that carries this communicator's collectives), event-ordered with s on both sides
  auto barrier = [&]() -> nseries_status {
    cudaError_t e = cudaEventRecord(h->ev_gready, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(gs, h->ev_gready, 0);
    if (e != cudaSuccess) return cuda_fail(h, e);
    nseries_status st = nccl_fail(h, nccl().all_reduce(h->bar_dev, h->bar_dev, 1, ncclInt32, ncclSum, h->comm, gs));
    if (st != NSERIES_OK) return st;
    e = cudaEventRecord(h->ev_bar, gs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, h->ev_bar, 0);
    return cuda_fail(h, e);
  };
  if (direct_mr) {
    if (!h->ev_bar) {
      cudaError_t e = cudaEventCreateWithFlags(&h->ev_bar, cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_fail(h, e);
    }
    // the peers may still read this arena (last op of their previous eval): meet first; then
    // A's local blocks go into the arena, and nobody reads a peer's A before every copy landed
    nseries_status st = barrier();
    for (int j = 0; j < n_local && st == NSERIES_OK; ++j) {
      const int aval = [&] { for (int v = 0; v < P.n_values; ++v) if (P.val_kind[v] == V_USER_A) return v; return -1; }();
      if (aval < 0) break;
      st = cuda_fail(h, cudaMemcpyAsync(arena_blk(arena, aval, j), A_sh[j], (size_t)rows[first + j] * d * sizeof(double),
                                        cudaMemcpyDeviceToDevice, s));
    }
    if (st == NSERIES_OK) st = barrier();
    if (st != NSERIES_OK) return st;
  }
  // producer op of every value (-1: A, I or never produced)
  std::vector<int> producer(P.n_values, -1);
  for (size_t i = 0; i < P.ops.size(); ++i)
    for (int o = 0; o < P.ops[i].n_out; ++o) producer[P.ops[i].out[o]] = (int)i;
  // full copies: A once, two gathered values (values are immutable: cached by id).  A gather
  // for the NEXT product whose factor already exists runs on the gather stream while the
  // current product computes (prefetch); pending[b] marks a buffer whose gather the main
  // stream has not yet waited for.
  bool a_full = false;
  int cached[2] = {-1, -1}, lru = 0;          // lru: the buffer to overwrite next
  bool pending[3] = {false, false, false};    // gathers into G[0], G[1], A_full not yet awaited on s
  auto cost = [&](int v) {
    if (addressable(v)) return 0;
    const int kd = P.val_kind[v];
    if (kd == V_IDENT) return 0;
    if (kd == V_USER_A) return a_full ? 0 : 1;
    return (cached[0] == v || cached[1] == v) ? 0 : 1;
  };
  // X.Y = Y.X: gather the cheaper factor; on a tie the one produced earlier (prefetchable)
  auto right_of = [&](const Op& op) -> int {
    const int cx = cost(op.X), cy = cost(op.Y);
    if (cx != cy) return cx < cy ? op.X : op.Y;
    return producer[op.X] < producer[op.Y] ? op.X : op.Y;
  };
  auto wait_pending = [&](int b) -> nseries_status {
    if (!pending[b]) return NSERIES_OK;
    pending[b] = false;
    return cuda_fail(h, cudaStreamWaitEvent(s, h->ev_gdone[b], 0));
  };
  auto full_of = [&](int v, const double** out) -> nseries_status {
    const int kd = P.val_kind[v];
    if (kd == V_IDENT) { *out = ident; return NSERIES_OK; }
    if (kd == V_USER_A) {
      if (!a_full) {
        nseries_status st = gather(v, A_full, 2);
        if (st != NSERIES_OK) return st;
        pending[2] = true;
        a_full = true;
      }
      *out = A_full;
      return wait_pending(2);
    }
    for (int b = 0; b < 2; ++b)
      if (cached[b] == v) {
        lru = 1 - b;
        nseries_status st = wait_pending(b);
        *out = G[b];
        return st;
      }
    const int b = lru;                          // earlier readers: ordered by the gather's event wait
    nseries_status st = wait_pending(b);
    if (st == NSERIES_OK) st = gather(v, G[b], b);
    if (st != NSERIES_OK) return st;
    pending[b] = true;
    cached[b] = v;
    lru = 1 - b;
    *out = G[b];
    return wait_pending(b);                     // on the critical path: s waits right away
  };
  for (size_t i = 0; i < P.ops.size(); ++i) {
    const Op& op = P.ops[i];
    int left = op.X, right = op.Y;
    const double* Yf = nullptr;
    int cur_buf = -1;
    const bool in_place = op.gemm && addressable(op.X) && addressable(op.Y);
    if (op.gemm) {
      right = right_of(op);
      left = right == op.X ? op.Y : op.X;
      if (!in_place) {
        nseries_status st = full_of(right, &Yf);
        if (st != NSERIES_OK) return st;
        cur_buf = Yf == G[0] ? 0 : (Yf == G[1] ? 1 : -1);
      }
    }
    // prefetch: the next product's gathered factor, if it exists before this op runs, into
    // the buffer this op does not read (the previous op's reads are ordered by the event)
    if (i + 1 < P.ops.size() && P.ops[i + 1].gemm) {
      const Op& nx = P.ops[i + 1];
      const int r2 = right_of(nx);
      const int b2 = cur_buf == 0 ? 1 : 0;
      if (cost(r2) && P.val_kind[r2] != V_USER_A && producer[r2] < (int)i) {
        // buffer b2's previous gather (if any) must have been consumed by s first: its event is
        // awaited, then the new gather waits for everything s has issued (incl. b2's readers)
        nseries_status st = wait_pending(b2);
        if (st != NSERIES_OK) return st;
        st = gather(r2, G[b2], b2);
        if (st != NSERIES_OK) return st;
        ++npf;
        cached[b2] = r2;
        pending[b2] = true;
        lru = 1 - b2;
      }
    }
    for (int j = 0; j < n_local; ++j) {
      const int g = first + j;
      EpiParams ep{};
      ep.rows = rows[g];
      ep.row0 = row0[g];
      ep.n_aux = op.n_aux;
      ep.n_out = op.n_out;
      for (int a = 0; a < op.n_aux; ++a) ep.aux[a] = blk(op.aux[a], j);
      for (int o = 0; o < op.n_out; ++o) {
        ep.out[o] = blk(op.out[o], j);
        ep.alpha[o] = op.alpha[o];
        ep.gamma[o] = op.gamma[o];
        for (int a = 0; a < kMaxAux; ++a) ep.beta[o][a] = op.beta[o][a];
      }
      if (in_place) {   // every block of the right factor, in row order (no output aliases it:
                        // the op list never writes an operand's buffer in the same op)
        ep.yrows = rows[0];
        for (int g2 = 0; g2 < nshards; ++g2) ep.yblk[g2] = any_blk(right, g2);
      }
      const int rc = op.gemm ? launch_gemm_f64(blk(left, j), Yf, d, ep, s) : launch_axpby_f64(d, ep, s);
      if (rc != 0) return cuda_fail(h, (cudaError_t)rc);
      ++nl;
    }
    if (direct_mr && i + 1 < P.ops.size()) {   // this op's blocks written everywhere before any peer reads them
      nseries_status st = barrier();
      if (st != NSERIES_OK) return st;
    }
  }
  for (int b = 0; b < 3; ++b) {                 // the caller's stream owns everything at exit
    nseries_status st = wait_pending(b);
    if (st != NSERIES_OK) return st;
  }
  *launches = nl;
  *gathers = ng;
  *prefetched = npf;
  return NSERIES_OK;
}

}  // namespace

extern "C" {

static nseries_status eval_batched_impl(nseries_handle h, const void* A, int64_t strideA,
                                        const void* const* A_ptrs, int32_t batch, int32_t d,
                                        int64_t k, const nseries_plan* plan, nseries_dtype dt,
                                        void* S, int64_t strideS, void* const* S_ptrs,
                                        uint32_t flags, void* stream);

const char* nseries_status_string(nseries_status s) {
  switch (s) {
    case NSERIES_OK: return "ok";
    case NSERIES_ERR_INVALID_ARG: return "invalid argument";
    case NSERIES_ERR_UNSUPPORTED_RADIX: return "unsupported radix";
    case NSERIES_ERR_PLAN_K_MISMATCH: return "plan does not reach k";
    case NSERIES_ERR_APPROX_TELESCOPE: return "approximate kernel requires the residual framework (NSERIES_ALLOW_APPROX)";
    case NSERIES_ERR_ALIAS: return "A aliases an output";
    case NSERIES_ERR_OOM: return "out of device memory";
    case NSERIES_ERR_CUDA: return "CUDA error";
    case NSERIES_ERR_NO_DEVICE: return "no sm_100 device";
    case NSERIES_ERR_UNSUPPORTED_SIZE: return "unsupported size";
    case NSERIES_ERR_NONFINITE: return "result has NaN / Inf entries";
  }
  return "unknown status";
}

const char* nseries_version(void) { return "nseries 0.1 (sm_100a; fp64 DMMA engine)"; }

nseries_status nseries_create(nseries_handle* out, int device) {
  if (!out) return NSERIES_ERR_INVALID_ARG;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
    cudaGetLastError();
    return NSERIES_ERR_NO_DEVICE;
  }
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, device) != cudaSuccess) return NSERIES_ERR_NO_DEVICE;
  if (!(p.major == 10 && p.minor == 0)) return NSERIES_ERR_NO_DEVICE;   // sm_100a cubins only
  if (cudaSetDevice(device) != cudaSuccess) return NSERIES_ERR_NO_DEVICE;
  nseries_ctx* h = new nseries_ctx();
  if (const char* m = std::getenv("NSERIES_SMALL_MODE")) h->small_mode = std::atoi(m);
  h->device = device;
  cudaEventCreate(&h->ev0);
  cudaEventCreate(&h->ev1);
  cudaEventCreateWithFlags(&h->ev_S, cudaEventDisableTiming);
  *out = h;
  return NSERIES_OK;
}

nseries_status nseries_destroy(nseries_handle h) {
  if (!h) return NSERIES_ERR_INVALID_ARG;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  if (h->ws) cudaFree(h->ws);
  if (h->sk_ws) cudaFree(h->sk_ws);
  if (h->full) cudaFree(h->full);
  if (h->comm && nccl().ok) nccl().comm_destroy(h->comm);
  if (h->ident) cudaFree(h->ident);
  for (size_t r = 0; r < h->peer_arena.size(); ++r)
    if ((int)r != h->rank && h->peer_arena[r]) cudaIpcCloseMemHandle(h->peer_arena[r]);
  if (h->arena) cudaFree(h->arena);
  if (h->bar_dev) cudaFree(h->bar_dev);
  if (h->ev_bar) cudaEventDestroy(h->ev_bar);
  if (h->stage) cudaFree(h->stage);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->ev_S) cudaEventDestroy(h->ev_S);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  if (h->gather_stream) cudaStreamDestroy(h->gather_stream);
  if (h->h2d_stream) cudaStreamDestroy(h->h2d_stream);
  for (int b = 0; b < 2; ++b) {
    if (h->astage[b]) cudaFree(h->astage[b]);
    if (h->ev_in[b]) cudaEventDestroy(h->ev_in[b]);
    if (h->ev_evaldone[b]) cudaEventDestroy(h->ev_evaldone[b]);
    if (h->ev_out[b]) cudaEventDestroy(h->ev_out[b]);
  }
  if (h->ev_gready) cudaEventDestroy(h->ev_gready);
  if (h->nf_dev) cudaFree(h->nf_dev);
  if (h->ssq) cudaFree(h->ssq);
  if (h->ev_use) cudaEventDestroy(h->ev_use);
  if (h->nf_host) cudaFreeHost(h->nf_host);
  for (cudaEvent_t e : h->ev_step) cudaEventDestroy(e);
  for (cudaEvent_t e : h->ev_gdone)
    if (e) cudaEventDestroy(e);
  for (auto& g : h->graphs) cudaGraphExecDestroy(g.second.exec);
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  delete h;
  return NSERIES_OK;
}

nseries_status nseries_plan_build(int64_t k, nseries_plan_kind kind, const int32_t* radices,
                                  int32_t n_radices, uint32_t flags, nseries_plan* out) {
  return build_plan(k, kind, radices, n_radices, flags, out);
}

nseries_status nseries_plan_finalize(nseries_plan* plan, int64_t k, uint32_t flags) {
  return finalize_plan(plan, k, flags);
}

nseries_status nseries_kernel_info(int32_t m, int32_t* mu, int32_t* exact, double* coeffs,
                                   int32_t* n_coeffs) {
  if (kernel_mu(m) < 0) return NSERIES_ERR_UNSUPPORTED_RADIX;
  if (mu) *mu = kernel_mu(m);
  if (exact) *exact = kernel_exact(m) ? 1 : 0;
  std::vector<double> f = kernel_poly(m);
  if (n_coeffs) {
    int cap = *n_coeffs;
    if (coeffs) {
      if (cap < (int)f.size()) return NSERIES_ERR_INVALID_ARG;
      for (size_t i = 0; i < f.size(); ++i) coeffs[i] = f[i];
    }
    *n_coeffs = (int32_t)f.size();
  }
  return NSERIES_OK;
}

nseries_status nseries_eval(nseries_handle h, const void* A, int32_t d, int64_t k,
                            const nseries_plan* plan, nseries_dtype dt, void* S, void* R_out,
                            uint32_t flags, void* stream) {
  if (!h) return NSERIES_ERR_INVALID_ARG;
  if (h->sticky != NSERIES_OK) return h->sticky;
  if (!A || !S || d < 1 || k < 1) return NSERIES_ERR_INVALID_ARG;
  if (dt != NSERIES_F64 && dt != NSERIES_F32) return NSERIES_ERR_INVALID_ARG;
  if (A == S || (R_out && (A == R_out || S == R_out))) return NSERIES_ERR_ALIAS;
  nseries_plan p;
  nseries_status st = resolve_plan(plan, k, flags, &p);
  if (st != NSERIES_OK) return st;
  if (dt == NSERIES_F32) {
    // fp32: radix-15 residual update in telescoping form R' = I - f + f R (same polynomial,
    // PAPER.md:573; avoids the |Y| ~ kappa cancellation of I - Y' + A Y' in fp32 storage)
    for (int i = 0; i < p.n_steps; ++i)
      if (p.step[i] == 15) p.form[i] = 2;
  }
  const bool want_R = R_out != nullptr;
  if (dt == NSERIES_F32 && d <= 64 && !want_R && !(flags & NSERIES_SYNC_STATS)) {
    // a small fp32 matrix runs the whole plan in ONE launch of the batched kernels (batch 1:
    // warp-group kernel for d <= 32, CTA kernel above) instead of ~2 launches per product of
    // the tiled engine (d = 32: 107 -> 17 us); same radix-15 residual form as the tiled path
    nseries_plan p1 = p;
    p1.flags |= NSERIES_RFORM_TELESCOPE;
    const nseries_status bst = eval_batched_impl(h, A, (int64_t)d * d, nullptr, 1, d, k, &p1, dt, S,
                                                 (int64_t)d * d, nullptr, flags, stream);
    if (bst != NSERIES_ERR_UNSUPPORTED_SIZE) {
      if (bst == NSERIES_OK && h->want_ev_S) cudaEventRecord(h->ev_S, static_cast<cudaStream_t>(stream));
      return bst;
    }
  }
  std::string key = plan_key(p, want_R);
  auto it = h->programs.find(key);
  if (it == h->programs.end()) {
    Program prog;
    st = compile_plan(p, want_R, &prog);
    if (st != NSERIES_OK) return st;
    it = h->programs.emplace(key, std::move(prog)).first;
  }
  const Program& P = it->second;
  cudaSetDevice(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  st = ensure_ws(h, dt == NSERIES_F64 ? (size_t)P.n_slots * d * d * sizeof(double) : f32_ws_bytes(P, d), s);
  if (st == NSERIES_OK && dt == NSERIES_F32) st = ensure_splitk(h, d, s);
  if (st != NSERIES_OK) return st;
  // the 4 x 2 cluster kernel (fp64, d <= 64) synthesises I in its fragments: no identity buffer
  const bool one_launch = dt == NSERIES_F64 && h->small_mode == 0 && cluster2d_fits(P, d);
  if (P.needs_identity && !one_launch) {
    st = ensure_identity(h, d, dt, s);
    if (st != NSERIES_OK) return st;
  }
  const bool timing = (flags & NSERIES_SYNC_STATS) != 0;
  const bool check = (flags & NSERIES_CHECK_FINITE) != 0;
  if (check && (st = begin_check(h, s)) != NSERIES_OK) return st;
  if (timing) {
    while ((int)h->ev_step.size() < p.n_steps) {
      cudaEvent_t e = nullptr;
      if (cudaEventCreate(&e) != cudaSuccess) return cuda_fail(h, cudaGetLastError());
      h->ev_step.push_back(e);
    }
    cudaEventRecord(h->ev0, s);
  }
  h->nf_active = check ? h->nf_dev : nullptr;
  h->nf_fused = false;
  h->step_timing = timing;
  h->steps_marked = 0;
  h->eager = timing || (flags & NSERIES_NO_GRAPH);
  struct Reset {   // per-call executor state, cleared on every return path
    nseries_ctx* h;
    ~Reset() { h->nf_active = nullptr; h->step_timing = false; h->eager = false; }
  } reset{h};
  int launches = 0;
  auto run = [&](cudaStream_t st_) {
    return dt == NSERIES_F64
               ? run_program(h, P, A, S, R_out, d, dt, st_, &launches, (flags & NSERIES_SYMMETRIC) != 0)
               : run_program_f32(h, P, static_cast<const float*>(A), static_cast<float*>(S),
                                 static_cast<float*>(R_out), d, st_, &launches,
                                 (flags & NSERIES_SYMMETRIC) != 0);
  };
  bool replayed = false;
  if (!h->eager) {
    // The op list is replayed as one CUDA graph: the pointers are baked in, so the key holds
    // them; capture runs on a private stream (the caller's may be the legacy NULL stream).
    char ptrs[224];
    std::snprintf(ptrs, sizeof(ptrs), "|%d|%d|%p|%p|%p|%p|%p|%p|%d|%d|%d", d, (int)dt, A, S, R_out, h->ws, h->ident,
                  h->sk_ws, (flags & NSERIES_SYMMETRIC) ? 1 : 0, h->want_ev_S ? 1 : 0, check ? 1 : 0);
    const std::string gkey = key + ptrs;
    auto git = h->graphs.find(gkey);
    if (git == h->graphs.end()) {
      if (h->graphs.size() >= 64) {          // bounded cache: drop everything (stream-ordered)
        cudaStreamSynchronize(s);
        for (auto& g : h->graphs) cudaGraphExecDestroy(g.second.exec);
        h->graphs.clear();
      }
      if (!h->cap_stream && cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
        return cuda_fail(h, cudaGetLastError());
      cudaGraph_t graph = nullptr;
      cudaError_t e = cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal);
      if (e != cudaSuccess) return cuda_fail(h, e);
      st = run(h->cap_stream);
      e = cudaStreamEndCapture(h->cap_stream, &graph);
      if (st != NSERIES_OK) { if (graph) cudaGraphDestroy(graph); return st; }
      if (e != cudaSuccess) return cuda_fail(h, e);
      cudaGraphExec_t exec = nullptr;
      e = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return cuda_fail(h, e);
      git = h->graphs.emplace(gkey, nseries_ctx::CachedGraph{exec, launches, h->nf_fused}).first;
    } else {
      replayed = true;
      launches = git->second.launches;
      h->nf_fused = git->second.nf_fused;
    }
    cudaError_t e = cudaGraphLaunch(git->second.exec, s);
    if (e != cudaSuccess) return cuda_fail(h, e);
  } else {
    st = run(s);
    if (st != NSERIES_OK) return st;
  }
  mark_use(h, s);
  if (check && !h->nf_fused) {   // paths without a fused count: one pass over S
    const int rc = launch_count_nonfinite(dt, S, 0, nullptr, 1, d, d, h->nf_dev, s);
    if (rc != 0) return cuda_fail(h, (cudaError_t)rc);
    ++launches;
  }
  h->stats = nseries_stats{};
  h->stats.products = P.products;
  h->stats.products_exec = P.products;
  h->stats.products_paper = paper_products(p);
  h->stats.launches = launches;
  h->stats.graph_replayed = replayed ? 1 : 0;
  h->stats.n_ops = (int)P.ops.size();
  h->stats.ms_total = 0.f;
  if (timing) {
    cudaEventRecord(h->ev1, s);
    cudaEventSynchronize(h->ev1);
    cudaEventElapsedTime(&h->stats.ms_total, h->ev0, h->ev1);
    // per-step times when the ops ran one launch per op (the single-launch d <= 64 kernel
    // records no step events)
    if (h->steps_marked == p.n_steps) {
      h->stats.n_steps_timed = p.n_steps;
      for (int i = 0; i < p.n_steps; ++i)
        cudaEventElapsedTime(&h->stats.ms_step[i], h->ev_step[i], i + 1 < p.n_steps ? h->ev_step[i + 1] : h->ev1);
    }
  }
  st = cuda_fail(h, cudaGetLastError());
  if (st == NSERIES_OK && check) st = finish_check(h, s);
  return st;
}

nseries_status nseries_eval_host(nseries_handle h, const void* A_host, int32_t d, int64_t k,
                                 const nseries_plan* plan, nseries_dtype dt, void* S_host,
                                 void* R_host, uint32_t flags, void* stream) {
  if (!h || !A_host || !S_host || d < 1 || k < 1) return NSERIES_ERR_INVALID_ARG;
  if (h->sticky != NSERIES_OK) return h->sticky;
  const size_t bytes = (size_t)d * d * elem_size(dt);
  const size_t need = bytes * (R_host ? 3 : 2);
  cudaSetDevice(h->device);
  if (flags & NSERIES_HOST_ASYNC) {
    // pipelined: set b's copy-in waits for the previous evaluation that read set b; that
    // evaluation's successor on set b waits for set b's copy-out
    if (!h->h2d_stream) {
      cudaError_t e = cudaStreamCreateWithFlags(&h->h2d_stream, cudaStreamNonBlocking);
      if (e == cudaSuccess && !h->copy_stream) e = cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking);
      for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
        e = cudaEventCreateWithFlags(&h->ev_in[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_evaldone[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_out[b], cudaEventDisableTiming);
      }
      if (e != cudaSuccess) return cuda_fail(h, e);
      for (int b = 0; b < 2; ++b) {      // recorded once so the first waits are satisfied
        cudaEventRecord(h->ev_evaldone[b], h->h2d_stream);
        cudaEventRecord(h->ev_out[b], h->h2d_stream);
      }
    }
    if (need > h->astage_bytes) {
      nseries_host_sync(h);
      for (int b = 0; b < 2; ++b) {
        if (h->astage[b]) cudaFree(h->astage[b]);
        h->astage[b] = nullptr;
      }
      h->astage_bytes = 0;
      for (int b = 0; b < 2; ++b)
        if (cudaMalloc(&h->astage[b], need) != cudaSuccess) { cudaGetLastError(); return NSERIES_ERR_OOM; }
      h->astage_bytes = need;
    }
    const int b = h->aset;
    h->aset ^= 1;
    char* dA = static_cast<char*>(h->astage[b]);
    char* dS = dA + bytes;
    char* dR = R_host ? dS + bytes : nullptr;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    h->last_eval_stream = s;
    cudaError_t e = cudaStreamWaitEvent(h->h2d_stream, h->ev_evaldone[b], 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dA, A_host, bytes, cudaMemcpyHostToDevice, h->h2d_stream);
    if (e == cudaSuccess) e = cudaEventRecord(h->ev_in[b], h->h2d_stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, h->ev_in[b], 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, h->ev_out[b], 0);
    if (e != cudaSuccess) return cuda_fail(h, e);
    h->want_ev_S = true;
    nseries_status st = nseries_eval(h, dA, d, k, plan, dt, dS, dR, flags & ~(NSERIES_SYNC_STATS | NSERIES_HOST_ASYNC),
                                     stream);
    h->want_ev_S = false;
    if (st != NSERIES_OK) return st;
    e = cudaEventRecord(h->ev_evaldone[b], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->copy_stream, h->ev_S, 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(S_host, dS, bytes, cudaMemcpyDeviceToHost, h->copy_stream);
    if (e == cudaSuccess && R_host) {
      e = cudaStreamWaitEvent(h->copy_stream, h->ev_evaldone[b], 0);
      if (e == cudaSuccess) e = cudaMemcpyAsync(R_host, dR, bytes, cudaMemcpyDeviceToHost, h->copy_stream);
    }
    if (e == cudaSuccess) e = cudaEventRecord(h->ev_out[b], h->copy_stream);
    return cuda_fail(h, e);
  }
  nseries_status st = grow_buffer(h, &h->stage, &h->stage_bytes, need, static_cast<cudaStream_t>(stream));
  if (st != NSERIES_OK) return st;
  char* dA = static_cast<char*>(h->stage);
  char* dS = dA + bytes;
  char* dR = R_host ? dS + bytes : nullptr;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(dA, A_host, bytes, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(h, e);
  // the copy-out of S starts as soon as the op writing S completes (a side stream waits on
  // ev_S recorded inside the executor), overlapping the plan's trailing product
  if (!h->copy_stream && cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking) != cudaSuccess)
    return cuda_fail(h, cudaGetLastError());
  h->want_ev_S = true;
  st = nseries_eval(h, dA, d, k, plan, dt, dS, dR, flags & ~NSERIES_SYNC_STATS, stream);
  h->want_ev_S = false;
  if (st != NSERIES_OK) return st;
  e = cudaStreamWaitEvent(h->copy_stream, h->ev_S, 0);
  if (e != cudaSuccess) return cuda_fail(h, e);
  e = cudaMemcpyAsync(S_host, dS, bytes, cudaMemcpyDeviceToHost, h->copy_stream);
  if (e != cudaSuccess) return cuda_fail(h, e);
  if (R_host) {
    e = cudaMemcpyAsync(R_host, dR, bytes, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(h, e);
  }
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(h, e);
  return cuda_fail(h, cudaStreamSynchronize(h->copy_stream));
}

nseries_status nseries_host_sync(nseries_handle h) {
  if (!h) return NSERIES_ERR_INVALID_ARG;
  cudaSetDevice(h->device);
  cudaError_t e = cudaSuccess;
  for (cudaStream_t st : {h->h2d_stream, h->last_eval_stream, h->copy_stream})
    if (st && e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (!h->last_eval_stream && e == cudaSuccess) e = cudaStreamSynchronize(nullptr);
  return cuda_fail(h, e);
}

static nseries_status eval_batched_impl(nseries_handle h, const void* A, int64_t strideA,
                                        const void* const* A_ptrs, int32_t batch, int32_t d,
                                        int64_t k, const nseries_plan* plan, nseries_dtype dt,
                                        void* S, int64_t strideS, void* const* S_ptrs,
                                        uint32_t flags, void* stream) {
  if (!h) return NSERIES_ERR_INVALID_ARG;
  if (h->sticky != NSERIES_OK) return h->sticky;
  if (batch < 0 || d < 1 || k < 1) return NSERIES_ERR_INVALID_ARG;
  if (dt != NSERIES_F64 && dt != NSERIES_F32) return NSERIES_ERR_INVALID_ARG;
  if ((dt == NSERIES_F32 && d > 64) || (dt == NSERIES_F64 && d > 32)) return NSERIES_ERR_UNSUPPORTED_SIZE;
  nseries_plan p;
  nseries_status st = resolve_plan(plan, k, flags, &p);
  if (st != NSERIES_OK) return st;
  std::string key = plan_key(p, false);
  auto it = h->programs.find(key);
  if (it == h->programs.end()) {
    Program prog;
    st = compile_plan(p, false, &prog);
    if (st != NSERIES_OK) return st;
    it = h->programs.emplace(key, std::move(prog)).first;
  }
  const Program& P = it->second;
  if ((int)P.ops.size() > kMaxBatchedOps) return NSERIES_ERR_UNSUPPORTED_SIZE;
  const bool check = (flags & NSERIES_CHECK_FINITE) != 0;
  WarpProgram wp{};
  nseries_status wst = (dt == NSERIES_F32 && d <= 32) ? build_warp_program(P, &wp) : NSERIES_ERR_UNSUPPORTED_SIZE;
  if (wst != NSERIES_OK && wst != NSERIES_ERR_UNSUPPORTED_SIZE) return wst;
  if (wst == NSERIES_OK) {   // else: the CTA-per-matrix kernel below
    h->stats = nseries_stats{};
    h->stats.products = h->stats.products_exec = P.products;
    h->stats.products_paper = paper_products(p);
    h->stats.n_ops = wp.n_ops;
    if (batch == 0) return NSERIES_OK;
    if ((!A && !A_ptrs) || (!S && !S_ptrs)) return NSERIES_ERR_INVALID_ARG;
    if (A && A == S) return NSERIES_ERR_ALIAS;
    cudaSetDevice(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (check && (st = begin_check(h, s)) != NSERIES_OK) return st;
    // NSERIES_CHECK_FINITE counted in the kernel's final epilogue
    int rc = launch_batched_warp_f32(A, strideA, A_ptrs, S, strideS, S_ptrs, batch, d, wp, stream,
                                     check ? h->nf_dev : nullptr);
    if (rc == -1) return NSERIES_ERR_UNSUPPORTED_SIZE;
    if (rc != 0) return cuda_fail(h, (cudaError_t)rc);
    mark_use(h, s);
    h->stats.launches = 1;
    return check ? finish_check(h, s) : NSERIES_OK;
  }
  BatchedProgram bp{};
  bp.n_ops = (int)P.ops.size();
  bp.a_slot = P.n_slots;
  bp.ident_slot = P.n_slots + 1;
  bp.s_slot = P.n_slots + 2;
  bp.n_slots = P.n_slots + 3;
  auto slot = [&](int v) -> int {
    switch (P.val_kind[v]) {
      case V_USER_A: return bp.a_slot;
      case V_IDENT: return bp.ident_slot;
      case V_USER_S: return bp.s_slot;
      case V_TEMP: return P.val_buf[v];
      default: return -1;
    }
  };
  for (int i = 0; i < bp.n_ops; ++i) {
    const Op& op = P.ops[i];
    BatchedOp& b = bp.ops[i];
    b.gemm = op.gemm ? 1 : 0;
    b.X = op.gemm ? (int8_t)slot(op.X) : 0;
    b.Y = op.gemm ? (int8_t)slot(op.Y) : 0;
    b.n_aux = (int8_t)op.n_aux;
    b.n_out = (int8_t)op.n_out;
    for (int a = 0; a < kMaxAux; ++a) b.aux[a] = a < op.n_aux ? (int8_t)slot(op.aux[a]) : 0;
    for (int j = 0; j < kMaxOut; ++j) {
      b.out[j] = j < op.n_out ? (int8_t)slot(op.out[j]) : 0;
      b.alpha[j] = op.alpha[j];
      b.gamma[j] = op.gamma[j];
      b.falpha[j] = (float)op.alpha[j];
      b.fgamma[j] = (float)op.gamma[j];
      for (int a = 0; a < kMaxAux; ++a) {
        b.beta[j][a] = op.beta[j][a];
        b.fbeta[j][a] = (float)op.beta[j][a];
      }
    }
  }
  h->stats = nseries_stats{};
  h->stats.products = h->stats.products_exec = P.products;
  h->stats.products_paper = paper_products(p);
  h->stats.n_ops = bp.n_ops;
  if (batch == 0) return NSERIES_OK;
  if ((!A && !A_ptrs) || (!S && !S_ptrs)) return NSERIES_ERR_INVALID_ARG;
  if (A && A == S) return NSERIES_ERR_ALIAS;
  cudaSetDevice(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (check && (st = begin_check(h, s)) != NSERIES_OK) return st;
  int rc = launch_batched(dt, A, strideA, A_ptrs, S, strideS, S_ptrs, batch, d, bp, stream);
  if (rc == -1) return NSERIES_ERR_UNSUPPORTED_SIZE;
  if (rc != 0) return cuda_fail(h, (cudaError_t)rc);
  if (check) {   // one pass over the batch's S
    rc = launch_count_nonfinite(dt, S, strideS, S_ptrs, batch, d, d, h->nf_dev, stream);
    if (rc != 0) return cuda_fail(h, (cudaError_t)rc);
  }
  mark_use(h, s);
  h->stats.launches = check ? 2 : 1;
  return check ? finish_check(h, s) : NSERIES_OK;
}

nseries_status nseries_eval_batched_strided(nseries_handle h, const void* A, int64_t strideA,
                                            int32_t batch, int32_t d, int64_t k,
                                            const nseries_plan* plan, nseries_dtype dt, void* S,
                                            int64_t strideS, uint32_t flags, void* stream) {
  if (strideA < (int64_t)d * d || strideS < (int64_t)d * d) return NSERIES_ERR_INVALID_ARG;
  return eval_batched_impl(h, A, strideA, nullptr, batch, d, k, plan, dt, S, strideS, nullptr,
                           flags, stream);
}

nseries_status nseries_eval_batched(nseries_handle h, const void* const* A_ptrs, int32_t batch,
                                    int32_t d, int64_t k, const nseries_plan* plan,
                                    nseries_dtype dt, void* const* S_ptrs, uint32_t flags,
                                    void* stream) {
  if (batch > 0 && (!A_ptrs || !S_ptrs)) return NSERIES_ERR_INVALID_ARG;
  return eval_batched_impl(h, nullptr, 0, A_ptrs, batch, d, k, plan, dt, nullptr, 0, S_ptrs, flags,
                           stream);
}

nseries_status nseries_solve(nseries_handle h, const void* A, int32_t d, int32_t m, double tol,
                             int32_t max_steps, nseries_dtype dt, void* Y, void* R_out,
                             uint32_t flags, void* stream, nseries_solve_info* info) {
  if (!h || !A || !Y || d < 1 || max_steps < 1 || max_steps > NSERIES_MAX_STEPS) return NSERIES_ERR_INVALID_ARG;
  if (h->sticky != NSERIES_OK) return h->sticky;
  if (dt != NSERIES_F64) return NSERIES_ERR_INVALID_ARG;
  if (A == Y || (R_out && (A == R_out || Y == R_out))) return NSERIES_ERR_ALIAS;
  if (kernel_mu(m) < 0) return NSERIES_ERR_UNSUPPORTED_RADIX;
  nseries_plan p{};
  p.n_steps = max_steps;
  __int128 k = 1;
  for (int i = 0; i < max_steps; ++i) {
    if (k * m > ((__int128)1 << 62)) { p.n_steps = i; break; }   // plans reach at most 2^62
    p.step[i] = m;
    k *= m;
  }
  const uint32_t pflags = (m == 15 ? NSERIES_ALLOW_APPROX : 0u) | (flags & NSERIES_RFORM_TELESCOPE);
  nseries_status st = finalize_plan(&p, (int64_t)k, pflags);
  if (st != NSERIES_OK) return st;
  Program P;
  st = compile_plan(p, R_out != nullptr, &P);
  if (st != NSERIES_OK) return st;
  cudaSetDevice(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  st = ensure_ws(h, (size_t)P.n_slots * d * d * sizeof(double), s);
  if (st != NSERIES_OK) return st;
  if (P.needs_identity) {
    st = ensure_identity(h, d, NSERIES_F64, s);
    if (st != NSERIES_OK) return st;
  }
  // per-step ||R||_F^2 accumulators: one handle buffer, allocated once
  st = grow_buffer(h, &h->ssq, &h->ssq_bytes, sizeof(double) * NSERIES_MAX_STEPS, s);
  if (st != NSERIES_OK) return st;
  double* const d_ssq = static_cast<double*>(h->ssq);
  cudaMemsetAsync(d_ssq, 0, sizeof(double) * NSERIES_MAX_STEPS, s);
  nseries_solve_info inf{};
  inf.radix = m;
  const size_t slot = (size_t)d * d * sizeof(double);
  auto ptr = [&](int v) -> void* {
    switch (P.val_kind[v]) {
      case V_USER_A: return const_cast<void*>(A);
      case V_IDENT: return h->ident;
      case V_USER_S: return Y;
      case V_USER_R: return R_out;
      default: return static_cast<char*>(h->ws) + (size_t)P.val_buf[v] * slot;
    }
  };
  int op0 = 0, products = 0, launches = 0;
  int64_t prefix = 1;
  for (int step = 0; step < p.n_steps; ++step) {
    int op1 = op0;
    while (op1 < (int)P.ops.size() && P.ops[op1].step == step) ++op1;
    // the op producing this step's residual B_n carries the fused norm
    int rop = -1, rout = -1;
    for (int i = op0; i < op1; ++i)
      for (int j = 0; j < P.ops[i].n_out; ++j)
        if (P.ops[i].out[j] == P.step_B[step]) { rop = i; rout = j; }
    int nl = 0;
    st = run_program_range(h, P, A, Y, R_out, d, s, op0, op1, &nl, rop, rout, d_ssq + step);
    if (st != NSERIES_OK) return st;
    for (int i = op0; i < op1; ++i) products += P.ops[i].gemm ? 1 : 0;
    launches += nl;
    op0 = op1;
    prefix *= m;
    double ssq = 0.0;
    cudaError_t e = cudaMemcpyAsync(&ssq, d_ssq + step, sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(h, e);
    const double res = std::sqrt(ssq) / std::sqrt((double)d);
    inf.history[step] = res;
    inf.steps = step + 1;
    inf.residual = res;
    if (res <= tol || step + 1 == p.n_steps) {
      inf.converged = res <= tol ? 1 : 0;
      // stopped early: the iterate / residual still live in workspace -> copy out
      void* ys = ptr(P.step_S[step]);
      if (ys != Y) cudaMemcpyAsync(Y, ys, slot, cudaMemcpyDeviceToDevice, s);
      if (R_out) {
        void* rs = ptr(P.step_B[step]);
        if (rs != R_out) cudaMemcpyAsync(R_out, rs, slot, cudaMemcpyDeviceToDevice, s);
      }
      break;
    }
  }
  inf.products = products;
  inf.prefix = prefix;
  mark_use(h, s);
  h->stats = nseries_stats{};
  h->stats.products = h->stats.products_exec = h->stats.products_paper = products;
  h->stats.launches = launches;
  h->stats.n_ops = op0;
  if (info) *info = inf;
  return cuda_fail(h, cudaGetLastError());
}

nseries_status nseries_matmul(nseries_handle h, nseries_dtype dt, const void* X, const void* Y,
                              void* C, int32_t d, void* stream) {
  if (!h || !X || !Y || !C || d < 1) return NSERIES_ERR_INVALID_ARG;
  if (h->sticky != NSERIES_OK) return h->sticky;
  if (C == X || C == Y) return NSERIES_ERR_ALIAS;
  EpiParams ep{};
  ep.n_aux = 0;
  ep.n_out = 1;
  ep.out[0] = C;
  ep.alpha[0] = 1.0;
  cudaSetDevice(h->device);
  int rc;
  int launches = 1;
  if (dt == NSERIES_F64) {
    rc = launch_gemm_f64(static_cast<const double*>(X), static_cast<const double*>(Y), d, ep,
                         stream);
  } else {
    const int ldp = padded_ld(d);
    const size_t plane = (size_t)d * ldp;
    nseries_status st = ensure_ws(h, 4 * plane * sizeof(float), static_cast<cudaStream_t>(stream));
    if (st == NSERIES_OK) st = ensure_splitk(h, d, static_cast<cudaStream_t>(stream));
    if (st != NSERIES_OK) return st;
    float* w = static_cast<float*>(h->ws);
    rc = launch_split_f32(static_cast<const float*>(X), d, w, w + plane, nullptr, nullptr, ldp, d, false, stream);
    if (!rc)
      rc = launch_split_f32(static_cast<const float*>(Y), d, nullptr, nullptr, w + 2 * plane, w + 3 * plane, ldp,
                            d, false, stream);
    EpiParamsF32 e32{};
    e32.ldp = ldp;
    e32.n_aux = 0;
    e32.n_out = 1;
    e32.out_x[0] = static_cast<float*>(C);
    e32.out_ld[0] = d;
    e32.alpha[0] = 1.f;
    if (!rc)
      rc = d <= tf32_small_maxd()
               ? launch_gemm_tf32x3_b128(w, w + plane, w + 2 * plane, w + 3 * plane, d, ldp, e32, stream, h->sk_ws)
               : launch_gemm_tf32x3(w, w + plane, w + 2 * plane, w + 3 * plane, d, ldp, e32, stream, h->sk_ws);
    launches = 3;
  }
  mark_use(h, static_cast<cudaStream_t>(stream));
  h->stats = nseries_stats{};
  h->stats.products = h->stats.products_exec = h->stats.products_paper = 1;
  h->stats.launches = launches;
  h->stats.n_ops = 1;
  return cuda_fail(h, (cudaError_t)rc);
}

nseries_status nseries_last_stats(nseries_handle h, nseries_stats* out) {
  if (!h || !out) return NSERIES_ERR_INVALID_ARG;
  *out = h->stats;
  return NSERIES_OK;
}

nseries_status nseries_shard_rows(int32_t d, int32_t nshards, int32_t shard, int32_t* row0, int32_t* rows) {
  if (!row0 || !rows || nshards < 1 || d < nshards || shard < 0 || shard >= nshards) return NSERIES_ERR_INVALID_ARG;
  int r0, n;
  shard_range(d, nshards, shard, &r0, &n);
  *row0 = r0;
  *rows = n;
  return NSERIES_OK;
}

nseries_status nseries_comm_unique_id(void* id_out) {
  if (!id_out) return NSERIES_ERR_INVALID_ARG;
  const NcclApi& nc = nccl();
  if (!nc.ok) return NSERIES_ERR_CUDA;
  ncclUniqueId id;
  if (nc.get_unique_id(&id) != ncclSuccess) return NSERIES_ERR_CUDA;
  std::memcpy(id_out, &id, sizeof(id));
  return NSERIES_OK;
}

nseries_status nseries_sharded_arena_bytes(int32_t d, int32_t nshards, int32_t n_local, int64_t k,
                                          const nseries_plan* plan, uint32_t flags, int32_t want_R,
                                          uint64_t* bytes) {
  if (!bytes || d < 1 || nshards < 1 || n_local < 1 || n_local > nshards || d < nshards || k < 1)
    return NSERIES_ERR_INVALID_ARG;
  nseries_plan p;
  nseries_status st = resolve_plan(plan, k, flags, &p);
  if (st != NSERIES_OK) return st;
  Program prog;
  st = compile_plan(p, want_R != 0, &prog);
  if (st != NSERIES_OK) return st;
  const size_t rows_max = (size_t)(d + nshards - 1) / nshards;
  *bytes = (uint64_t)n_local * (prog.n_slots + 1) * rows_max * d * sizeof(double);
  return NSERIES_OK;
}

nseries_status nseries_peer_export(nseries_handle h, uint64_t bytes, void* handle_out) {
  if (!h || !handle_out || bytes == 0) return NSERIES_ERR_INVALID_ARG;
  if (h->sticky != NSERIES_OK) return h->sticky;
  cudaSetDevice(h->device);
  cudaError_t e = cudaDeviceSynchronize();   // setup call: nothing may still use an old arena
  if (e == cudaSuccess && h->arena_bytes < bytes) {
    for (size_t r = 0; r < h->peer_arena.size(); ++r)
      if ((int)r != h->rank && h->peer_arena[r]) cudaIpcCloseMemHandle(h->peer_arena[r]);
    h->peer_arena.clear();
    if (h->arena) cudaFree(h->arena);
    h->arena = nullptr;
    h->arena_bytes = 0;
    e = cudaMalloc(&h->arena, bytes);   // plain allocation: pool (cudaMallocAsync) memory is not IPC-exportable
    if (e == cudaSuccess) h->arena_bytes = bytes;
  }
  if (e == cudaSuccess && !h->bar_dev) {
    e = cudaMalloc(&h->bar_dev, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(h->bar_dev, 0, sizeof(int));
  }
  cudaIpcMemHandle_t ih;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&ih, h->arena);
  if (e != cudaSuccess) return cuda_fail(h, e);
  std::memcpy(handle_out, &ih, sizeof(ih));
  return NSERIES_OK;
}

nseries_status nseries_peer_import(nseries_handle h, const void* handles, int32_t nranks) {
  if (!h || !handles || nranks < 1) return NSERIES_ERR_INVALID_ARG;
  if (h->sticky != NSERIES_OK) return h->sticky;
  if (!h->comm || nranks != h->nranks || !h->arena) return NSERIES_ERR_INVALID_ARG;
  cudaSetDevice(h->device);
  for (size_t r = 0; r < h->peer_arena.size(); ++r)
    if ((int)r != h->rank && h->peer_arena[r]) cudaIpcCloseMemHandle(h->peer_arena[r]);
  h->peer_arena.assign(nranks, nullptr);
  for (int r = 0; r < nranks; ++r) {
    if (r == h->rank) {
      h->peer_arena[r] = h->arena;
      continue;
    }
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, static_cast<const char*>(handles) + (size_t)r * sizeof(ih), sizeof(ih));
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, ih, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      h->peer_arena.clear();
      return cuda_fail(h, e);
    }
    h->peer_arena[r] = ptr;
  }
  return NSERIES_OK;
}

nseries_status nseries_comm_init(nseries_handle h, const void* id, int32_t nranks, int32_t rank) {
  if (!h || !id || nranks < 1 || rank < 0 || rank >= nranks) return NSERIES_ERR_INVALID_ARG;
  if (h->sticky != NSERIES_OK) return h->sticky;
  const NcclApi& nc = nccl();
  if (!nc.ok) return NSERIES_ERR_CUDA;
  cudaSetDevice(h->device);
  if (h->comm) {
    nc.comm_destroy(h->comm);
    h->comm = nullptr;
  }
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  nseries_status st = nccl_fail(h, nc.comm_init_rank(&c, nranks, uid, rank));
  if (st != NSERIES_OK) return st;
  h->comm = c;
  h->nranks = nranks;
  h->rank = rank;
  return NSERIES_OK;
}

nseries_status nseries_eval_sharded(nseries_handle h, const void* const* A_shards, int32_t n_local,
                                    int32_t first_shard, int32_t nshards, int32_t d, int64_t k,
                                    const nseries_plan* plan, nseries_dtype dt, void* const* S_shards,
                                    void* const* R_shards, uint32_t flags, void* stream) {
  if (!h) return NSERIES_ERR_INVALID_ARG;
  if (h->sticky != NSERIES_OK) return h->sticky;
  if (!A_shards || !S_shards || n_local < 1 || nshards < n_local || d < nshards || k < 1 || first_shard < 0 ||
      first_shard + n_local > nshards)
    return NSERIES_ERR_INVALID_ARG;
  if (dt != NSERIES_F64) return NSERIES_ERR_UNSUPPORTED_SIZE;
  if (flags & NSERIES_SYMMETRIC) return NSERIES_ERR_INVALID_ARG;
  if (n_local < nshards && (!h->comm || nshards != h->nranks * n_local || first_shard != h->rank * n_local))
    return NSERIES_ERR_INVALID_ARG;
  for (int j = 0; j < n_local; ++j) {
    if (!A_shards[j] || !S_shards[j]) return NSERIES_ERR_INVALID_ARG;
    if (A_shards[j] == S_shards[j] || (R_shards && (!R_shards[j] || R_shards[j] == A_shards[j] ||
                                                    R_shards[j] == S_shards[j])))
      return NSERIES_ERR_ALIAS;
  }
  nseries_plan p;
  nseries_status st = resolve_plan(plan, k, flags, &p);
  if (st != NSERIES_OK) return st;
  const bool want_R = R_shards != nullptr;
  std::string key = plan_key(p, want_R);
  auto it = h->programs.find(key);
  if (it == h->programs.end()) {
    Program prog;
    st = compile_plan(p, want_R, &prog);
    if (st != NSERIES_OK) return st;
    it = h->programs.emplace(key, std::move(prog)).first;
  }
  const Program& P = it->second;
  cudaSetDevice(h->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t rows_max = (size_t)(d + nshards - 1) / nshards;
  st = ensure_ws(h, (size_t)n_local * P.n_slots * rows_max * d * sizeof(double), s);
  if (st != NSERIES_OK) return st;
  st = grow_buffer(h, &h->full, &h->full_bytes, 3 * (size_t)d * d * sizeof(double), s);
  if (st != NSERIES_OK) return st;
  st = ensure_identity(h, d, NSERIES_F64, s);    // I as a full right factor / its row blocks
  if (st != NSERIES_OK) return st;
  const bool timing = (flags & NSERIES_SYNC_STATS) != 0;
  const bool check = (flags & NSERIES_CHECK_FINITE) != 0;
  if (check && (st = begin_check(h, s)) != NSERIES_OK) return st;
  if (timing) cudaEventRecord(h->ev0, s);
  int launches = 0, gathers = 0, prefetched = 0;
  st = run_sharded(h, P, reinterpret_cast<const double* const*>(A_shards), reinterpret_cast<double* const*>(S_shards),
                   reinterpret_cast<double* const*>(R_shards), n_local, first_shard, nshards, d, s,
                   (flags & NSERIES_SHARDED_DIRECT) != 0, &launches, &gathers, &prefetched);
  if (st != NSERIES_OK) return st;
  mark_use(h, s);
  if (check) {   // this process's row blocks of S
    for (int i = 0; i < n_local; ++i) {
      int r0, rows;
      shard_range(d, nshards, first_shard + i, &r0, &rows);
      const int rc = launch_count_nonfinite(NSERIES_F64, S_shards[i], 0, nullptr, 1, rows, d, h->nf_dev, s);
      if (rc != 0) return cuda_fail(h, (cudaError_t)rc);
      ++launches;
    }
  }
  h->stats = nseries_stats{};
  h->stats.products = h->stats.products_exec = P.products;
  h->stats.products_paper = paper_products(p);
  h->stats.launches = launches;
  h->stats.n_ops = (int)P.ops.size();
  h->stats.gathers = gathers;
  h->stats.gathers_prefetched = prefetched;
  if (timing) {
    cudaEventRecord(h->ev1, s);
    cudaEventSynchronize(h->ev1);
    cudaEventElapsedTime(&h->stats.ms_total, h->ev0, h->ev1);
  }
  st = cuda_fail(h, cudaGetLastError());
  if (st == NSERIES_OK && check) st = finish_check(h, s);
  return st;
}

}  // extern "C"
