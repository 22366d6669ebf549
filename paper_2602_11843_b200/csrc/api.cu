// api.cu -- C ABI (include/nseries.h): handle, workspace, plan compilation cache and the
// stream executor that launches one fused GEMM kernel per op.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

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
  int ident_d = 0;
  nseries_dtype ident_dt = NSERIES_F64;
  // host-API staging
  void* stage = nullptr;
  size_t stage_bytes = 0;
  // compiled programs keyed by plan bytes + want_R
  std::map<std::string, Program> programs;
  nseries_stats stats{};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

namespace {

nseries_status cuda_fail(nseries_ctx* h, cudaError_t e) {
  if (e == cudaSuccess) return NSERIES_OK;
  if (h) h->sticky = NSERIES_ERR_CUDA;
  std::fprintf(stderr, "[nseries] CUDA error: %s\n", cudaGetErrorString(e));
  return NSERIES_ERR_CUDA;
}

size_t elem_size(nseries_dtype dt) { return dt == NSERIES_F64 ? sizeof(double) : sizeof(float); }

nseries_status ensure_ws(nseries_ctx* h, size_t bytes) {
  if (bytes <= h->ws_bytes) return NSERIES_OK;
  if (h->ws) {
    cudaDeviceSynchronize();
    cudaFree(h->ws);
    h->ws = nullptr;
    h->ws_bytes = 0;
  }
  cudaError_t e = cudaMalloc(&h->ws, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return NSERIES_ERR_OOM;
  }
  h->ws_bytes = bytes;
  return NSERIES_OK;
}

nseries_status ensure_identity(nseries_ctx* h, int d, nseries_dtype dt, cudaStream_t s) {
  if (h->ident && h->ident_d == d && h->ident_dt == dt) return NSERIES_OK;
  if (h->ident) {
    cudaStreamSynchronize(s);
    cudaFree(h->ident);
    h->ident = nullptr;
  }
  cudaError_t e = cudaMalloc(&h->ident, (size_t)d * d * elem_size(dt));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return NSERIES_ERR_OOM;
  }
  h->ident_d = d;
  h->ident_dt = dt;
  int rc = launch_identity_f64(static_cast<double*>(h->ident), d, s);
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

// Execute a compiled program on the stream.
nseries_status run_program(nseries_ctx* h, const Program& P, const void* A, void* S, void* R,
                           int d, nseries_dtype dt, cudaStream_t s, int* launches) {
  const size_t slot = (size_t)d * d * elem_size(dt);
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
  for (const Op& op : P.ops) {
    EpiParams ep{};
    ep.n_aux = op.n_aux;
    ep.n_out = op.n_out;
    for (int i = 0; i < op.n_aux; ++i) ep.aux[i] = ptr(op.aux[i]);
    for (int j = 0; j < op.n_out; ++j) {
      ep.out[j] = ptr(op.out[j]);
      ep.alpha[j] = op.alpha[j];
      ep.gamma[j] = op.gamma[j];
      for (int i = 0; i < kMaxAux; ++i) ep.beta[j][i] = op.beta[j][i];
    }
    int rc;
    if (dt == NSERIES_F64) {
      rc = op.gemm ? launch_gemm_f64(static_cast<const double*>(ptr(op.X)),
                                     static_cast<const double*>(ptr(op.Y)), d, ep, s)
                   : launch_axpby_f64(d, ep, s);
    } else {
      return NSERIES_ERR_INVALID_ARG;
    }
    if (rc != 0) return cuda_fail(h, (cudaError_t)rc);
    ++nl;
  }
  *launches = nl;
  return NSERIES_OK;
}

}  // namespace

extern "C" {

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
  h->device = device;
  cudaEventCreate(&h->ev0);
  cudaEventCreate(&h->ev1);
  *out = h;
  return NSERIES_OK;
}

nseries_status nseries_destroy(nseries_handle h) {
  if (!h) return NSERIES_ERR_INVALID_ARG;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  if (h->ws) cudaFree(h->ws);
  if (h->ident) cudaFree(h->ident);
  if (h->stage) cudaFree(h->stage);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
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
  if (dt == NSERIES_F32) return NSERIES_ERR_INVALID_ARG;   // fp32 engine: see DESIGN.md status
  nseries_plan p;
  nseries_status st = resolve_plan(plan, k, flags, &p);
  if (st != NSERIES_OK) return st;
  const bool want_R = R_out != nullptr;
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
  st = ensure_ws(h, (size_t)P.n_slots * d * d * elem_size(dt));
  if (st != NSERIES_OK) return st;
  if (P.needs_identity) {
    st = ensure_identity(h, d, dt, s);
    if (st != NSERIES_OK) return st;
  }
  const bool timing = (flags & NSERIES_SYNC_STATS) != 0;
  if (timing) cudaEventRecord(h->ev0, s);
  int launches = 0;
  st = run_program(h, P, A, S, R_out, d, dt, s, &launches);
  if (st != NSERIES_OK) return st;
  h->stats.products = P.products;
  h->stats.launches = launches;
  h->stats.graph_replayed = 0;
  h->stats.n_ops = (int)P.ops.size();
  h->stats.ms_total = 0.f;
  if (timing) {
    cudaEventRecord(h->ev1, s);
    cudaEventSynchronize(h->ev1);
    cudaEventElapsedTime(&h->stats.ms_total, h->ev0, h->ev1);
  }
  return cuda_fail(h, cudaGetLastError());
}

nseries_status nseries_eval_host(nseries_handle h, const void* A_host, int32_t d, int64_t k,
                                 const nseries_plan* plan, nseries_dtype dt, void* S_host,
                                 void* R_host, uint32_t flags, void* stream) {
  if (!h || !A_host || !S_host || d < 1 || k < 1) return NSERIES_ERR_INVALID_ARG;
  if (h->sticky != NSERIES_OK) return h->sticky;
  const size_t bytes = (size_t)d * d * elem_size(dt);
  const size_t need = bytes * (R_host ? 3 : 2);
  cudaSetDevice(h->device);
  if (need > h->stage_bytes) {
    if (h->stage) { cudaDeviceSynchronize(); cudaFree(h->stage); h->stage = nullptr; h->stage_bytes = 0; }
    if (cudaMalloc(&h->stage, need) != cudaSuccess) { cudaGetLastError(); return NSERIES_ERR_OOM; }
    h->stage_bytes = need;
  }
  char* dA = static_cast<char*>(h->stage);
  char* dS = dA + bytes;
  char* dR = R_host ? dS + bytes : nullptr;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(dA, A_host, bytes, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return cuda_fail(h, e);
  nseries_status st = nseries_eval(h, dA, d, k, plan, dt, dS, dR, flags & ~NSERIES_SYNC_STATS, stream);
  if (st != NSERIES_OK) return st;
  e = cudaMemcpyAsync(S_host, dS, bytes, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return cuda_fail(h, e);
  if (R_host) {
    e = cudaMemcpyAsync(R_host, dR, bytes, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(h, e);
  }
  return cuda_fail(h, cudaStreamSynchronize(s));
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
      for (int a = 0; a < kMaxAux; ++a) b.beta[j][a] = op.beta[j][a];
    }
  }
  h->stats = nseries_stats{};
  h->stats.products = P.products;
  h->stats.n_ops = bp.n_ops;
  if (batch == 0) return NSERIES_OK;
  if ((!A && !A_ptrs) || (!S && !S_ptrs)) return NSERIES_ERR_INVALID_ARG;
  if (A && A == S) return NSERIES_ERR_ALIAS;
  cudaSetDevice(h->device);
  int rc = launch_batched(dt, A, strideA, A_ptrs, S, strideS, S_ptrs, batch, d, bp, stream);
  if (rc == -1) return NSERIES_ERR_UNSUPPORTED_SIZE;
  if (rc != 0) return cuda_fail(h, (cudaError_t)rc);
  h->stats.launches = 1;
  return NSERIES_OK;
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
  if (dt == NSERIES_F64)
    rc = launch_gemm_f64(static_cast<const double*>(X), static_cast<const double*>(Y), d, ep,
                         stream);
  else
    return NSERIES_ERR_INVALID_ARG;
  h->stats = nseries_stats{};
  h->stats.products = 1;
  h->stats.launches = 1;
  h->stats.n_ops = 1;
  return cuda_fail(h, (cudaError_t)rc);
}

nseries_status nseries_last_stats(nseries_handle h, nseries_stats* out) {
  if (!h || !out) return NSERIES_ERR_INVALID_ARG;
  *out = h->stats;
  return NSERIES_OK;
}

}  // extern "C"
