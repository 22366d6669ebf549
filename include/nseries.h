/*
 * nseries.h -- C ABI of the B200-native truncated-Neumann-series library
 * (arXiv 2602.11843, "radix kernels").  sm_100a only.
 *
 * Problem (Eq. series): given A in R^{d x d} and k >= 1,
 * return S_k(A) = I + A + ... + A^{k-1}.  Cost is counted in d x d matrix
 * products.  S_k is reached by radix-kernel splitting
 * S_{mn}(A) = S_n(A) T_m(A^n) (Eq. decomposition) with
 *   - binary splitting (m=2) and ternary splitting (m=3),
 *   - the radix-5 kernel,
 *   - the exact 3-product radix-9 kernel (Theorem 1),
 *   - the approximate 4-product radix-15 kernel
 *     inside the residual framework Y_{n+1} = Y_n f(R_n), R_{n+1} = I - M Y_{n+1}
 *     (PAPER.md:551-558),
 *   - "+1" steps S_{n+1} = S_n + A^n for arbitrary k (no paper counterpart;
 *     DESIGN.md reading R5),
 * composed into plans by a fewest-product plan builder.
 *
 * Conventions for every entry point:
 *   - Matrices are dense, row-major, contiguous, leading dimension d.
 *   - Pointers named A, S, R_out, X, Y, C are DEVICE pointers (cudaMalloc /
 *     torch CUDA tensors) unless the function name ends in _host.
 *   - The caller owns A, S, R_out; the library owns its workspace (allocated
 *     lazily per handle, freed by nseries_destroy).  A is read-only and must
 *     not alias S or R_out.
 *   - Work is enqueued asynchronously on `stream` (a cudaStream_t passed as
 *     void*; NULL = legacy default stream).  Argument errors are returned
 *     synchronously before anything is enqueued.  CUDA errors are returned as
 *     NSERIES_ERR_CUDA and are sticky for the handle.
 *   - A handle is not thread-safe; use one handle per host thread / stream.
 *   - There is no CPU fallback: every arithmetic step runs in this library's
 *     sm_100a kernels; without a usable sm_100a device, create() fails.
 */
#ifndef NSERIES_H
#define NSERIES_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nseries_ctx* nseries_handle;

typedef enum {
  NSERIES_OK = 0,
  NSERIES_ERR_INVALID_ARG = 1,      /* bad pointer / size / flag combination          */
  NSERIES_ERR_UNSUPPORTED_RADIX = 2,/* radix outside 2..32 (or "+1" = 1)              */
  NSERIES_ERR_PLAN_K_MISMATCH = 3,  /* plan does not reach k (pure plan with k!=m^t) */
  NSERIES_ERR_APPROX_TELESCOPE = 4, /* approximate kernel in a telescoping-form step,
                                       or approximate radix without ALLOW_APPROX      */
  NSERIES_ERR_ALIAS = 5,            /* A aliases S or R_out                          */
  NSERIES_ERR_OOM = 6,              /* workspace allocation failed                   */
  NSERIES_ERR_CUDA = 7,             /* CUDA runtime / launch error (sticky)          */
  NSERIES_ERR_NO_DEVICE = 8,        /* no sm_100 device                              */
  NSERIES_ERR_UNSUPPORTED_SIZE = 9, /* e.g. batched path with d > 64                 */
  NSERIES_ERR_NONFINITE = 10        /* NSERIES_CHECK_FINITE: S has NaN / Inf entries (the
                                       result is written; not sticky)                  */
} nseries_status;

typedef enum {
  NSERIES_F64 = 0, /* IEEE binary64 throughout; FP64 tensor cores (DMMA)               */
  NSERIES_F32 = 1  /* fp32 in/out; products as 3xTF32 on tcgen05 with fp32 accumulate  */
} nseries_dtype;

typedef enum {
  NSERIES_PLAN_AUTO = 0,     /* fewest products over the radix set (default {9,5,2},
                                {15,9,5,2} with NSERIES_ALLOW_APPROX)                 */
  NSERIES_PLAN_BINARY = 2,   /* pure plans: k must equal m^t          */
  NSERIES_PLAN_TERNARY = 3,
  NSERIES_PLAN_RADIX5 = 5,
  NSERIES_PLAN_RADIX9 = 9,
  NSERIES_PLAN_RADIX15 = 15,
  NSERIES_PLAN_CUSTOM = -1   /* caller fills nseries_plan.step[] itself               */
} nseries_plan_kind;

/* flags (bitwise OR) */
#define NSERIES_ELIDE_TRIVIAL    0x1u /* skip the S_1 = I concatenation and the unused final
                                         power/residual product; default is the
                                         paper's counting (mu_m + 2) t of Table 2.  With
                                         R_out the final power is used, so it is computed
                                         (one product more than plan.products_exec)      */
#define NSERIES_ALLOW_APPROX     0x2u /* allow the approximate radix-15 kernel (residual form) */
#define NSERIES_RFORM_TELESCOPE  0x4u /* radix-15 residual update as R' = I - f + f R instead
                                         of the paper's R' = I - M Y' (PAPER.md:557 vs 573)   */
#define NSERIES_NO_GRAPH         0x8u /* do not capture/replay the op list as a CUDA graph     */
#define NSERIES_SYNC_STATS       0x10u/* time the eval on the device: the op list runs eagerly
                                         (no graph), an event at every plan-step boundary gives
                                         stats.ms_step[], the call synchronizes the stream; also
                                         one NVTX range per plan step                          */
#define NSERIES_SYMMETRIC        0x20u/* caller asserts A = A^T (fp64, d > 64): every value of
                                         the plan is a polynomial in A, hence symmetric, so each
                                         product computes only the tiles on/above the diagonal and
                                         mirrors them (same products, ~half the tile work).  The
                                         result is unspecified if A is not symmetric.           */
#define NSERIES_HOST_ASYNC       0x40u/* nseries_eval_host only: return without synchronizing;
                                         consecutive calls alternate two device staging sets so
                                         the copy-in of one matrix overlaps the evaluation of the
                                         previous one.  S_host / R_host are valid and A_host may
                                         be reused only after nseries_host_sync.                */
#define NSERIES_CHECK_FINITE     0x80u/* count NaN / Inf entries of S (fused into the final
                                         epilogue of the tiled fp64 engine and the batched
                                         warp kernel, one extra pass over S elsewhere); the
                                         call synchronizes the stream and returns
                                         NSERIES_ERR_NONFINITE if the count is nonzero
                                         (stats.nonfinite).  SURVEY F5: config 4's divergent
                                         matrices (rho > 1) overflow fp32 for large k.      */

#define NSERIES_SHARDED_DIRECT   0x100u/* nseries_eval_sharded: read the right factor of every
                                         product in place, straight from its row blocks (the GEMM's
                                         k-tile loads pick the block that holds rows k0..k0+BK),
                                         instead of gathering it into a full buffer first.  Needs
                                         every block of the factor addressable by this process:
                                         all shards local (one GPU), or the peers' arenas mapped
                                         with nseries_peer_import; uniform blocks (d divisible by
                                         nshards, rows a multiple of 32, nshards <= 16).  Factors
                                         that are not addressable (the user's A or S blocks of a
                                         peer) are still gathered.  Falls back to gathers where
                                         the conditions do not hold.                          */

#define NSERIES_MAX_STEPS 128

/* A plan: a sequence of steps from n = 1 to n = k.  step[i] = m in 2..32 multiplies n by m;
 * step[i] = 1 is a "+1" step.  Kernels: m = 2 binary, 3 ternary, 5 the radix-5 kernel, 9 the
 * exact radix-9 kernel (Theorem 1), 15 the approximate radix-15 kernel (residual framework);
 * every other m is naive radix-m splitting: the powers B^2 .. B^{m-1}
 * (m - 2 products) with T_m = I + B + ... + B^{m-1} accumulated in their epilogues, then the
 * concatenation and the next power -- C(m) = m products per step.  form[i] is filled by the
 * builder: 0 = telescoping power update R' = I - T + T R (exact kernels,
 * PAPER.md:211-212), 1 = paper residual update R' = I - M Y',
 * 2 = telescoping-form residual R' = I - f + f R.  products = GEMMs executed
 * under `flags`.  approx = 1 if any step is radix 15 (then the result is the
 * residual-framework polynomial Y_n, which agrees with S_k on degrees < k;
 * Y_n - S_k = M^{-1}(A^k - R_n)). */
typedef struct {
  int32_t n_steps;
  int32_t step[NSERIES_MAX_STEPS];
  int32_t form[NSERIES_MAX_STEPS];
  int32_t products;
  int32_t approx;
  uint32_t flags;
  int64_t k;
} nseries_plan;

typedef struct {
  int32_t products;        /* GEMMs executed by the last eval (== products_exec)            */
  int32_t launches;        /* kernel launches of the last eval (GEMMs + degenerate ops; 1 for
                              the single-launch small / batched kernels; + the finite check) */
  int32_t graph_replayed;  /* 1 if the last eval replayed a cached CUDA graph                */
  int32_t n_ops;
  float   ms_total;        /* device time of the last eval (NSERIES_SYNC_STATS only, else 0) */
  int32_t gathers;         /* row-block gathers of the last nseries_eval_sharded (else 0)   */
  int32_t gathers_prefetched; /* of which issued ahead, overlapping the previous product    */
  int32_t products_paper;  /* the paper's count for the plan (Table 2 counting, PAPER.md:693-709:
                              mu_m + 2 per radix step incl. S_1 = I and the final power, 1 per
                              "+1"), whatever the flags                                    */
  int32_t products_exec;   /* GEMMs actually executed (ELIDE_TRIVIAL: -2; R_out keeps the final
                              power); a batched eval counts per matrix                      */
  int32_t n_steps_timed;   /* entries of ms_step[] set (NSERIES_SYNC_STATS with per-op launches;
                              0 for the single-launch small / batched kernels)              */
  float   ms_step[NSERIES_MAX_STEPS]; /* device time of each plan step                      */
  int32_t nonfinite;       /* NSERIES_CHECK_FINITE: NaN / Inf entries of S (else 0)         */
} nseries_stats;

/* ---- lifecycle ---------------------------------------------------------------------- */
/* Create a handle bound to CUDA device `device`.  Fails with NSERIES_ERR_NO_DEVICE if the
 * device is not sm_100 (the only architecture the kernels are built for). */
nseries_status nseries_create(nseries_handle* h, int device);
nseries_status nseries_destroy(nseries_handle h);
const char*    nseries_status_string(nseries_status s);
/* Version string of the library build (arch, git-independent). */
const char*    nseries_version(void);

/* ---- host-only plan builder (no device needed) ----------------------------------------
 * Pure kinds require k = m^t.  AUTO searches plans over `radices` (NULL -> default set) for
 * the fewest products, tie-break: fewest "+1", fewest steps, larger radices first
 * (reading R6).  Returns NSERIES_ERR_PLAN_K_MISMATCH / _UNSUPPORTED_RADIX /
 * _APPROX_TELESCOPE on invalid requests.  k in [1, 2^62]. */
nseries_status nseries_plan_build(int64_t k, nseries_plan_kind kind, const int32_t* radices,
                                  int32_t n_radices, uint32_t flags, nseries_plan* out);
/* Validate a CUSTOM plan (steps filled by caller), fill form/products/approx/k. */
nseries_status nseries_plan_finalize(nseries_plan* plan, int64_t k, uint32_t flags);

/* Monomial coefficients [f]_0..[f]_D of the radix-m kernel polynomial as this library
 * evaluates it (binary64 circuit parameters).  coeffs may be NULL to query
 * the count; *n_coeffs in: capacity, out: D+1.  mu = products of the circuit. */
nseries_status nseries_kernel_info(int32_t m, int32_t* mu, int32_t* exact, double* coeffs,
                                   int32_t* n_coeffs);

/* ---- evaluation -----------------------------------------------------------------------
 * S <- S_k(A) (exact plans) or the plan polynomial Y_n (approximate plans), d x d, dtype dt.
 * plan == NULL builds an AUTO plan from k and flags.  R_out (nullable) receives the final
 * power A^k (exact plans) or residual R_n = I - (I-A) Y_n -- the paper's accuracy metric
 * I - (I-A)S_k.  Each radix-m step is exactly mu_m + 2 GEMM launches with all
 * linear combinations fused into GEMM epilogues. */
nseries_status nseries_eval(nseries_handle h, const void* A, int32_t d, int64_t k,
                            const nseries_plan* plan, nseries_dtype dt, void* S, void* R_out,
                            uint32_t flags, void* stream);

/* Same with HOST pointers: copies A host->device, evaluates, copies S (and R_out) back,
 * then synchronizes `stream`.  Pinned host memory gives asynchronous copies.  With
 * NSERIES_HOST_ASYNC the call only enqueues (copy-in on a private stream, the evaluation on
 * `stream`, copy-out on a private stream, ordered by events) and a stream of calls pipelines
 * copy-in / evaluate / copy-out across matrices; nseries_host_sync waits for all of them. */
nseries_status nseries_eval_host(nseries_handle h, const void* A_host, int32_t d, int64_t k,
                                 const nseries_plan* plan, nseries_dtype dt, void* S_host,
                                 void* R_host, uint32_t flags, void* stream);
nseries_status nseries_host_sync(nseries_handle h);

/* Batched small-matrix path: `batch` independent d x d matrices (d <= 64), A_b at
 * A + b*strideA elements, S_b at S + b*strideS.  One kernel launch evaluates the whole plan
 * for every matrix with the matrix resident in shared memory; products are counted per
 * matrix (stats.products = plan products, stats.launches = 1). */
nseries_status nseries_eval_batched_strided(nseries_handle h, const void* A, int64_t strideA,
                                            int32_t batch, int32_t d, int64_t k,
                                            const nseries_plan* plan, nseries_dtype dt, void* S,
                                            int64_t strideS, uint32_t flags, void* stream);
/* Pointer-array form: A_ptrs / S_ptrs are DEVICE arrays of `batch` device pointers. */
nseries_status nseries_eval_batched(nseries_handle h, const void* const* A_ptrs, int32_t batch,
                                    int32_t d, int64_t k, const nseries_plan* plan,
                                    nseries_dtype dt, void* const* S_ptrs, uint32_t flags,
                                    void* stream);

/* ---- adaptive approximate inverse -----------------------------
 * Y ~ (I - A)^{-1} by the residual radix-kernel iteration Y_{n+1} = Y_n f(R_n),
 * R_{n+1} = I - (I - A) Y_{n+1} with kernel m in {2,3,5,9,15}; m = 2 is
 * Hensel lifting Y' = Y(2I - MY).  After every step the fused epilogue of
 * the residual product accumulates ||R_n||_F^2 on the device; the host reads it (one stream
 * synchronisation per step) and stops once ||R_n||_F / sqrt(d) <= tol (the normalised residual
 * of App. A.3) or after max_steps.  Costs (mu_m + 2) products per step.
 * fp64 only.  Y (and R_out if non-NULL) receive the iterate and residual of the last step. */
typedef struct {
  int32_t steps;        /* radix steps executed                                            */
  int32_t products;     /* GEMMs executed                                                  */
  int32_t converged;    /* 1 if the tolerance was reached                                  */
  int32_t radix;
  int64_t prefix;       /* m^steps: Y matches the Neumann series through degree prefix-1   */
  double residual;      /* final ||I - (I - A) Y||_F / sqrt(d)                              */
  double history[NSERIES_MAX_STEPS];  /* normalised residual after each executed step      */
} nseries_solve_info;

nseries_status nseries_solve(nseries_handle h, const void* A, int32_t d, int32_t m, double tol,
                             int32_t max_steps, nseries_dtype dt, void* Y, void* R_out,
                             uint32_t flags, void* stream, nseries_solve_info* info);

/* Single fused-engine product C = X Y (d x d) -- the GEMM engine the plans run on, exposed
 * for accuracy micro-tests and peak measurement.  Counts as one product. */
nseries_status nseries_matmul(nseries_handle h, nseries_dtype dt, const void* X, const void* Y,
                              void* C, int32_t d, void* stream);

/* ---- row-sharded chain -----------------------------------
 * One A too large (or too slow) for one GPU: rows [0, d) are split into `nshards` contiguous
 * row blocks (nseries_shard_rows), and every value of the plan (A, the temporaries, S, R) is
 * held as those row blocks.  A product X.Y needs, for its row block of the result, the row
 * block of X and ALL of Y ("1D row-block shards with an allgather of the right
 * operand per GEMM"); every value is a polynomial in A, so X.Y = Y.X and the executor gathers
 * whichever factor is cheaper (I is never gathered: the identity buffer is full; A is gathered
 * once; two gathered values are cached).  fp64 only (the DMMA engine with row-block launches).
 *
 * nseries_shard_rows: host-only, pure.  Shard s of nshards over d rows starts at
 *   row0 = s*floor(d/nshards) + min(s, d mod nshards) and has floor(d/nshards) (+1 for the
 *   first d mod nshards shards) rows.  INVALID_ARG unless 1 <= nshards <= d, 0 <= s < nshards.
 * nseries_comm_unique_id / nseries_comm_init: the NCCL communicator the gathers run over
 *   (libnccl.so.2 is opened at run time; the caller ships the 128-byte id from rank 0 to the
 *   others over any side channel).  One rank per GPU; the handle keeps the
 *   communicator until nseries_destroy.  CUDA error -> NSERIES_ERR_CUDA.
 * nseries_eval_sharded: this process holds n_local consecutive shards first_shard ..
 *   first_shard + n_local - 1 (HOST arrays of DEVICE pointers, each shard rows_s x d,
 *   row-major, contiguous).  If the handle has a communicator with nshards == nranks *
 *   n_local and first_shard == rank * n_local, each gather is an allgather-v (grouped
 *   ncclBroadcast of every shard from its owner into the full-size buffer; with one rank all
 *   broadcasts are local).  Otherwise every shard must be local (n_local == nshards) and the
 *   gathers are device copies (one GPU; also the single-process test of the sharded
 *   arithmetic); n_local < nshards without a matching communicator is INVALID_ARG.  S_shards / R_shards (nullable) receive the
 *   row blocks of S and R.  Workspace per process: n_local x slots x (rows_max x d) doubles
 *   plus three d x d buffers (gathered A and two gathered operands).  Same plans, flags and
 *   product counts as nseries_eval (NSERIES_SYMMETRIC is rejected); eager launches (no
 *   graph).  stats.launches counts GEMM/axpby launches, stats.gathers the gathers. */
nseries_status nseries_shard_rows(int32_t d, int32_t nshards, int32_t shard, int32_t* row0, int32_t* rows);

/* ---- in-place right factors across GPUs (NSERIES_SHARDED_DIRECT with a communicator) ------
 * SURVEY.md 8(f) NEXT-3 "TMA-over-NVLink" variant: instead of an allgather of the right factor
 * before every product, each GEMM's k-tile loads read the factor's row blocks where they live
 * -- in the owning rank's arena, mapped into this process over NVLink by CUDA IPC -- and a
 * one-int ncclAllReduce after every op is the barrier that orders the owners' writes before
 * the readers' loads (and the loads before the next overwrite).
 * nseries_sharded_arena_bytes: host-only, pure: the arena size one rank needs for this plan
 *   (n_local x (value slots + 1 copy of A) x rows_max x d doubles).
 * nseries_peer_export: allocate (or grow to `bytes`; every rank must pass the same size) this
 *   handle's arena -- a plain cudaMalloc allocation; synchronizes the device -- and write its
 *   64-byte cudaIpcMemHandle_t to handle_out.
 * nseries_peer_import: `handles` holds nranks consecutive 64-byte handles indexed by rank (the
 *   caller all-gathers them over any side channel); maps every peer's arena
 *   (cudaIpcOpenMemHandle, P2P access enabled lazily), this rank's own entry is skipped.  Needs
 *   nseries_comm_init first with the same nranks.  Afterwards nseries_eval_sharded with
 *   NSERIES_SHARDED_DIRECT and a matching shard map reads right factors in place (the user's S
 *   / R blocks of peers are still gathered).  Handles stay mapped until nseries_destroy or the
 *   next import.  Every rank exports once, with the same size, before its first direct eval: a
 *   later export that has to grow the arena frees the old one, which invalidates the peers'
 *   mappings of it -- all ranks must then export and import again. */
nseries_status nseries_sharded_arena_bytes(int32_t d, int32_t nshards, int32_t n_local, int64_t k,
                                          const nseries_plan* plan, uint32_t flags, int32_t want_R,
                                          uint64_t* bytes);
nseries_status nseries_peer_export(nseries_handle h, uint64_t bytes, void* handle_out /* 64 bytes */);
nseries_status nseries_peer_import(nseries_handle h, const void* handles /* nranks x 64 bytes */, int32_t nranks);
nseries_status nseries_comm_unique_id(void* id_out /* 128 bytes */);
nseries_status nseries_comm_init(nseries_handle h, const void* id /* 128 bytes */, int32_t nranks, int32_t rank);
nseries_status nseries_eval_sharded(nseries_handle h, const void* const* A_shards, int32_t n_local,
                                    int32_t first_shard, int32_t nshards, int32_t d, int64_t k,
                                    const nseries_plan* plan, nseries_dtype dt, void* const* S_shards,
                                    void* const* R_shards, uint32_t flags, void* stream);

/* Statistics of the last eval on this handle (valid after the stream is synchronized). */
nseries_status nseries_last_stats(nseries_handle h, nseries_stats* out);

#ifdef __cplusplus
}
#endif
#endif /* NSERIES_H */
