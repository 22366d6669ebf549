/*
 * nseries_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the truncated Neumann series
 * path of arXiv 2602.11843.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code, header, table or helper with the CUDA library under
 * paper_2602_11843_b200/ and neither side includes the other.
 *
 * Arithmetic: x87 80-bit long double throughout (the paper computes in IEEE
 * binary64, PAPER.md:672 (Sec. 6); the oracle is run in higher precision so
 * that its own rounding is negligible against the 1e-11 parity tolerance).
 * Inputs A are binary64 (fp32 inputs are passed widened, which is exact).
 *
 * Functions
 *   or_series_sum   -- C-1: S_k(A) V = sum_{j<k} A^j V, the definition
 *                      PAPER.md:56-59 (Eq. neumann) / PAPER.md:125-128
 *                      (Eq. series), accumulated as the naive method does:
 *                      "accumulates powers I, A, A^2, ..., requiring k-1
 *                      matrix products".  Optional
 *                      rigorous early stop for matrices with ||A||_2 <= q < 1.
 *   or_plan_apply   -- C-2: the polynomial a radix-kernel plan evaluates,
 *                      following the general radix-kernel iteration
 *                      Y_0 = I, R_0 = A, Y_{n+1} = Y_n f(R_n),
 *                      R_{n+1} = I - M Y_{n+1}, M = I - A
 *                      (Eq. generalradix), applied to a
 *                      block of vectors without forming matrices.  f is given
 *                      by its monomial coefficients and applied by Horner in
 *                      R_n.  "+1" steps (no paper counterpart; DESIGN.md
 *                      reading R5) are Y' = Y + R, R' = A R.
 *   or_series_sum_batch -- C-1 for a batch of small independent matrices
 *                      (config 4): the same Horner sum per matrix, OpenMP
 *                      over matrices instead of rows.
 *   or_matvec       -- W = X V in long double (used to form S_gpu V on the
 *                      host for probe-mode parity).
 *
 * Parallelism: rows of each matrix-vector block product are split across
 * OpenMP threads; the summation order inside one dot product is the plain
 * left-to-right loop, so results do not depend on the thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef long double ld;

/* W[d][p] = X[d][d] * V[d][p]; X is binary64 row-major, V/W long double row-major. */
static void matvec_block(const double* X, int d, const ld* V, int p, ld* W) {
  /* Each output element is the plain left-to-right dot product
   * W[i][c] = sum_j X[i][j] V[j][c]; four columns share one pass over row i so
   * their accumulators stay in x87 registers. */
#pragma omp parallel for schedule(static)
  for (int i = 0; i < d; ++i) {
    const double* xr = X + (size_t)i * d;
    int c = 0;
    for (; c + 4 <= p; c += 4) {
      ld a0 = 0.0L, a1 = 0.0L, a2 = 0.0L, a3 = 0.0L;
      const ld* vc = V + c;
      for (int j = 0; j < d; ++j) {
        ld x = (ld)xr[j];
        const ld* vr = vc + (size_t)j * p;
        a0 += x * vr[0]; a1 += x * vr[1]; a2 += x * vr[2]; a3 += x * vr[3];
      }
      ld* wr = W + (size_t)i * p + c;
      wr[0] = a0; wr[1] = a1; wr[2] = a2; wr[3] = a3;
    }
    for (; c < p; ++c) {
      ld a0 = 0.0L;
      for (int j = 0; j < d; ++j) a0 += (ld)xr[j] * V[(size_t)j * p + c];
      W[(size_t)i * p + c] = a0;
    }
  }
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* W = X V for a binary64 matrix X and long double block V. */
int or_matvec(const double* X, int d, const ld* V, int p, ld* W) {
  if (d < 1 || p < 1 || !X || !V || !W) return 1;
  matvec_block(X, d, V, p, W);
  return 0;
}

static ld block_fro2(const ld* V, size_t n) {
  ld s = 0.0L;
  for (size_t i = 0; i < n; ++i) s += V[i] * V[i];
  return s;
}

/*
 * C-1.  out[d][p] = sum_{j=0}^{k-1} A^j V.
 *   w_0 = V, out = w_0;  for j = 1..k-1: w_j = A w_{j-1}, out += w_j.
 * If q in (0,1) is given (a certified bound ||A||_2 <= q), the loop may stop
 * after term j once  ||w_j||_F * q / (1 - q) <= tail_tol * ||out||_F ; the
 * omitted tail sum_{i>j} A^i V is then bounded in Frobenius norm by exactly
 * that quantity (||A^{i-j} w_j|| <= q^{i-j} ||w_j||).  q <= 0 disables it.
 * *terms_used receives the number of terms summed (k without early stop).
 */
int or_series_sum(const double* A, int d, int64_t k, const ld* V, int p,
                  ld q, ld tail_tol, ld* out, int64_t* terms_used) {
  if (d < 1 || p < 1 || k < 1 || !A || !V || !out) return 1;
  size_t n = (size_t)d * p;
  ld* w = (ld*)malloc(n * sizeof(ld));
  ld* w2 = (ld*)malloc(n * sizeof(ld));
  if (!w || !w2) { free(w); free(w2); return 2; }
  memcpy(w, V, n * sizeof(ld));
  memcpy(out, V, n * sizeof(ld));
  int64_t j = 1;
  for (; j < k; ++j) {
    matvec_block(A, d, w, p, w2);
    ld* t = w; w = w2; w2 = t;
    for (size_t i = 0; i < n; ++i) out[i] += w[i];
    if (q > 0.0L && q < 1.0L) {
      ld wn = sqrtl(block_fro2(w, n)), on = sqrtl(block_fro2(out, n));
      if (wn * q / (1.0L - q) <= tail_tol * on) { ++j; break; }
    }
  }
  if (terms_used) *terms_used = j;
  free(w); free(w2);
  return 0;
}

/* ---------------- C-2: plan polynomial by compositional Horner ---------------- */

typedef struct {
  const double* A; int d; int p;
  int n_steps;
  const int* kind;       /* per step: 0 = "x m" kernel step, 1 = "+1" step       */
  const int* coef_off;   /* offset of step's monomial coefficients in coefs[]    */
  const int* coef_len;   /* number of coefficients ([f]_0 .. [f]_D)              */
  const ld* coefs;
} plan_t;

static void apply_R(const plan_t* P, int i, const ld* v, ld* out);

/* out = Y_i v */
static void apply_Y(const plan_t* P, int i, const ld* v, ld* out) {
  size_t n = (size_t)P->d * P->p;
  if (i == 0) { memcpy(out, v, n * sizeof(ld)); return; }
  int s = i - 1;  /* step taking state i-1 to state i */
  if (P->kind[s] == 1) {
    /* "+1": Y_i = Y_{i-1} + R_{i-1} */
    ld* t = (ld*)malloc(n * sizeof(ld));
    apply_Y(P, i - 1, v, out);
    apply_R(P, i - 1, v, t);
    for (size_t e = 0; e < n; ++e) out[e] += t[e];
    free(t);
    return;
  }
  /* Y_i = Y_{i-1} f(R_{i-1}):  first w = f(R_{i-1}) v by Horner, then Y_{i-1} w. */
  const ld* c = P->coefs + P->coef_off[s];
  int D = P->coef_len[s] - 1;
  ld* w = (ld*)malloc(n * sizeof(ld));
  ld* t = (ld*)malloc(n * sizeof(ld));
  for (size_t e = 0; e < n; ++e) w[e] = c[D] * v[e];
  for (int j = D - 1; j >= 0; --j) {
    apply_R(P, i - 1, w, t);                       /* t = R_{i-1} w   */
    for (size_t e = 0; e < n; ++e) w[e] = t[e] + c[j] * v[e];
  }
  apply_Y(P, i - 1, w, out);
  free(w); free(t);
}

/* out = R_i v */
static void apply_R(const plan_t* P, int i, const ld* v, ld* out) {
  size_t n = (size_t)P->d * P->p;
  if (i == 0) { matvec_block(P->A, P->d, v, P->p, out); return; }   /* R_0 = A */
  int s = i - 1;
  if (P->kind[s] == 1) {
    /* "+1": R_i = A R_{i-1} */
    ld* t = (ld*)malloc(n * sizeof(ld));
    apply_R(P, i - 1, v, t);
    matvec_block(P->A, P->d, t, P->p, out);
    free(t);
    return;
  }
  /* R_i = I - M Y_i = I - Y_i + A Y_i   (M = I - A) */
  ld* y = (ld*)malloc(n * sizeof(ld));
  apply_Y(P, i, v, y);
  matvec_block(P->A, P->d, y, P->p, out);         /* out = A Y_i v */
  for (size_t e = 0; e < n; ++e) out[e] += v[e] - y[e];
  free(y);
}

/* Y_out = Y_n V and (optionally) R_out = R_n V for the plan's final state n. */
int or_plan_apply(const double* A, int d, int n_steps, const int* kind, const int* coef_off,
                  const int* coef_len, const ld* coefs, const ld* V, int p, ld* Y_out, ld* R_out) {
  if (d < 1 || p < 1 || n_steps < 0 || !A || !V || !Y_out) return 1;
  for (int s = 0; s < n_steps; ++s)
    if (kind[s] != 1 && (coef_len[s] < 1 || !coefs)) return 1;
  plan_t P = {A, d, p, n_steps, kind, coef_off, coef_len, coefs};
  apply_Y(&P, n_steps, V, Y_out);
  if (R_out) apply_R(&P, n_steps, V, R_out);
  return 0;
}

/*
 * C-1 for `batch` independent matrices (config 4's batched small path):
 *   out_b[d][p] = sum_{j=0}^{k-1} A_b^j V_b, b = 0..batch-1,
 * A_b at A + b*d*d (binary64), V_b / out_b at V / out + b*d*p (long double).
 * Per matrix the plain power sum of or_series_sum (w <- A w,
 * out += w) with the plain left-to-right dot product; the parallel loop runs
 * over matrices, so the result of each matrix does not depend on threads.
 */
int or_series_sum_batch(const double* A, int batch, int d, int64_t k, const ld* V, int p, ld* out) {
  if (batch < 0 || d < 1 || p < 1 || k < 1 || (batch > 0 && (!A || !V || !out))) return 1;
  const size_t n = (size_t)d * p;
  int bad = 0;
#pragma omp parallel
  {
    ld* w = (ld*)malloc(n * sizeof(ld));
    ld* w2 = (ld*)malloc(n * sizeof(ld));
    if (!w || !w2) {
#pragma omp atomic write
      bad = 2;
    }
#pragma omp for schedule(dynamic, 16)
    for (int b = 0; b < batch; ++b) {
      if (!w || !w2) continue;
      const double* Ab = A + (size_t)b * d * d;
      ld* ob = out + (size_t)b * n;
      memcpy(w, V + (size_t)b * n, n * sizeof(ld));
      memcpy(ob, w, n * sizeof(ld));
      for (int64_t j = 1; j < k; ++j) {
        for (int i = 0; i < d; ++i)
          for (int c = 0; c < p; ++c) {
            ld acc = 0.0L;
            for (int q = 0; q < d; ++q) acc += (ld)Ab[(size_t)i * d + q] * w[(size_t)q * p + c];
            w2[(size_t)i * p + c] = acc;
          }
        ld* t = w; w = w2; w2 = t;
        for (size_t i = 0; i < n; ++i) ob[i] += w[i];
      }
    }
    free(w);
    free(w2);
  }
  return bad;
}
