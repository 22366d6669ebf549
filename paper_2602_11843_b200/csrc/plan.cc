// plan.cc -- kernel circuit tables and the fewest-product plan builder (host C++).
//
// Cost model: one radix-m update costs C(m) = mu_m + 2 products (kernel,
// concatenation S_{mn} = S_n T_m(A^n), next power / residual).  The residual framework has the
// same cost (Eq. generalcost).  A "+1" step S_{n+1} = S_n + A^n,
// A^{n+1} = A^n A costs one product (reading R5).
#include <cmath>
#include <cstring>
#include <map>
#include <vector>

#include "internal.h"

namespace nseries {

// Polished radix-15 circuit (reading R1): the minimum-norm projection of the printed
// Appendix B parameters onto the exact-prefix manifold [f]_j = 1, j <= 14.
// Every value rounds to the printed 3 decimals.  Transcribed from SURVEY.md Appendix B
// (an independent computation from the oracle's own polish; tests compare the two).
static const Radix15Params kRadix15 = {
    /*L2*/ {0.23798562608592442714, 0.24132143289582745154, 1.5739454994873966057},
    /*R2*/ {0.047794178281130494098, -0.046503130075732822141, 0.88902417651856190023},
    /*L3*/ {0.26298160043686175756, 0.91880846825430773215, 0.84207398441870344515,
            0.81923074341166513175},
    /*R3*/ {0.1838768351522736632, 0.068226111280048395974, 0.13415513230878943561,
            -1.4050405093708177266},
    /*L4*/ {-0.0045843624901695308791, -1.385012555109953889, 0.021935800067016966607,
            0.12214402366871098804, 0.27484644418371743566},
    /*R4*/ {-0.70108400659942373242, 0.60160009408829510405, -0.62407662189370208321,
            -0.13710451318328109982, 0.32833221202427062201},
    /*gamma*/ {0.077997690670988478238, 1.7781979706155444214, 0.66356397165443442187,
               -0.024153284107253202139},
};

const Radix15Params& radix15_params() { return kRadix15; }

int kernel_mu(int m) {
  switch (m) {
    case 2: return 0;   // T_2 = I + B
    case 3: return 1;   // U = B^2, T_3 = I + B + U (ternary)
    case 5: return 2;   // U = B^2, V = U(B+U)
    case 9: return 3;   // U, V = U(B+2U), W = PQ
    case 15: return 4;  // P1..P4
    default:            // naive radix-m splitting: powers B^2 .. B^{m-1} PAPER.md:140-151
      return (m >= 4 && m <= kMaxNaiveRadix) ? m - 2 : -1;
  }
}

bool kernel_exact(int m) { return kernel_mu(m) >= 0 && m != 15; }

using Poly = std::vector<double>;
static Poly pmul(const Poly& a, const Poly& b) {
  Poly r(a.size() + b.size() - 1, 0.0);
  for (size_t i = 0; i < a.size(); ++i)
    for (size_t j = 0; j < b.size(); ++j) r[i + j] += a[i] * b[j];
  return r;
}
static Poly padd(const Poly& a, const Poly& b, double s) {
  Poly r(std::max(a.size(), b.size()), 0.0);
  for (size_t i = 0; i < a.size(); ++i) r[i] += a[i];
  for (size_t i = 0; i < b.size(); ++i) r[i] += s * b[i];
  return r;
}
static Poly lin(const std::vector<Poly>& basis, const double* w, int n) {
  Poly r{0.0};
  for (int i = 0; i < n; ++i) r = padd(r, basis[i], w[i]);
  return r;
}

std::vector<double> kernel_poly(int m) {
  const Poly I{1.0}, B{0.0, 1.0};
  if (m == 2) return {1.0, 1.0};
  if (m == 3) return padd(padd(I, B, 1.0), pmul(B, B), 1.0);
  if (m != 5 && m != 9 && m != 15 && kernel_mu(m) == m - 2) {
    // naive radix-m: T_m = I + B + B^2 + ... + B^{m-1} through the power chain B^j = B^{j-1} B
    Poly T = padd(I, B, 1.0), Pj = B;
    for (int j = 2; j < m; ++j) {
      Pj = pmul(Pj, B);
      T = padd(T, Pj, 1.0);
    }
    return T;
  }
  if (m == 5) {
    Poly U = pmul(B, B), V = pmul(U, padd(B, U, 1.0));
    return padd(padd(padd(I, B, 1.0), U, 1.0), V, 1.0);
  }
  if (m == 9) {
    Poly U = pmul(B, B), V = pmul(U, padd(B, U, 2.0));
    Poly P = padd(padd(padd(Poly{0.0}, B, 0.15), U, 2.0), V, 1.0);
    Poly Q = padd(padd(padd(Poly{0.0}, B, 0.275), U, -0.125), V, 0.25);
    Poly W = pmul(P, Q);
    Poly T = padd(padd(padd(padd(W, I, 1.0), B, 1.0), U, 767.0 / 800.0), V, 15.0 / 32.0);
    return T;
  }
  if (m == 15) {
    const Radix15Params& p = kRadix15;
    std::vector<Poly> basis{I, B, pmul(B, B)};
    basis.push_back(pmul(lin(basis, p.L2, 3), lin(basis, p.R2, 3)));
    basis.push_back(pmul(lin(basis, p.L3, 4), lin(basis, p.R3, 4)));
    Poly P4 = pmul(lin(basis, p.L4, 5), lin(basis, p.R4, 5));
    Poly f = padd(I, basis[1], p.gamma[0]);
    f = padd(f, basis[2], p.gamma[1]);
    f = padd(f, basis[3], p.gamma[2]);
    f = padd(f, basis[4], p.gamma[3]);
    f = padd(f, P4, 1.0);
    while (f.size() > 1 && f.back() == 0.0) f.pop_back();
    return f;
  }
  return {};
}

// ---------------------------------------------------------------- plan builder

int step_products(int step, bool first, bool last, uint32_t flags) {
  if (step == 1) return 1;
  int c = kernel_mu(step) + 2;
  if (flags & NSERIES_ELIDE_TRIVIAL) {
    if (first) c -= 1;   // concatenation with S_1 = I
    if (last) c -= 1;    // final power / residual not needed
  }
  return c;
}

namespace {

struct Key {
  int products, plus, steps;
  std::vector<int> lex;   // -step, compared lexicographically (larger radix first)
  bool operator<(const Key& o) const {
    if (products != o.products) return products < o.products;
    if (plus != o.plus) return plus < o.plus;
    if (steps != o.steps) return steps < o.steps;
    return lex < o.lex;
  }
};

Key key_of(const std::vector<int>& s, bool final_discount, uint32_t flags) {
  Key k{0, 0, (int)s.size(), {}};
  for (size_t i = 0; i < s.size(); ++i) {
    bool last = final_discount && (i + 1 == s.size());
    k.products += step_products(s[i], i == 0, last, flags);
    k.plus += s[i] == 1;
    k.lex.push_back(-s[i]);
  }
  return k;
}

struct Searcher {
  std::vector<int> radices;
  uint32_t flags;
  std::map<int64_t, std::vector<int>> memo;
  std::map<int64_t, bool> ok;

  // Best plan from 1 to T (no final-step discount).  Only non-dominated plans are explored:
  // a run of "+1" steps directly followed by "x m" (or ending the plan after "x m") is never
  // longer than m-1, so T -> floor(T/m) with T mod m trailing "+1".
  bool best(int64_t T, bool top, std::vector<int>* out) {
    if (!top) {
      auto it = ok.find(T);
      if (it != ok.end()) {
        if (it->second) *out = memo[T];
        return it->second;
      }
    }
    bool have = false;
    std::vector<int> bestseq;
    Key bestkey;
    auto consider = [&](std::vector<int>&& cand) {
      if (cand.size() > NSERIES_MAX_STEPS) return;
      Key kk = key_of(cand, top, flags);
      if (!have || kk < bestkey) { have = true; bestkey = kk; bestseq = std::move(cand); }
    };
    if (T == 1) {
      have = true;
      bestseq.clear();
    } else {
      if (T - 1 <= NSERIES_MAX_STEPS) consider(std::vector<int>((size_t)(T - 1), 1));
      for (int m : radices) {
        int64_t pred = T / m, r = T % m;
        if (pred < 1) continue;
        std::vector<int> pre;
        if (!best(pred, false, &pre)) continue;
        pre.push_back(m);
        for (int64_t i = 0; i < r; ++i) pre.push_back(1);
        consider(std::move(pre));
      }
    }
    if (!top) {
      ok[T] = have;
      if (have) memo[T] = bestseq;
    }
    if (have) *out = bestseq;
    return have;
  }
};

}  // namespace

nseries_status finalize_plan(nseries_plan* plan, int64_t k, uint32_t flags) {
  if (!plan || k < 1 || plan->n_steps < 0 || plan->n_steps > NSERIES_MAX_STEPS)
    return NSERIES_ERR_INVALID_ARG;
  __int128 n = 1;
  int approx = 0, products = 0;
  for (int i = 0; i < plan->n_steps; ++i) {
    int s = plan->step[i];
    if (s != 1 && kernel_mu(s) < 0) return NSERIES_ERR_UNSUPPORTED_RADIX;
    if (s == 15) {
      if (!(flags & NSERIES_ALLOW_APPROX)) return NSERIES_ERR_APPROX_TELESCOPE;
      approx = 1;
      plan->form[i] = (flags & NSERIES_RFORM_TELESCOPE) ? 2 : 1;
    } else {
      plan->form[i] = 0;
    }
    n = (s == 1) ? n + 1 : n * s;
    if (n > ((__int128)1 << 62)) return NSERIES_ERR_PLAN_K_MISMATCH;
    products += step_products(s, i == 0, i + 1 == plan->n_steps, flags);
  }
  if (n != k) return NSERIES_ERR_PLAN_K_MISMATCH;
  for (int i = plan->n_steps; i < NSERIES_MAX_STEPS; ++i) { plan->step[i] = 0; plan->form[i] = 0; }
  plan->products = products;
  plan->approx = approx;
  plan->flags = flags & (NSERIES_ELIDE_TRIVIAL | NSERIES_ALLOW_APPROX | NSERIES_RFORM_TELESCOPE);
  plan->k = k;
  return NSERIES_OK;
}

nseries_status build_plan(int64_t k, nseries_plan_kind kind, const int32_t* radices, int32_t n,
                          uint32_t flags, nseries_plan* out) {
  if (!out || k < 1 || k > ((int64_t)1 << 62)) return NSERIES_ERR_INVALID_ARG;
  std::memset(out, 0, sizeof(*out));
  std::vector<int> steps;
  if ((int)kind >= 2 && kernel_mu((int)kind) >= 0) {   // pure radix-m plan (any supported m)
    int m = (int)kind;
    if (m == 15 && !(flags & NSERIES_ALLOW_APPROX)) flags |= NSERIES_ALLOW_APPROX;  // explicit request
    int64_t v = 1;
    while (v < k) {
      v *= m;
      steps.push_back(m);
      if ((int)steps.size() > NSERIES_MAX_STEPS) return NSERIES_ERR_PLAN_K_MISMATCH;
    }
    if (v != k) return NSERIES_ERR_PLAN_K_MISMATCH;   // pure plans: k = m^t
  } else if (kind == NSERIES_PLAN_AUTO) {
    Searcher s;
    s.flags = flags;
    if (radices && n > 0) {
      for (int i = 0; i < n; ++i) {
        if (kernel_mu(radices[i]) < 0) return NSERIES_ERR_UNSUPPORTED_RADIX;
        if (radices[i] == 15 && !(flags & NSERIES_ALLOW_APPROX)) return NSERIES_ERR_APPROX_TELESCOPE;
        s.radices.push_back(radices[i]);
      }
    } else {
      s.radices = {9, 5, 2};
      if (flags & NSERIES_ALLOW_APPROX) s.radices.insert(s.radices.begin(), 15);
    }
    if (!s.best(k, true, &steps)) return NSERIES_ERR_PLAN_K_MISMATCH;
  } else {
    return NSERIES_ERR_INVALID_ARG;
  }
  out->n_steps = (int32_t)steps.size();
  for (size_t i = 0; i < steps.size(); ++i) out->step[i] = steps[i];
  return finalize_plan(out, k, flags);
}

}  // namespace nseries
