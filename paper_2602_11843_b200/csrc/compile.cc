// compile.cc -- plan -> list of fused GEMM ops with workspace slot assignment (host C++).
//
// State per step is the pair (S, B): (S_n, A^n) in the telescoping framework
// or (Y_n, R_n) in the residual framework.  The two coincide for exact
// kernels, so one state machine serves all steps.  Operands of the form
// X +- I are never materialised: every linear combination of the circuits, the concatenation
// and the power / residual updates is an epilogue of the GEMM that produces its last term
// (SURVEY.md 8(a) rows a-3..a-6).  I is implicit (gamma coefficients) except where the paper's
// counting multiplies by S_1 = I (then the identity buffer is a real GEMM operand).
#include <algorithm>
#include <initializer_list>
#include <utility>

#include "internal.h"

namespace nseries {
namespace {

struct Builder {
  Program& P;
  int ident;
  int userA;

  explicit Builder(Program& p) : P(p) {
    userA = newval(V_USER_A);
    ident = newval(V_IDENT);
  }
  int newval(int kind) {
    P.val_kind.push_back(kind);
    return P.n_values++;
  }
  Op& gemm(int X, int Y, int step, const char* tag) {
    Op op;
    op.gemm = true;
    op.X = X;
    op.Y = Y;
    op.step = step;
    op.tag = tag;
    if (X == ident || Y == ident) P.needs_identity = true;
    P.ops.push_back(op);
    return P.ops.back();
  }
  Op& axpby(int step, const char* tag) {
    Op op;
    op.gemm = false;
    op.step = step;
    op.tag = tag;
    P.ops.push_back(op);
    return P.ops.back();
  }
  // Add an output  alpha*acc + sum terms + gamma*I  to op; returns the new value id.
  int out(Op& op, double alpha, std::initializer_list<std::pair<int, double>> terms,
          double gamma = 0.0) {
    int j = op.n_out++;
    op.alpha[j] = alpha;
    op.gamma[j] = gamma;
    for (auto& t : terms) {
      if (t.second == 0.0) continue;
      if (t.first == ident) {               // I is generated from tile coordinates
        op.gamma[j] += t.second;
        continue;
      }
      int a = -1;
      for (int i = 0; i < op.n_aux; ++i)
        if (op.aux[i] == t.first) a = i;
      if (a < 0) {
        a = op.n_aux++;
        op.aux[a] = t.first;
      }
      op.beta[j][a] += t.second;
    }
    int v = newval(V_TEMP);
    op.out[j] = v;
    return v;
  }
};

}  // namespace

nseries_status compile_plan(const nseries_plan& plan, bool want_R, Program* prog) {
  Program& P = *prog;
  P = Program();
  size_t n_ops_max = 8;
  for (int i = 0; i < plan.n_steps; ++i) n_ops_max += (size_t)std::max(kernel_mu(plan.step[i]), 1) + 2;
  P.ops.reserve(n_ops_max);   // Op& references stay valid while building
  Builder b(P);
  const bool elide = (plan.flags & NSERIES_ELIDE_TRIVIAL) != 0;
  int S = b.ident;   // S_1 = I  (Y_0 = I)
  int B = b.userA;   // A^1 = A  (R_0 = A)
  const int A = b.userA, I = b.ident;
  const int n = plan.n_steps;

  for (int i = 0; i < n; ++i) {
    if (i > 0) { P.step_S.push_back(S); P.step_B.push_back(B); }
    const int m = plan.step[i];
    const bool first = (i == 0), last = (i + 1 == n);
    const bool skip_concat = elide && first;        // S_1 = I: concatenation is a copy
    // the final power is "unused" (elided) only when the caller does not ask for R_out
    const bool need_power = !(elide && last) || want_R;
    if (m == 1) {
      // "+1": B' = B A, S' = S + B  (residual form: R' = A R, Y' = Y + R)      [reading R5]
      Op& op = b.gemm(B, A, i, "plus1");
      int Bn = b.out(op, 1.0, {}, 0.0);
      int Sn = b.out(op, 0.0, {{S, 1.0}, {B, 1.0}});
      S = Sn;
      B = Bn;
      continue;
    }
    if (m == 2) {
      // binary splitting: S' = S (I + B), B' = B B
      if (skip_concat) {
        if (need_power) {
          Op& op = b.gemm(B, B, i, "x2.square");
          int Bn = b.out(op, 1.0, {});
          int Sn = b.out(op, 0.0, {{B, 1.0}}, 1.0);
          S = Sn;
          B = Bn;
        } else {
          Op& op = b.axpby(i, "x2.I+B");
          S = b.out(op, 0.0, {{B, 1.0}}, 1.0);
        }
      } else {
        Op& op1 = b.gemm(S, B, i, "x2.concat");
        int Sn = b.out(op1, 1.0, {{S, 1.0}});
        int Bn = B;
        if (need_power) {
          Op& op2 = b.gemm(B, B, i, "x2.square");
          Bn = b.out(op2, 1.0, {});
        }
        S = Sn;
        B = Bn;
      }
      continue;
    }
    int T = -1;   // kernel value T_m(B) / f(R)
    int f_for_tele = -1;
    if (m == 3 || (m != 5 && m != 9 && m != 15 && kernel_mu(m) == m - 2)) {
      // ternary and naive radix-m splitting: the powers
      // B^2 = B B, B^j = B^{j-1} B (m - 2 products), T_m = I + B + ... + B^{m-1} accumulated
      // in the same epilogues (T_j = T_{j-1} + B^j); concatenation and next power below
      Op& g1 = b.gemm(B, B, i, m == 3 ? "x3.U" : "xm.P2");
      int Tacc = b.out(g1, 1.0, {{B, 1.0}}, 1.0);           // I + B + B^2
      int Pj = m > 3 ? b.out(g1, 1.0, {}) : -1;             // B^2
      for (int j = 3; j < m; ++j) {
        Op& gj = b.gemm(Pj, B, i, "xm.Pj");                   // acc = B^j
        const int Tn = b.out(gj, 1.0, {{Tacc, 1.0}});
        Pj = j + 1 < m ? b.out(gj, 1.0, {}) : -1;
        Tacc = Tn;
      }
      T = Tacc;
    } else if (m == 5) {
      // quinary (Eqs. quinary-U/V/final 866-873)
      Op& g1 = b.gemm(B, B, i, "x5.U");
      int U = b.out(g1, 1.0, {});
      int F = b.out(g1, 1.0, {{B, 1.0}});                   // B + U
      Op& g2 = b.gemm(U, F, i, "x5.V");
      T = b.out(g2, 1.0, {{B, 1.0}, {U, 1.0}}, 1.0);        // I + B + U + V
    } else if (m == 9) {
      // radix-9, Theorem 1
      Op& g1 = b.gemm(B, B, i, "x9.U");
      int U = b.out(g1, 1.0, {});
      int F = b.out(g1, 2.0, {{B, 1.0}});                   // B + 2U
      Op& g2 = b.gemm(U, F, i, "x9.V");                     // acc = V = B^3 + 2B^4
      int Pm = b.out(g2, 1.0, {{B, 3.0 / 20.0}, {U, 2.0}});                 // P = 3/20 B + 2U + V
      int Qm = b.out(g2, 1.0 / 4.0, {{B, 11.0 / 40.0}, {U, -1.0 / 8.0}});  // Q = 11/40 B - 1/8 U + 1/4 V
      int Tp = b.out(g2, 15.0 / 32.0, {{B, 1.0}, {U, 767.0 / 800.0}}, 1.0); // I + B + 767/800 U + 15/32 V
      Op& g3 = b.gemm(Pm, Qm, i, "x9.W");
      T = b.out(g3, 1.0, {{Tp, 1.0}});                      // T = W + Tp
    } else if (m == 15) {
      // radix-15 circuit (parameters: reading R1)
      const Radix15Params& p = radix15_params();
      Op& g1 = b.gemm(B, B, i, "x15.P1");
      int P1 = b.out(g1, 1.0, {});
      int L2 = b.out(g1, p.L2[2], {{B, p.L2[1]}}, p.L2[0]);
      int R2 = b.out(g1, p.R2[2], {{B, p.R2[1]}}, p.R2[0]);
      Op& g2 = b.gemm(L2, R2, i, "x15.P2");
      int P2 = b.out(g2, 1.0, {});
      int L3 = b.out(g2, p.L3[3], {{B, p.L3[1]}, {P1, p.L3[2]}}, p.L3[0]);
      int R3 = b.out(g2, p.R3[3], {{B, p.R3[1]}, {P1, p.R3[2]}}, p.R3[0]);
      Op& g3 = b.gemm(L3, R3, i, "x15.P3");                 // acc = P3 (not stored)
      int L4 = b.out(g3, p.L4[4], {{B, p.L4[1]}, {P1, p.L4[2]}, {P2, p.L4[3]}}, p.L4[0]);
      int R4 = b.out(g3, p.R4[4], {{B, p.R4[1]}, {P1, p.R4[2]}, {P2, p.R4[3]}}, p.R4[0]);
      int Fp = b.out(g3, p.gamma[3], {{B, p.gamma[0]}, {P1, p.gamma[1]}, {P2, p.gamma[2]}}, 1.0);
      Op& g4 = b.gemm(L4, R4, i, "x15.P4");
      T = b.out(g4, 1.0, {{Fp, 1.0}});                      // f = I + g1 B + g2 P1 + g3 P2 + g4 P3 + P4
    } else {
      return NSERIES_ERR_UNSUPPORTED_RADIX;
    }
    f_for_tele = T;
    // concatenation S' = S T   (residual: Y' = Y f(R))
    int Sn;
    if (skip_concat) {
      Sn = T;
    } else {
      Op& gc = b.gemm(S, T, i, "concat");
      Sn = b.out(gc, 1.0, {});
    }
    // power / residual update
    int Bn = B;
    if (need_power) {
      if (plan.form[i] == 1) {
        // paper residual form R' = I - M Y' = I - Y' + A Y'
        Op& gr = b.gemm(A, Sn, i, "residual");
        Bn = b.out(gr, 1.0, {{Sn, -1.0}}, 1.0);
      } else {
        // telescoping I - T(I - B) = I - T + T B; for an
        // approximate f this is E(R) = I - (I - R) f(R)   (form 2)
        Op& gr = b.gemm(f_for_tele, B, i, "power");
        Bn = b.out(gr, 1.0, {{f_for_tele, -1.0}}, 1.0);
      }
    }
    S = Sn;
    B = Bn;
  }

  if (n > 0) { P.step_S.push_back(S); P.step_B.push_back(B); }
  // final S -> user S; final B -> user R (optional)
  if (S == I) {   // k = 1: S = I   (degenerate, no product)
    Op& op = b.axpby(-1, "k1.identity");
    S = b.out(op, 0.0, {}, 1.0);
  }
  if (want_R && B == A) {   // k = 1 (or elided k=2 binary): R = A^k needs a copy
    Op& op = b.axpby(-1, "copy.R");
    B = b.out(op, 0.0, {{A, 1.0}});
  }
  P.val_kind[S] = V_USER_S;
  P.final_S = S;
  if (want_R) {
    if (P.val_kind[B] != V_TEMP) {   // final B is the user S value (cannot happen) -> copy
      Op& op = b.axpby(-1, "copy.R");
      B = b.out(op, 0.0, {{B, 1.0}});
    }
    P.val_kind[B] = V_USER_R;
    P.final_R = B;
  }

  // ---- liveness + slot assignment for V_TEMP values
  const int nv = P.n_values;
  std::vector<int> last_use(nv, -1), producer(nv, -1);
  for (int i = 0; i < (int)P.ops.size(); ++i) {
    const Op& op = P.ops[i];
    if (op.gemm) { last_use[op.X] = i; last_use[op.Y] = i; }
    for (int a = 0; a < op.n_aux; ++a) last_use[op.aux[a]] = i;
    for (int j = 0; j < op.n_out; ++j) producer[op.out[j]] = i;
  }
  for (int v = 0; v < nv; ++v)
    if (last_use[v] < producer[v]) last_use[v] = producer[v];
  P.val_buf.assign(nv, -1);
  std::vector<int> free_slots;
  int n_slots = 0;
  for (int i = 0; i < (int)P.ops.size(); ++i) {
    const Op& op = P.ops[i];
    for (int j = 0; j < op.n_out; ++j) {
      int v = op.out[j];
      if (P.val_kind[v] != V_TEMP) continue;
      int s;
      if (!free_slots.empty()) { s = free_slots.back(); free_slots.pop_back(); }
      else s = n_slots++;
      P.val_buf[v] = s;
    }
    for (int v = 0; v < nv; ++v)
      if (last_use[v] == i && P.val_buf[v] >= 0) free_slots.push_back(P.val_buf[v]);
  }
  P.n_slots = n_slots;
  int prods = 0;
  for (const Op& op : P.ops) prods += op.gemm ? 1 : 0;
  P.products = prods;
  // internal consistency; an elided plan asked for R_out computes its final power (+1)
  const int extra = (elide && want_R && n > 0 && plan.step[n - 1] != 1) ? 1 : 0;
  if (prods != plan.products + extra) return NSERIES_ERR_INVALID_ARG;
  return NSERIES_OK;
}

}  // namespace nseries

namespace nseries {

// Slot assignment for the shared-memory executors.  inplace = true: for executors whose ops read
// every operand before writing any output (the warp-per-matrix batched kernel computes a whole
// product in registers): a value whose last use is op i frees its slot BEFORE op i's outputs
// are placed, so an output may overwrite an operand or aux it was computed from.  inplace =
// false: outputs never share a slot with a value read by the same op (the cluster kernel, whose
// CTAs read each other's operand rows while writing their own outputs).  Only values with
// needs_slot[v] get a slot; the others get -1.
int assign_slots_inplace(const Program& P, const std::vector<bool>& needs_slot,
                         std::vector<int>* slot_of_value, bool inplace) {
  const int nv = P.n_values;
  std::vector<int> last_use(nv, -1), producer(nv, -1);
  for (int i = 0; i < (int)P.ops.size(); ++i) {
    const Op& op = P.ops[i];
    if (op.gemm) { last_use[op.X] = i; last_use[op.Y] = i; }
    for (int a = 0; a < op.n_aux; ++a) last_use[op.aux[a]] = i;
    for (int j = 0; j < op.n_out; ++j) producer[op.out[j]] = i;
  }
  std::vector<int>& slot = *slot_of_value;
  slot.assign(nv, -1);
  std::vector<int> free_slots;
  int n_slots = 0;
  for (int i = 0; i < (int)P.ops.size(); ++i) {
    const Op& op = P.ops[i];
    if (inplace)
      for (int v = 0; v < nv; ++v)
        if (last_use[v] == i && slot[v] >= 0 && producer[v] < i) free_slots.push_back(slot[v]);
    for (int j = 0; j < op.n_out; ++j) {
      int v = op.out[j];
      if (!needs_slot[v]) continue;
      int s;
      if (!free_slots.empty()) { s = free_slots.back(); free_slots.pop_back(); }
      else s = n_slots++;
      slot[v] = s;
    }
    if (!inplace)   // operands / aux dying here are freed only after the outputs are placed
      for (int v = 0; v < nv; ++v)
        if (last_use[v] == i && slot[v] >= 0 && producer[v] < i) free_slots.push_back(slot[v]);
    // outputs never read again (e.g. the final power in the paper's counting) die at once
    for (int j = 0; j < op.n_out; ++j) {
      int v = op.out[j];
      if (slot[v] >= 0 && last_use[v] < 0) free_slots.push_back(slot[v]);
    }
  }
  return n_slots;
}

}  // namespace nseries

namespace nseries {
std::vector<int> value_last_use(const Program& P) {
  std::vector<int> last_use(P.n_values, -1);
  for (int i = 0; i < (int)P.ops.size(); ++i) {
    const Op& op = P.ops[i];
    if (op.gemm) { last_use[op.X] = i; last_use[op.Y] = i; }
    for (int a = 0; a < op.n_aux; ++a) last_use[op.aux[a]] = i;
  }
  return last_use;
}
}  // namespace nseries
