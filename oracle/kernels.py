"""Kernel circuits as scalar polynomials -- TEST INFRASTRUCTURE ONLY (oracle side).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import
anything under oracle/.  Nothing here is shared with the CUDA library.

Each radix kernel of the paper is a *circuit*: a short list of products
P_i = L_i * R_i whose factors are linear combinations of earlier basis
elements {I, B, P_1, ...}, followed by a final linear combination
(Eq. factors / Eq. radix15kernel).  Replacing
B by the indeterminate z turns the circuit into a polynomial f(z); its monomial
coefficients [f]_j are what the C oracle's compositional Horner
consumes.

Circuits encoded here, each following the paper's text line by line:
  * T_2 binary:    f = 1 + z
  * T_3 ternary:   U = B^2; T = I + B + U
  * T_m naive:     P_2 = B^2, P_j = P_{j-1} B; T = I + B + P_2 + ... + P_{m-1}
                   (m = 4..32 except 5, 9, 15)
  * T_5 quinary:   U = B^2; V = U(B+U); T = I+B+U+V
  * T_9 radix-9:   U = B^2; V = U(B+2U); P = 3/20 B + 2U + V;
                   Q = 11/40 B - 1/8 U + 1/4 V; W = PQ;
                   T = W + I + B + 767/800 U + 15/32 V
  * T~15 radix-15: P1 = B^2; P_i = L_i R_i over {I,B,P1..P_{i-1}};
                   f = I + g1 B + g2 P1 + g3 P2 + g4 P3 + P4
    with either the printed 3-decimal parameters or the
    polished parameters produced by oracle/polish_radix15.py (reading R1).
"""
from __future__ import annotations

import json
import os
from fractions import Fraction

_HERE = os.path.dirname(os.path.abspath(__file__))

# ---------------------------------------------------------------- polynomial helpers


def poly_mul(a, b):
    """Coefficient convolution [a*b]_j = sum_i [a]_i [b]_{j-i}."""
    if not a or not b:
        return []
    out = [0 * a[0]] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        if x == 0:
            continue
        for j, y in enumerate(b):
            out[i + j] = out[i + j] + x * y
    return out


def poly_add_scaled(acc, p, s):
    if len(acc) < len(p):
        acc = acc + [0 * s] * (len(p) - len(acc))
    acc = list(acc)
    for i, x in enumerate(p):
        acc[i] = acc[i] + s * x
    return acc


def eval_circuit(steps, final, one=Fraction(1)):
    """Evaluate a circuit symbolically.

    steps: list of (left, right) where left/right are lists of weights over the
           basis [I, B, P_1, ..., P_{i-1}] (shorter lists pad with zeros).
    final: weights over [I, B, P_1, ..., P_mu].
    Returns the coefficient list of f(z).
    """
    zero = one - one
    basis = [[one], [zero, one]]  # I -> 1, B -> z
    for left, right in steps:
        lp, rp = [], []
        for w, x in zip(left, basis):
            if w != 0:
                lp = poly_add_scaled(lp, x, w)
        for w, x in zip(right, basis):
            if w != 0:
                rp = poly_add_scaled(rp, x, w)
        basis.append(poly_mul(lp, rp))
    f = []
    for w, x in zip(final, basis):
        if w != 0:
            f = poly_add_scaled(f, x, w)
    while len(f) > 1 and f[-1] == 0:
        f.pop()
    return f


# ---------------------------------------------------------------- the paper's circuits

F = Fraction


def circuit_binary():
    """T_2(B) = I + B, no products."""
    return [], [F(1), F(1)]


def circuit_ternary():
    """Ternary splitting kernel T_3 = I + B + B^2: one product.
    basis: [I, B, U]."""
    steps = [([0, 1], [0, 1])]                                  # U = B * B
    final = [F(1), F(1), F(1)]
    return steps, final


def circuit_naive(m):
    """Naive radix-m splitting kernel ("Radix-m splitting"): the powers
    A^{2n}, ..., A^{(m-1)n} from A^n -- P_2 = B * B, P_j = P_{j-1} * B (m - 2 products) --
    and T_m = I + B + P_2 + ... + P_{m-1}.  basis: [I, B, P_2, ..., P_{m-1}]."""
    if m < 3:
        raise ValueError("naive radix-m needs m >= 3 (m = 2 is binary splitting)")
    steps = [([0, 1], [0, 1])]                                  # P_2 = B * B
    for j in range(3, m):
        left = [0] * j
        left[j - 1] = 1                                         # P_{j-1} (basis index j - 1)
        steps.append((left, [0, 1]))                            # P_j = P_{j-1} * B
    final = [F(1)] * m
    return steps, final


def circuit_quinary():
    """Gustafsson et al. quinary kernel, PAPER.md:229-235 / Eqs. quinary-U,V,final (866-873).
    basis: [I, B, U, V]."""
    steps = [
        ([0, 1], [0, 1]),          # U = B * B
        ([0, 0, 1], [0, 1, 1]),    # V = U * (B + U)
    ]
    final = [F(1), F(1), F(1), F(1)]  # T = I + B + U + V
    return steps, final


def circuit_radix9(c_u=F(767, 800), c_v=F(15, 32)):
    """Theorem 1: basis [I, B, U, V, W]."""
    steps = [
        ([0, 1], [0, 1]),                                    # MM1: U = B^2
        ([0, 0, 1], [0, 1, 2]),                              # MM2: V = U (B + 2U)
        ([0, F(3, 20), 2, 1], [0, F(11, 40), F(-1, 8), F(1, 4)]),  # MM3: W = P Q
    ]
    final = [F(1), F(1), c_u, c_v, F(1)]                    # T = W + I + B + 767/800 U + 15/32 V
    return steps, final


# Appendix B, printed to 3 decimals.
RADIX15_PRINTED = {
    "L2": ["0.238", "0.241", "1.574"],
    "R2": ["0.048", "-0.047", "0.889"],
    "L3": ["0.263", "0.919", "0.842", "0.819"],
    "R3": ["0.184", "0.068", "0.134", "-1.405"],
    "L4": ["-0.005", "-1.385", "0.022", "0.122", "0.275"],
    "R4": ["-0.701", "0.602", "-0.624", "-0.137", "0.328"],
    "gamma": ["0.078", "1.778", "0.664", "-0.024"],
}
PARAM_ORDER = ["L2", "R2", "L3", "R3", "L4", "R4", "gamma"]


def radix15_flat(params):
    out = []
    for key in PARAM_ORDER:
        out.extend(params[key])
    return out


def radix15_unflat(flat):
    sizes = {"L2": 3, "R2": 3, "L3": 4, "R3": 4, "L4": 5, "R4": 5, "gamma": 4}
    out, i = {}, 0
    for key in PARAM_ORDER:
        out[key] = list(flat[i:i + sizes[key]])
        i += sizes[key]
    return out


def circuit_radix15(params, one=Fraction(1)):
    """Eq. factors + Eq. radix15kernel.  basis [I, B, P1, P2, P3, P4]."""
    zero = one - one
    steps = [
        ([zero, one], [zero, one]),              # P1 = B^2
        (params["L2"], params["R2"]),            # P2 = L2 R2 over {I,B,P1}
        (params["L3"], params["R3"]),            # P3 = L3 R3 over {I,B,P1,P2}
        (params["L4"], params["R4"]),            # P4 = L4 R4 over {I,B,P1,P2,P3}
    ]
    g = params["gamma"]
    final = [one, g[0], g[1], g[2], g[3], one]   # I + g1 B + g2 P1 + g3 P2 + g4 P3 + P4
    return steps, final


def printed_radix15_fractions():
    return {k: [F(x) for x in v] for k, v in RADIX15_PRINTED.items()}


def polished_radix15_strings():
    """Polished parameters written by oracle/polish_radix15.py (50+ digits)."""
    with open(os.path.join(_HERE, "radix15_polished.json")) as fh:
        return json.load(fh)["params"]


def polished_radix15_binary64():
    """Polished parameters rounded to IEEE binary64 (what a binary64 circuit uses)."""
    return {k: [float(x) for x in v] for k, v in polished_radix15_strings().items()}


def radix15_binary64_fractions():
    """The binary64-rounded polished parameters as exact rationals."""
    return {k: [F(x) for x in v] for k, v in polished_radix15_binary64().items()}


# ---------------------------------------------------------------- coefficient vectors


def kernel_coeffs(m, variant="polished"):
    """Monomial coefficients [f]_0..[f]_D of the radix-m kernel as exact Fractions.

    m in {2, 5, 9}: exact circuits (all-ones, length m).
    m == 15: circuit with binary64-rounded polished parameters (variant="polished")
             or the printed 3-decimal ones (variant="printed"); exact rational
             convolution of those parameters.
    """
    if m == 2:
        steps, final = circuit_binary()
    elif m == 3:
        steps, final = circuit_ternary()
    elif m in NAIVE:
        steps, final = circuit_naive(m)
    elif m == 5:
        steps, final = circuit_quinary()
    elif m == 9:
        steps, final = circuit_radix9()
    elif m == 15:
        params = radix15_binary64_fractions() if variant == "polished" else printed_radix15_fractions()
        steps, final = circuit_radix15(params)
    else:
        raise ValueError(f"unsupported radix {m}")
    return eval_circuit(steps, final)


# naive radix-m splitting for the other m up to 32: m - 2 products
NAIVE = tuple(m for m in range(4, 33) if m not in (5, 9, 15))
MU = {2: 0, 3: 1, 5: 2, 9: 3, 15: 4}    # products per kernel
MU.update({m: m - 2 for m in NAIVE})
EXACT = {m: m != 15 for m in MU}


def circuit_products(m):
    if m == 2:
        return len(circuit_binary()[0])
    if m == 3:
        return len(circuit_ternary()[0])
    if m == 5:
        return len(circuit_quinary()[0])
    if m == 9:
        return len(circuit_radix9()[0])
    if m == 15:
        return len(circuit_radix15(printed_radix15_fractions())[0])
    if m in NAIVE:
        return len(circuit_naive(m)[0])
    raise ValueError(m)
