"""Pins for oracle/kernels.py and oracle/polish_radix15.py (kernel circuits as polynomials).

Every expected value is printed in the paper or fixed by exact mathematics.
"""
import json
import math
import os
from decimal import ROUND_HALF_EVEN, Decimal
from fractions import Fraction as F

import mpmath as mp
import pytest

from oracle import kernels as K

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_poly_mul_worked_examples():
    # SPEC.md:57-60 examples, themselves quoting PAPER.md:276 and 232
    assert K.poly_mul([1, 1], [1, 1]) == [1, 2, 1]
    assert K.poly_mul([0, 1, 2], [0, 0, 1]) == [0, 0, 0, 1, 2]       # V = U(B+2U) = B^3 + 2B^4
    assert K.poly_mul([0, 0, 1], [0, 1, 1]) == [0, 0, 0, 1, 1]       # quinary V = B^3 + B^4


def test_binary_kernel():
    assert K.kernel_coeffs(2) == [1, 1]                                 # f = 1 + z


def test_ternary_all_ones_exact():
    assert K.kernel_coeffs(3) == [F(1)] * 3          # T_3 = I + B + B^2
    assert K.circuit_products(3) == 1


def test_quinary_all_ones_exact():
    # "Direct verification confirms T_5(B) = I + B + B^2 + B^3 + B^4"
    f = K.kernel_coeffs(5)
    assert f == [F(1)] * 5


def test_radix9_all_ones_exact():
    # Theorem 1: T_9 = I + B + ... + B^8 exactly over Q
    f = K.kernel_coeffs(9)
    assert f == [F(1)] * 9
    assert all(isinstance(c, F) for c in f)


def test_radix9_P_Q_vectors_match_proof():
    # Proof of Theorem 1: p = [0.15, 2, 1, 2], q = [0.275, -0.125, 0.25, 0.5]
    # in powers B^1..B^4, with U = B^2, V = B^3 + 2 B^4.
    U = [0, 0, 1]
    V = K.poly_mul(U, [0, 1, 2])
    P = K.poly_add_scaled(K.poly_add_scaled([0, F(3, 20)], U, 2), V, 1)
    Q = K.poly_add_scaled(K.poly_add_scaled([0, F(11, 40)], U, F(-1, 8)), V, F(1, 4))
    assert P == [0, F(3, 20), 2, 1, 2]
    assert Q == [0, F(11, 40), F(-1, 8), F(1, 4), F(1, 2)]
    W = K.poly_mul(P, Q)
    assert W[5:9] == [1, 1, 1, 1]        # "coefficient 1 for B^5 through B^8"


def test_radix9_corruption_detected():
    # 767/800 -> 766/800 must break exactness at degree 2 (799/800)
    steps, final = K.circuit_radix9(c_u=F(766, 800))
    f = K.eval_circuit(steps, final)
    assert f[2] == F(799, 800)
    assert f != [1] * 9


def test_radix9_rationals_denominators_divide_800():
    # Remark 1
    steps, final = K.circuit_radix9()
    coeffs = [c for lr in steps for side in lr for c in side] + list(final)
    for c in coeffs:
        assert 800 % F(c).denominator == 0


def test_product_counts_and_lower_bound():
    # mu_2=0, mu_5=2, mu_9=3, mu_15=4 (App. A.3 927-935)
    for m, mu in [(2, 0), (3, 1), (5, 2), (9, 3), (15, 4)]:
        assert K.circuit_products(m) == mu == K.MU[m]
    # degree-doubling bound ceil(log2(m-1)) attained with equality
    for m in (5, 9, 15):
        lb = (m - 2).bit_length()          # integer ceil(log2(m-1))
        assert lb == math.ceil(math.log2(m - 1))
        assert K.MU[m] == lb


def test_radix15_printed_prefix_error_and_spillover():
    f = K.kernel_coeffs(15, "printed")
    assert len(f) == 17                      # deg f = 16 (4 chained products from {I,B})
    prefix = max(abs(float(f[j]) - 1) for j in range(15))
    # F1: the 3-decimal circuit misses the claimed 9e-7 prefix error by far
    assert 2.5e-3 < prefix < 3.2e-3
    # spillover "0.185 B^15 + 0.458 B^16" within the 3-decimal rounding
    assert abs(float(f[15]) - 0.185) < 0.02
    assert abs(float(f[16]) - 0.458) < 0.05


def _polished():
    with open(os.path.join(ROOT, "oracle", "radix15_polished.json")) as fh:
        return json.load(fh)


def test_polished_params_round_to_printed_decimals():
    pol = _polished()["params"]
    for key, printed in K.RADIX15_PRINTED.items():
        for s_pol, s_pr in zip(pol[key], printed):
            r = Decimal(s_pol).quantize(Decimal("0.001"), rounding=ROUND_HALF_EVEN)
            assert r == Decimal(s_pr), (key, s_pol, s_pr)


def test_polished_kernel_prefix_spillover_c():
    f = K.kernel_coeffs(15, "polished")     # exact rational convolution of binary64 params
    assert len(f) == 17
    prefix = max(abs(float(f[j] - 1)) for j in range(15))
    assert prefix <= 1e-15
    # printed spillover and c = 1 - [f]_15 ~ 0.81 (Lemma 1)
    assert round(float(f[15]), 3) == 0.185
    assert round(float(f[16]), 3) == 0.458
    c = 1 - float(f[15])
    assert round(c, 2) == 0.81
    assert abs(c) < 1                         # stability regime, Remark 3


def test_polish_converged_at_high_precision():
    d = _polished()
    hist = d["history_max_abs_residual"]
    assert 2.5e-3 < hist[0] < 3.2e-3
    assert hist[-1] < 1e-60
    assert d["max_param_move"] < 5e-4
    # the 80-digit coefficients reproduce an all-ones prefix to ~1e-40
    mp.mp.dps = 50
    fc = [mp.mpf(x) for x in d["f_coeffs"]]
    assert max(abs(fc[j] - 1) for j in range(15)) < mp.mpf(10) ** -40


def _error_map(f, cap):
    # E(z) = 1 - (1-z) f(z)   (Definition 2)
    one_minus_z_f = K.poly_mul([F(1), F(-1)], f)
    E = [-c for c in one_minus_z_f]
    E[0] += 1
    return (E + [0] * cap)[:cap]


def _compose(E, inner, cap):
    # E(inner(z)) truncated at degree cap
    out = [F(0)] * cap
    power = [F(1)] + [F(0)] * (cap - 1)
    for c in E:
        if c != 0:
            for i in range(cap):
                out[i] += c * power[i]
        power = K.poly_mul(power, inner)[:cap]
        power += [F(0)] * (cap - len(power))
        if all(x == 0 for x in power):
            break
    return out


def test_lemma1_error_order():
    # [E]_j = 0 for j < m; [E]_m = c = 1 - [f]_m (Lemma 1)
    for m in (2, 5, 9):
        E = _error_map(K.kernel_coeffs(m), m + 3)
        assert E[:m] == [0] * m and E[m] == 1 and all(x == 0 for x in E[m + 1:])   # E = z^m
    f = K.kernel_coeffs(15, "polished")
    E = _error_map(f, 20)
    assert max(abs(float(x)) for x in E[:15]) < 1e-15
    assert abs(float(E[15]) - (1 - float(f[15]))) < 1e-15


def test_lemma4_leading_coefficient_two_lifts():
    # Lemma 4: E^[2](z) = c^{m+1} z^{m^2} + ...; for radix 15: c^16 at z^225.
    # Use the truncated composition over Q with the exactly-prefix-exact polynomial that keeps
    # only [f]_15, [f]_16 spillover (the binary64 prefix error would leak at degree 15*14).
    f = K.kernel_coeffs(15, "polished")
    f_exact_prefix = [F(1)] * 15 + [f[15], f[16]]
    cap = 226
    E = _error_map(f_exact_prefix, cap)
    EE = _compose(E, E, cap)
    c = 1 - f[15]
    assert all(x == 0 for x in EE[:225])
    assert EE[225] == c ** 16
    assert abs(float(c ** 16) - 0.0377) < 5e-4      # c^16 = 0.037738


def test_lemma3_prefix_growth_radix15():
    # f(z) f(E(z)) agrees with (1-z)^{-1} through degree m^2 - 1 = 224 (Lemma 3)
    f = K.kernel_coeffs(15, "polished")
    f_exact_prefix = [F(1)] * 15 + [f[15], f[16]]
    cap = 230
    E = _error_map(f_exact_prefix, cap)
    fE = _compose(f_exact_prefix, E, cap)
    prod = K.poly_mul(f_exact_prefix, fE)[:cap]
    assert all(x == 1 for x in prod[:225])
    assert prod[225] != 1


@pytest.mark.parametrize("m", [4, 6, 7, 11, 13, 32])
def test_naive_kernel_all_ones_exact(m):
    # naive radix-m kernel: T_m = I + B + ... + B^{m-1} through the power
    # chain -- exact rational convolution gives m ones and m - 2 products
    c = K.kernel_coeffs(m)
    assert c == [F(1)] * m
    assert K.circuit_products(m) == m - 2 == K.MU[m]
    # a broken chain is detected: the last power taken as P_{m-2} * P_2 instead of P_{m-2} * B
    steps, final = K.circuit_naive(m)
    bad = steps[:-1] + [(steps[-1][0], [0, 0, 1])]
    assert K.eval_circuit(bad, final) != [F(1)] * m
