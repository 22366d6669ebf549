"""Pins for oracle/plan.py: the paper's product counts and brute-force optimality."""
import math

import pytest

from oracle import plan as P

RADICES = [15, 9, 5, 2]


@pytest.mark.parametrize("m,k,binary,radix", [
    (5, 125, 14, 12), (5, 625, 20, 16), (9, 81, 14, 10),
    (9, 729, 20, 15), (15, 225, 16, 12), (15, 3375, 24, 18)])
def test_table2_counts(m, k, binary, radix):
    # Table 2: (mu+2) t for k = m^t; binary baseline 2 ceil(log2 k)
    # ("giving 2 ceil(log_2 k) total", reading R4)
    assert P.plan_products(P.pure_plan(m, k)) == radix
    t2 = math.ceil(math.log2(k))
    assert P.plan_products(P.pure_plan(2, 2 ** t2)) == binary


def test_table1_coefficients():
    # coefficient C(m)/log2(m): 2.00, 1.72, 1.58, 1.54
    printed = {2: 2.00, 3: 1.89, 5: 1.72, 9: 1.58, 15: 1.54}
    for m, c in printed.items():
        mu = P.MU[m]
        assert round((mu + 2) / math.log2(m), 2) == c


def test_radix9_vs_binary_9_pow_10():
    # k = 9^10 needs 50 products (radix-9) vs 63 binary (2 log2 k, no ceiling)
    assert P.plan_products(P.pure_plan(9, 9 ** 10)) == 50
    assert round(2 * math.log2(9 ** 10)) == 63


def test_lei_nakamura_with_plus_one():
    # binary-only plans with "+1" steps reproduce Lei--Nakamura's 2 log2 k - 1 for k = 2^t
    # (Table 1): the first doubling S_2 = I + A is one product as a "+1" step.
    for t in range(1, 11):
        steps = P.best_plan_dp(2 ** t, [2])
        assert steps == [1] + [2] * (t - 1)
        assert P.plan_products(steps) == 2 * t - 1


def test_dp_vs_bruteforce_small_k():
    for radices in ([2], [5, 2], [9, 5, 2], RADICES, [15, 9], [3, 2], [9, 5, 3, 2], [13, 11, 7, 2], [7, 3]):
        for elide in (False, True):
            for k in range(2, 61):
                allp = P.enumerate_plans(k, radices)
                best = min(allp, key=lambda s: P.plan_key(s, elide))
                assert P.best_plan_dp(k, radices, elide) == best, (radices, k, elide)


def test_known_plans():
    # SURVEY.md 8(a) a-1 (verified by exhaustive DP there; re-derived here)
    assert P.best_plan_dp(10000, RADICES) == [15, 1, 5, 5, 5, 5]
    assert P.plan_products([15, 1, 5, 5, 5, 5]) == 23
    assert P.plan_products([15, 1, 5, 5, 5, 5], elide=True) == 21
    assert P.plan_products(P.best_plan_dp(10000, [2])) == 29
    assert P.best_plan_dp(81, [9, 5, 2]) == [9, 9]
    assert P.best_plan_dp(125, [9, 5, 2]) == [5, 5, 5]
    assert P.best_plan_dp(3375, RADICES) == [15, 15, 15]
    assert P.best_plan_dp(6561, RADICES) == [9, 9, 9, 9]


def test_elided_counts():
    # S_1 = I makes the first concatenation free; the last power is unused
    assert P.plan_products([9, 9, 9], elide=True) == 13
    assert P.plan_products([9], elide=True) == 3
    assert P.plan_products([2], elide=True) == 0


def test_ternary_counts():
    # ternary splitting: 3 products per step, 3 log3 k; App. A.3 C(3) = 3
    assert P.plan_products(P.pure_plan(3, 81)) == 12
    assert P.plan_products(P.pure_plan(3, 3 ** 7)) == 21


def test_naive_radix_counts():
    # naive radix-m splitting: m - 2 powers + concatenation + next power =
    # C(m) = m products per step, coefficient m / log2 m (Table 1's naive column)
    for m in (4, 7, 11, 13, 32):
        assert P.plan_products(P.pure_plan(m, m ** 2)) == 2 * m
        assert P.plan_products(P.pure_plan(m, m ** 2), elide=True) == 2 * m - 2
    # naive prime radices are options of the DP, rarely optimal: 49 = 7^2 costs 14 as x7 x7,
    # 13 as six "+1" then x7, and 11 as +1 +1 x2^4 +1 (3 * 16 + 1)
    assert P.best_plan_dp(49, [7]) == [1] * 6 + [7]
    assert P.plan_products(P.best_plan_dp(49, [7])) == 13
    assert P.best_plan_dp(49, [7, 2]) == [1, 1, 2, 2, 2, 2, 1]
    assert P.plan_products(P.best_plan_dp(49, [7, 2])) == 11
    # where a naive radix is chosen: k = 7 in elided counting -- x7 costs 7 - 2 = 5, as does
    # +1 +1 x2 +1; the tie goes to fewer "+1" steps
    assert P.best_plan_dp(7, [7, 2], elide=True) == [7]
    assert P.best_plan_dp(7, [7, 2]) == [1, 1, 2, 1]
