"""Fewest-product plan search -- TEST INFRASTRUCTURE ONLY (oracle side).

A plan reaches k from the initial state n = 1 (S_1 = I, B = A) through steps
    "x m"  : n -> m n, cost mu_m + 2   (kernel + concatenation + power/residual,
             PAPER.md:206-216 cost model C(m) = mu_m + 2; Eq. generalcost 589-594)
    "+1"   : n -> n + 1, cost 1        (S' = S + A^n, A^{n+1} = A^n A; reading R5)
Plans are ranked by the key (products, number of "+1" steps, number of steps,
radices read first-to-last with larger radix preferred; "+1" counts as radix 1)
-- DESIGN.md reading R6.

This is the plain version: forward dynamic programming over EVERY integer
1..k (O(k * |radices|)), plus an exhaustive enumerator for tiny k.  It exists to
pin the library's fast plan builder.

Elided counting (flag ELIDE): an "x m" step taken at n = 1 costs
one product less (its concatenation multiplies by S_1 = I), and a final "x m"
step costs one less (the last power/residual is not needed).
"""
from __future__ import annotations

from oracle.kernels import MU


def step_cost(step, first, last, elide):
    if step == 1:
        return 1
    c = MU[step] + 2
    if elide and first:
        c -= 1
    if elide and last:
        c -= 1
    return c


def plan_products(steps, elide=False):
    n = len(steps)
    return sum(step_cost(s, i == 0, i == n - 1, elide) for i, s in enumerate(steps))


def plan_reaches(steps):
    n = 1
    for s in steps:
        n = n + 1 if s == 1 else n * s
    return n


def plan_key(steps, elide=False):
    return (plan_products(steps, elide), sum(1 for s in steps if s == 1), len(steps),
            tuple(-s for s in steps))


def best_plan_dp(k, radices, elide=False):
    """Forward DP over all n in 1..k.  best[n] = best plan from 1 to n ignoring
    the last-step discount; the final step into k is scored separately."""
    if k < 1:
        raise ValueError("k >= 1")
    if k == 1:
        return []
    radices = sorted(set(radices), reverse=True)
    best = [None] * (k + 1)
    best[1] = []

    def key_inner(steps):
        n = len(steps)
        prod = sum(step_cost(s, i == 0, False, elide) for i, s in enumerate(steps))
        return (prod, sum(1 for s in steps if s == 1), n, tuple(-s for s in steps))

    keys = [None] * (k + 1)
    keys[1] = key_inner([])
    for n in range(1, k):
        if best[n] is None:
            continue
        cands = [(n + 1, 1)] + [(n * m, m) for m in radices if n * m < k]
        for nxt, s in cands:
            if nxt >= k:
                continue
            cand = best[n] + [s]
            kk = key_inner(cand)
            if keys[nxt] is None or kk < keys[nxt]:
                best[nxt], keys[nxt] = cand, kk
    # final step into k
    final_best, final_key = None, None
    preds = [(k - 1, 1)] + [(k // m, m) for m in radices if k % m == 0]
    for pred, s in preds:
        if pred < 1 or best[pred] is None:
            continue
        cand = best[pred] + [s]
        kk = plan_key(cand, elide)
        if final_key is None or kk < final_key:
            final_best, final_key = cand, kk
    return final_best


def enumerate_plans(k, radices):
    """All step sequences (with "+1" = 1) from 1 that land exactly on k (tiny k only)."""
    out = []

    def rec(n, steps):
        if n == k:
            out.append(list(steps))
            return
        if n > k:
            return
        rec(n + 1, steps + [1])
        for m in radices:
            if n * m <= k:
                rec(n * m, steps + [m])

    rec(1, [])
    return out


def pure_plan(m, k):
    """t x m steps when k = m^t (experiments restrict to k = m^t)."""
    steps, n = [], 1
    while n < k:
        n *= m
        steps.append(m)
    if n != k:
        raise ValueError(f"k={k} is not a power of {m}")
    return steps
