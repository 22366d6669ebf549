"""Polish the paper's printed radix-15 circuit onto the exact-prefix manifold.

TEST INFRASTRUCTURE ONLY (oracle side); calls nothing outside oracle/.

Why (reading R1): Appendix B prints the 28 circuit parameters to 3
decimals while Sec. 4 claims prefix error < 9e-7
(PAPER.md:365-366).  At 3 decimals the prefix error is ~2.8e-3.  Remark 2
 says the framework applies to any prefix-exact kernel; we
therefore take the minimum-norm Gauss-Newton projection of the printed point
onto {p : [f_p]_j = 1, j = 0..14}:

    p <- p - J^T (J J^T)^{-1} r(p),   r_j(p) = [f_p]_j - 1  (j = 0..14)

in mpmath at 80 digits, starting from the printed values.  J is exact: each
[f]_j is a polynomial in p; we get dr/dp by forward-mode differentiation of the
circuit (dual numbers over mpmath).  The result is written to
oracle/radix15_polished.json together with its diagnostics.

Run:  python -m oracle.polish_radix15   (or python oracle/polish_radix15.py)
"""
from __future__ import annotations

import json
import os
import sys

import mpmath as mp

if __package__ in (None, ""):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.kernels import (PARAM_ORDER, RADIX15_PRINTED, circuit_radix15, eval_circuit,
                            radix15_flat, radix15_unflat)

mp.mp.dps = 80
N_PARAMS = 28
N_EQ = 15


class Dual:
    """a + sum_i b_i eps_i (first-order forward-mode AD over mpmath)."""
    __slots__ = ("a", "b")

    def __init__(self, a, b=None):
        self.a = mp.mpf(a)
        self.b = b if b is not None else [mp.mpf(0)] * N_PARAMS

    def __add__(self, o):
        o = o if isinstance(o, Dual) else Dual(o)
        return Dual(self.a + o.a, [x + y for x, y in zip(self.b, o.b)])

    __radd__ = __add__

    def __sub__(self, o):
        o = o if isinstance(o, Dual) else Dual(o)
        return Dual(self.a - o.a, [x - y for x, y in zip(self.b, o.b)])

    def __rsub__(self, o):
        return Dual(o) - self

    def __mul__(self, o):
        o = o if isinstance(o, Dual) else Dual(o)
        return Dual(self.a * o.a, [self.a * y + o.a * x for x, y in zip(self.b, o.b)])

    __rmul__ = __mul__

    def __eq__(self, o):
        o = o if isinstance(o, Dual) else Dual(o)
        return self.a == o.a and all(x == y for x, y in zip(self.b, o.b))

    def __ne__(self, o):
        return not self.__eq__(o)


def residual_and_jacobian(p):
    flat = [Dual(x, [mp.mpf(1) if i == j else mp.mpf(0) for j in range(N_PARAMS)])
            for i, x in enumerate(p)]
    params = radix15_unflat(flat)
    steps, final = circuit_radix15(params, one=Dual(1))
    f = eval_circuit(steps, final, one=Dual(1))
    r = mp.matrix(N_EQ, 1)
    J = mp.matrix(N_EQ, N_PARAMS)
    for j in range(N_EQ):
        c = f[j] if j < len(f) else Dual(0)
        r[j] = c.a - 1
        for i in range(N_PARAMS):
            J[j, i] = c.b[i]
    return r, J, f


def polish(max_iter=8, verbose=True):
    p = [mp.mpf(x) for x in radix15_flat(RADIX15_PRINTED)]
    p0 = list(p)
    history = []
    for it in range(max_iter):
        r, J, _ = residual_and_jacobian(p)
        rn = max(abs(x) for x in r)
        history.append(float(rn) if rn > 0 else 0.0)
        if verbose:
            print(f"iter {it}: max|r| = {mp.nstr(rn, 5)}")
        if rn < mp.mpf(10) ** (-70):
            break
        JJt = J * J.T
        y = mp.lu_solve(JJt, r)
        dp = J.T * y
        p = [p[i] - dp[i] for i in range(N_PARAMS)]
    r, J, f = residual_and_jacobian(p)
    return p, p0, history, [c.a for c in f]


def main():
    p, p0, history, f = polish()
    params = radix15_unflat([mp.nstr(x, 50) for x in p])
    max_move = max(abs(a - b) for a, b in zip(p, p0))
    out = {
        "source": "min-norm Gauss-Newton projection of PAPER.md:1009-1020 onto [f]_j = 1 (j<=14); oracle/polish_radix15.py",
        "param_order": PARAM_ORDER,
        "params": params,
        "history_max_abs_residual": history,
        "max_param_move": float(max_move),
        "f_coeffs": [mp.nstr(c, 40) for c in f],
        "c": mp.nstr(1 - f[15], 30),
    }
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "radix15_polished.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", path)
    print("spillover [f]_15 =", mp.nstr(f[15], 12), " [f]_16 =", mp.nstr(f[16], 12), " c =", mp.nstr(1 - f[15], 12))


if __name__ == "__main__":
    main()
