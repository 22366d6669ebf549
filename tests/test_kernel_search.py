"""CPU tests of the radix-kernel search tool (tools/kernel_search.py; SURVEY.md 8(f) NEXT-4,
PAPER.md:333-396).  Every search result is re-checked with the oracle's independent circuit
evaluator (oracle/kernels.py, exact rational convolution)."""
import os
import sys
from fractions import Fraction as F

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import kernel_search as KS  # noqa: E402
from oracle import kernels as OK  # noqa: E402


def _oracle_coeffs(x, p):
    """[f]_j of the ansatz circuit with parameters x, by the oracle's exact evaluator."""
    steps, g = KS.unpack(x, p)
    one = F(1)
    circ = [([0, one], [0, one])] + [([F(float(v)) for v in l], [F(float(v)) for v in r]) for l, r in steps]
    final = [one] + [F(float(v)) for v in g] + [one]
    return OK.eval_circuit(circ, final, one)


def test_parameter_count_and_zero_point():
    # 28 free parameters for radix 15 with 4 products
    assert KS.n_params(4) == 28 and KS.n_params(3) == 17
    # all-zero parameters: f = 1 + P4 with P4 = 0, so [f]_j = 0 for 1 <= j <= 14 -> 14
    assert KS.objective(np.zeros(28), 15, 4) == 14.0


def test_gradient_matches_central_differences():
    rng = np.random.default_rng(5)
    for _ in range(20):
        x = rng.uniform(-1.5, 1.5, 28)
        _, g = KS.objective_and_grad(x, 15, 4)
        h = 1e-6
        fd = np.array([(KS.objective(x + h * e, 15, 4) - KS.objective(x - h * e, 15, 4)) / (2 * h)
                       for e in np.eye(28)])
        assert np.max(np.abs(fd - g)) <= 1e-6 * max(1.0, np.max(np.abs(g)))


def test_theorem1_radix9_is_a_zero_of_the_objective():
    # Theorem 1's circuit in the p = 3 ansatz: U = B^2, V = U(B + 2U),
    # W = P Q, T = I + B + 767/800 U + 15/32 V + W  -> objective 0 up to binary64 rounding
    x = KS.pack([(np.array([0, 0, 1.0]), np.array([0, 1.0, 2.0])),
                 (np.array([0, 3 / 20, 2, 1.0]), np.array([0, 11 / 40, -1 / 8, 1 / 4]))],
                [1.0, 767 / 800, 15 / 32])
    assert KS.objective(x, 9, 3) <= 1e-28
    # and the tool's forward pass equals the oracle's exact convolution of the same circuit
    _, f = KS.forward(x, 3)
    ref = [float(c) for c in _oracle_coeffs(x, 3)]
    assert np.allclose(f[: len(ref)], ref, rtol=0, atol=1e-14)


def test_printed_and_polished_radix15_points():
    # printed Appendix B parameters: prefix error 2.83e-3 (reading R1);
    # the polished point used by the library: prefix exact to binary64 rounding
    printed = np.array([float(v) for v in OK.radix15_flat(OK.RADIX15_PRINTED)])
    polished = np.array([float(v) for v in OK.radix15_flat(OK.polished_radix15_strings())])
    rp = KS.report(printed, 15, 4)
    assert 2.5e-3 < rp["prefix_max_error"] < 3.2e-3
    assert KS.objective(polished, 15, 4) <= 1e-26
    rq = KS.report(polished, 15, 4)
    assert abs(rq["spillover"][0] - 0.185204) < 1e-6 and abs(rq["spillover"][1] - 0.458360) < 1e-6
    assert abs(rq["c"] - 0.814796) < 1e-6


def test_search_recovers_an_exact_radix9_kernel():
    # an exact 3-product radix-9 kernel exists (Theorem 1); the search must find one
    res = KS.multistart(9, 3, starts=10, seed=0)
    assert res["best_objective"] <= 1e-20
    coeffs = _oracle_coeffs(res["best"], 3)
    assert max(abs(float(c) - 1) for c in coeffs[:9]) <= 1e-8
    # deg f = 2^3 = 8: a prefix-exact 3-product circuit IS T_9 (no room for spillover),
    # unlike the 4-product radix-15 ansatz (deg 16)
    assert len(coeffs) == 9


def test_search_finds_prefix_exact_radix15_kernels_with_spillover():
    # L-BFGS-B over the 28 parameters reaches a prefix-exact kernel whose
    # degree >= 15 coefficients do not vanish (an approximate kernel)
    res = KS.multistart(15, 4, starts=10, seed=0)
    assert res["best_objective"] <= 1e-20
    coeffs = [float(c) for c in _oracle_coeffs(res["best"], 4)]
    assert max(abs(c - 1) for c in coeffs[:15]) <= 1e-8
    assert abs(coeffs[15] - 1) > 1e-3                          # not the exact T_15 pattern
    rep = KS.report(res["best"], 15, 4)
    assert 0 < abs(rep["c"]) < 2                               # Lemma 1: [E]_m = c = 1 - [f]_m
    # E(z) = 1 - (1 - z) f(z) starts at z^15 with coefficient c (Lemma 1)
    one_minus_z_f = [coeffs[0]] + [coeffs[j] - coeffs[j - 1] for j in range(1, len(coeffs))] + [-coeffs[-1]]
    E = [-v for v in one_minus_z_f]
    E[0] += 1.0
    assert max(abs(v) for v in E[:15]) <= 1e-8 and abs(E[15] - rep["c"]) <= 1e-8


def test_nonuniqueness_across_seeds():
    # Remark 2: different starts give different circuits (different c)
    cs = []
    for seed in (0, 1, 2):
        res = KS.multistart(15, 4, starts=6, seed=seed)
        if res["best_objective"] <= 1e-20:
            cs.append(KS.report(res["best"], 15, 4)["c"])
    assert len(cs) >= 2 and max(cs) - min(cs) > 1e-3


def test_deterministic_given_seed():
    a = KS.multistart(9, 3, starts=3, seed=7)
    b = KS.multistart(9, 3, starts=3, seed=7)
    assert np.array_equal(a["best"], b["best"]) and a["objectives"] == b["objectives"]


@pytest.mark.parametrize("bad", [np.zeros(27), np.zeros(29)])
def test_unpack_rejects_wrong_length(bad):
    with pytest.raises(ValueError):
        KS.unpack(bad, 4)
