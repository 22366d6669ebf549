"""Host-side checks of the C-ABI library (no GPU needed): symbol exports, the plan builder
against the oracle's plain DP, and the library's kernel polynomials against the oracle's."""
import os
import re

import pytest

import paper_2602_11843_b200 as P
from oracle import kernels as K
from oracle import plan as OP

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2602_11843_b200 import build as B
    B.build()
    return P.load_library()


def test_exports_match_header(lib):
    hdr = open(os.path.join(ROOT, "include", "nseries.h")).read()
    declared = sorted(set(re.findall(r"\b(nseries_[a-z_]+)\s*\(", hdr)))
    assert declared == sorted(P.EXPORTED)
    syms = os.popen(f"nm -D --defined-only {P._binding._LIB_PATH}").read()
    exported = sorted(set(re.findall(r" T (nseries_[a-z_]+)", syms)))
    assert exported == declared
    for name in declared:
        assert hasattr(lib, name)


def test_no_torch_in_abi():
    hdr = open(os.path.join(ROOT, "include", "nseries.h")).read()
    assert "torch" not in hdr.lower().replace("torch cuda tensors", "")


def test_version_and_status(lib):
    assert "sm_100a" in P.nseries_version()
    assert P.nseries_status_string(0) == "ok"
    assert "alias" in P.nseries_status_string(5)


@pytest.mark.parametrize("m,k,products", [
    (5, 125, 12), (5, 625, 16), (9, 81, 10), (9, 729, 15), (15, 225, 12), (15, 3375, 18),
    (2, 128, 14), (2, 512, 18), (2, 4096, 24), (9, 6561, 20), (3, 81, 12), (3, 729, 18)])
def test_pure_plans_table2(lib, m, k, products):
    plan = P.nseries_plan_build(k, kind=m)
    assert plan.steps == [m] * len(plan.steps)
    assert plan.products == products
    assert plan.approx == (1 if m == 15 else 0)


def test_pure_plan_k_mismatch(lib):
    with pytest.raises(P.NSeriesError) as e:
        P.nseries_plan_build(100, kind=9)
    assert e.value.status == 3


def test_approx_requires_flag(lib):
    with pytest.raises(P.NSeriesError) as e:
        P.nseries_plan_build(225, radices=[15, 9])
    assert e.value.status == 4
    with pytest.raises(P.NSeriesError) as e:
        P.nseries_plan_finalize([15], 15, 0)
    assert e.value.status == 4
    with pytest.raises(P.NSeriesError) as e:
        P.nseries_plan_finalize([33], 33, 0)          # naive radices stop at 32
    assert e.value.status == 2
    with pytest.raises(P.NSeriesError) as e:
        P.nseries_plan_finalize([0], 1, 0)
    assert e.value.status == 2


RADIX_SETS = [[2], [5, 2], [9, 5, 2], [15, 9, 5, 2], [15, 9], [9], [5], [3, 2], [9, 5, 3, 2],
              [13, 11, 7, 2], [15, 13, 11, 9, 7, 5, 3, 2], [7], [11, 4]]


@pytest.mark.parametrize("elide", [0, 1])
def test_auto_plan_matches_oracle_dp(lib, elide):
    for radices in RADIX_SETS:
        flags = (P.NSERIES_ALLOW_APPROX if 15 in radices else 0) | (P.NSERIES_ELIDE_TRIVIAL if elide else 0)
        for k in list(range(1, 400)) + [729, 1000, 3375, 4096, 6561, 10000, 12345]:
            ref = OP.best_plan_dp(k, radices, bool(elide))
            plan = P.nseries_plan_build(k, radices=radices, flags=flags)
            assert plan.steps == ref, (radices, k, elide)
            assert plan.products == OP.plan_products(ref, bool(elide))


def test_auto_plan_large_k(lib):
    # k up to 2^62: the plan exists, reaches k, and never costs more than binary with +1
    for k in [2 ** 40, 3 ** 30, 10 ** 15, 2 ** 62, 2 ** 62 - 1]:
        plan = P.nseries_plan_build(k, radices=[15, 9, 5, 2], flags=P.NSERIES_ALLOW_APPROX)
        assert OP.plan_reaches(plan.steps) == k
        binary = P.nseries_plan_build(k, radices=[2])
        assert plan.products <= binary.products


def test_forms(lib):
    p = P.nseries_plan_finalize([15, 1, 9, 2], 15 * 2 * 9 * 2 // 1 // 1 if False else 16 * 9 * 2,
                                P.NSERIES_ALLOW_APPROX)
    assert p.forms == [1, 0, 0, 0]
    p = P.nseries_plan_finalize([15], 15, P.NSERIES_ALLOW_APPROX | P.NSERIES_RFORM_TELESCOPE)
    assert p.forms == [2]


@pytest.mark.parametrize("m,k,products", [(7, 343, 21), (11, 121, 22), (13, 13, 13), (4, 64, 12), (32, 1024, 64)])
def test_pure_naive_plans(lib, m, k, products):
    # naive radix-m splitting: C(m) = m products per step
    plan = P.nseries_plan_build(k, kind=m)
    assert plan.steps == [m] * len(plan.steps) and plan.products == products and plan.approx == 0
    assert products == OP.plan_products(OP.pure_plan(m, k))


@pytest.mark.parametrize("m", [2, 3, 4, 5, 7, 9, 11, 13, 15, 32])
def test_kernel_info_vs_oracle(lib, m):
    info = P.nseries_kernel_info(m)
    assert info["mu"] == K.MU[m]
    assert info["exact"] == K.EXACT[m]
    ref = [float(c) for c in K.kernel_coeffs(m)]
    assert len(info["coeffs"]) == len(ref)
    for a, b in zip(info["coeffs"], ref):
        assert abs(a - b) <= 1e-15 * max(1.0, abs(b))


def test_library_radix15_params_vs_oracle_polish(lib):
    # the library's transcribed polished parameters agree with the oracle's own polish
    src = open(os.path.join(ROOT, "paper_2602_11843_b200", "csrc", "plan.cc")).read()
    block = src[src.index("kRadix15 = {"):src.index("};", src.index("kRadix15 = {"))]
    nums = [float(x) for x in re.findall(r"-?\d+\.\d+(?:e-?\d+)?", block)]
    ref = [float(x) for x in K.radix15_flat(K.polished_radix15_strings())]
    assert len(nums) == 28
    for a, b in zip(nums, ref):
        assert abs(a - b) <= 2e-16 * max(1.0, abs(b))


# ---------------------------------------------------------------- row shards (NEXT-3), host-only

@pytest.mark.parametrize("d,n", [(1, 1), (7, 7), (100, 3), (1100, 8), (4096, 8), (8192, 3), (16384, 8)])
def test_shard_rows_partition(lib, d, n):
    # contiguous, disjoint, covering [0, d), sizes differ by at most one, larger blocks first
    blocks = [P.nseries_shard_rows(d, n, s) for s in range(n)]
    assert blocks[0][0] == 0
    for (r0, m), (r1, _) in zip(blocks, blocks[1:]):
        assert r0 + m == r1
    assert blocks[-1][0] + blocks[-1][1] == d
    sizes = [m for _, m in blocks]
    assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True) and min(sizes) >= 1


@pytest.mark.parametrize("d,n,s", [(5, 0, 0), (5, 6, 0), (5, 2, 2), (5, 2, -1), (0, 1, 0)])
def test_shard_rows_rejects(lib, d, n, s):
    with pytest.raises(P.NSeriesError) as e:
        P.nseries_shard_rows(d, n, s)
    assert e.value.status == 1


def test_eval_sharded_rejects_without_device(lib):
    # argument checks happen before any device work: a NULL handle is INVALID_ARG
    import ctypes
    arr = (ctypes.c_void_p * 1)(None)
    st = lib.nseries_eval_sharded(None, arr, 1, 0, 1, 8, 4, None, 0, arr, None, 0, None)
    assert st == 1


def test_binding_struct_layouts_match_header(tmp_path):
    # the ctypes structs mirror include/nseries.h: sizes and field offsets from a C compile
    import ctypes
    import subprocess
    src = tmp_path / "layout.c"
    fields = {"nseries_stats": [f for f, _ in P.nseries_stats._fields_],
              "nseries_plan": [f for f, _ in P.nseries_plan._fields_],
              "nseries_solve_info": [f for f, _ in P._binding.nseries_solve_info._fields_]}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "nseries.h"', "int main(void) {"]
    for st, fs in fields.items():
        lines.append(f'printf("{st} %zu\\n", sizeof({st}));')
        for f in fs:
            lines.append(f'printf("{st}.{f} %zu\\n", offsetof({st}, {f}));')
    lines.append("return 0; }")
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = dict(l.split() for l in subprocess.check_output([str(exe)], text=True).splitlines())
    classes = {"nseries_stats": P.nseries_stats, "nseries_plan": P.nseries_plan,
               "nseries_solve_info": P._binding.nseries_solve_info}
    for st, cls in classes.items():
        assert int(out[st]) == ctypes.sizeof(cls), st
        for f in fields[st]:
            assert int(out[f"{st}.{f}"]) == getattr(cls, f).offset, (st, f)
