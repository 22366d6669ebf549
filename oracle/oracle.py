"""Python front end of the long-double C oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use
this module.  It builds and loads oracle/liboracle.so (oracle/nseries_oracle.c)
and exposes:

  series_sum(A, k, V)          C-1: S_k(A) V = sum_{j<k} A^j V
  series_sum_batch(Ab, k, Vb)  C-1 per matrix of a batch (config 4)
  plan_apply(A, steps, V)      C-2: Y_n V (and R_n V) of a radix plan
  full_series(A, k)            C-1 with V = I (small d)
  kernel_coeff_vectors(...)    [f]_j per step, exact rationals -> long double

Inputs A are numpy float64 (or float32, widened exactly).  Results are numpy
longdouble arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from fractions import Fraction

import numpy as np

from oracle.kernels import kernel_coeffs

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nseries_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

LD = np.longdouble
_ld_p = ctypes.POINTER(ctypes.c_longdouble)
_d_p = ctypes.POINTER(ctypes.c_double)
_i_p = ctypes.POINTER(ctypes.c_int)


def build(force=False):
    """Compile the C oracle (gcc, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".%d.tmp" % os.getpid()       # built aside, then renamed: a process that
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"]   # has the old
        subprocess.check_call(cmd)                                                   # .so keeps it
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.or_series_sum.argtypes = [_d_p, ctypes.c_int, ctypes.c_int64, _ld_p, ctypes.c_int,
                                    ctypes.c_longdouble, ctypes.c_longdouble, _ld_p,
                                    ctypes.POINTER(ctypes.c_int64)]
        L.or_series_sum.restype = ctypes.c_int
        L.or_plan_apply.argtypes = [_d_p, ctypes.c_int, ctypes.c_int, _i_p, _i_p, _i_p, _ld_p,
                                    _ld_p, ctypes.c_int, _ld_p, _ld_p]
        L.or_plan_apply.restype = ctypes.c_int
        L.or_series_sum_batch.argtypes = [_d_p, ctypes.c_int, ctypes.c_int, ctypes.c_int64, _ld_p,
                                          ctypes.c_int, _ld_p]
        L.or_series_sum_batch.restype = ctypes.c_int
        L.or_matvec.argtypes = [_d_p, ctypes.c_int, _ld_p, ctypes.c_int, _ld_p]
        L.or_matvec.restype = ctypes.c_int
        L.or_num_threads.argtypes = []
        L.or_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def num_threads():
    return lib().or_num_threads()


def _as_f64(A):
    A = np.ascontiguousarray(A)
    if A.dtype == np.float32:
        A = A.astype(np.float64)  # exact widening
    if A.dtype != np.float64:
        raise TypeError("A must be float64 or float32")
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise ValueError("A must be square")
    return np.ascontiguousarray(A)


def _as_ld_block(V, d):
    V = np.asarray(V)
    if V.ndim == 1:
        V = V[:, None]
    if V.shape[0] != d:
        raise ValueError("V rows must equal d")
    return np.ascontiguousarray(V.astype(LD))


def series_sum(A, k, V, norm_bound=None, tail_tol=0.0):
    """sum_{j<k} A^j V in long double (C-1).

    norm_bound: optional certified q >= ||A||_2 (q < 1) enabling a rigorous
    early stop once the remaining tail is <= tail_tol * ||partial sum||_F.
    Returns (out, terms_used)."""
    A = _as_f64(A)
    d = A.shape[0]
    Vb = _as_ld_block(V, d)
    p = Vb.shape[1]
    out = np.empty((d, p), dtype=LD)
    used = ctypes.c_int64(0)
    q = LD(norm_bound) if norm_bound is not None else LD(0)
    rc = lib().or_series_sum(A.ctypes.data_as(_d_p), d, int(k), Vb.ctypes.data_as(_ld_p), p,
                             q, LD(tail_tol), out.ctypes.data_as(_ld_p), ctypes.byref(used))
    if rc != 0:
        raise RuntimeError(f"or_series_sum failed rc={rc}")
    return out, int(used.value)


def series_sum_batch(Ab, k, Vb):
    """C-1 per matrix of a batch: out[b] = sum_{j<k} A_b^j V_b in long double.
    Ab: (batch, d, d) float64/float32 (widened exactly); Vb: (batch, d, p)."""
    Ab = np.asarray(Ab)
    if Ab.dtype == np.float32:
        Ab = Ab.astype(np.float64)
    Ab = np.ascontiguousarray(Ab, dtype=np.float64)
    batch, d, _ = Ab.shape
    Vb = np.ascontiguousarray(np.asarray(Vb).astype(LD))
    if Vb.shape[:2] != (batch, d):
        raise ValueError("Vb must be (batch, d, p)")
    p = Vb.shape[2]
    out = np.empty((batch, d, p), dtype=LD)
    rc = lib().or_series_sum_batch(Ab.ctypes.data_as(_d_p), batch, d, int(k), Vb.ctypes.data_as(_ld_p), p,
                                   out.ctypes.data_as(_ld_p))
    if rc != 0:
        raise RuntimeError(f"or_series_sum_batch failed rc={rc}")
    return out


def full_series(A, k):
    A = _as_f64(A)
    d = A.shape[0]
    out, _ = series_sum(A, k, np.eye(d))
    return out


def kernel_coeff_vectors(steps, variant="polished"):
    """Monomial coefficients of each step's kernel as exact Fractions."""
    vecs = []
    for s in steps:
        vecs.append(None if s == 1 else kernel_coeffs(s, variant))
    return vecs


def _frac_to_ld(x: Fraction):
    # exact enough: numerator/denominator in long double (denominators are powers of two
    # times small integers; both fit in 64-bit mantissa only approximately) -> round via
    # high-precision decimal string.
    from decimal import Decimal, getcontext
    getcontext().prec = 40
    return LD(str(Decimal(x.numerator) / Decimal(x.denominator)))


def plan_apply(A, steps, V, variant="polished", want_R=False, coeffs=None):
    """C-2: Y_n V (and R_n V) for the plan `steps` (list of radices m, 1 = "+1")."""
    A = _as_f64(A)
    d = A.shape[0]
    Vb = _as_ld_block(V, d)
    p = Vb.shape[1]
    if coeffs is None:
        coeffs = kernel_coeff_vectors(steps, variant)
    kind, off, length, flat = [], [], [], []
    for s, c in zip(steps, coeffs):
        if s == 1:
            kind.append(1); off.append(len(flat)); length.append(0)
        else:
            kind.append(0); off.append(len(flat)); length.append(len(c))
            flat.extend(_frac_to_ld(Fraction(x)) for x in c)
    n = len(steps)
    kind_a = (ctypes.c_int * max(n, 1))(*kind)
    off_a = (ctypes.c_int * max(n, 1))(*off)
    len_a = (ctypes.c_int * max(n, 1))(*length)
    flat_a = np.ascontiguousarray(np.array(flat if flat else [0], dtype=LD))
    Y = np.empty((d, p), dtype=LD)
    R = np.empty((d, p), dtype=LD) if want_R else None
    rc = lib().or_plan_apply(A.ctypes.data_as(_d_p), d, n, kind_a, off_a, len_a,
                             flat_a.ctypes.data_as(_ld_p), Vb.ctypes.data_as(_ld_p), p,
                             Y.ctypes.data_as(_ld_p), R.ctypes.data_as(_ld_p) if want_R else None)
    if rc != 0:
        raise RuntimeError(f"or_plan_apply failed rc={rc}")
    return (Y, R) if want_R else Y


def matvec(X, V):
    """X V in long double for a float64 (or float32) matrix X."""
    X = _as_f64(X)
    d = X.shape[0]
    Vb = _as_ld_block(V, d)
    p = Vb.shape[1]
    W = np.empty((d, p), dtype=LD)
    rc = lib().or_matvec(X.ctypes.data_as(_d_p), d, Vb.ctypes.data_as(_ld_p), p, W.ctypes.data_as(_ld_p))
    if rc != 0:
        raise RuntimeError("or_matvec failed")
    return W


def rel_fro(X, Y):
    """||X - Y||_F / ||Y||_F in long double."""
    X = np.asarray(X, dtype=LD)
    Y = np.asarray(Y, dtype=LD)
    num = np.sqrt(np.sum((X - Y) ** 2))
    den = np.sqrt(np.sum(Y ** 2))
    return float(num / den) if den != 0 else float(num)
