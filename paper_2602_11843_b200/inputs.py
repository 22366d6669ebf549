"""Seeded synthetic input generators (shared by tests, bench and smoke).

This module holds NONE of the method's arithmetic: it only draws the matrices
of BASELINE.json's configs (recipes in DESIGN.md "Input recipe", following
SURVEY.md 8(d)) and the probe blocks used for column-wise parity.  Both the
CUDA path and the oracle receive exactly the arrays produced here.

Random draws always come from numpy's PCG64 `default_rng(seed)` in the order
listed per config (reading R9).  The dense linear algebra that turns
draws into a matrix (Householder QR for Haar factors, the products Q diag Q^T)
runs in float64 either with numpy (device="cpu") or torch on a CUDA device
(device="cuda", much faster at d >= 4096).  The two devices give matrices that
differ by rounding; a test always hands the SAME array to both sides.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
import tempfile

import numpy as np

CONFIG_NAMES = {
    1: "cfg1_d64_fp64",
    2: "cfg2_d1024_fp64",
    3: "cfg3_d4096_spectrum_0_0995",
    4: "cfg4_mimo_16384x32x32_fp32",
    5: "cfg5_d8192_nonnormal",
}


def _qr_haar(Z, device):
    """Haar orthogonal factor: QR of a Gaussian with the sign fix Q <- Q diag(sign(diag R))."""
    if device == "cpu":
        Q, R = np.linalg.qr(Z)
        s = np.sign(np.diag(R))
        s[s == 0] = 1.0
        return Q * s[None, :]
    import torch
    Zt = torch.from_numpy(Z).to(device)
    Q, R = torch.linalg.qr(Zt)
    s = torch.sign(torch.diagonal(R))
    s[s == 0] = 1.0
    return Q * s[None, :]


def cfg1(d=64, seed=0):
    """A = 0.5 G / sqrt(d), G iid N(0,1) (BASELINE.json configs[0])."""
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((d, d))
    return 0.5 * G / np.sqrt(d)


def cfg2(d=1024, seed=1):
    """A = 0.9 G / sqrt(d) (BASELINE.json configs[1])."""
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((d, d))
    return 0.9 * G / np.sqrt(d)


def cfg3(d=4096, seed=2, device="cpu", lam_lo=0.005, lam_hi=1.0, alpha=1.0):
    """A = I - alpha Q diag(lam) Q^T = Q diag(1 - alpha lam) Q^T, Q Haar, lam ~ U[lam_lo, lam_hi]
    drawn after Z (BASELINE.json configs[2]); symmetrised.  Returns (A, Q, lam)."""
    rng = np.random.default_rng(seed)
    Z = rng.standard_normal((d, d))
    lam = rng.uniform(lam_lo, lam_hi, d)
    ev = 1.0 - alpha * lam
    Q = _qr_haar(Z, device)
    if device == "cpu":
        A = (Q * ev[None, :]) @ Q.T
        A = 0.5 * (A + A.T)
        return np.ascontiguousarray(A), Q, ev
    import torch
    evt = torch.from_numpy(ev).to(device)
    A = (Q * evt[None, :]) @ Q.T
    A = 0.5 * (A + A.T)
    return A.contiguous(), Q, ev


def cfg4(batch=16384, n=32, rows=128, seed=3):
    """MIMO-style: H_b rows x n iid N(0,1), G_b = H_b^T H_b, A_b = I - D_b^{-1} G_b,
    D_b = diag(G_b); cast to float32 (BASELINE.json configs[3]).  rows=256 gives the
    convergent variant (reading R12)."""
    rng = np.random.default_rng(seed)
    H = rng.standard_normal((batch, rows, n))
    G = np.einsum("bri,brj->bij", H, H)
    dg = np.einsum("bii->bi", G)
    A = np.eye(n)[None] - G / dg[:, :, None]
    return np.ascontiguousarray(A.astype(np.float32))


def cfg5(d=8192, seed=4, device="cpu"):
    """A = 0.99 U diag(s) V^T, U, V Haar (two sequential Gaussian draws), s ~ U[0,1]
    (BASELINE.json configs[4]).  ||A||_2 <= 0.99 up to rounding."""
    rng = np.random.default_rng(seed)
    Z1 = rng.standard_normal((d, d))
    Z2 = rng.standard_normal((d, d))
    s = rng.uniform(0.0, 1.0, d)
    U = _qr_haar(Z1, device)
    V = _qr_haar(Z2, device)
    if device == "cpu":
        return np.ascontiguousarray(0.99 * (U * s[None, :]) @ V.T)
    import torch
    st = torch.from_numpy(s).to(device)
    return (0.99 * (U * st[None, :]) @ V.T).contiguous()


def table3_matrix(d=500, alpha=0.9, seed=7):
    """The paper's Sec. 6 model A = alpha Omega D Omega^T with D = linspace(-1, 1, d)
    (reading R13).  Returns (A, Omega, diag)."""
    rng = np.random.default_rng(seed)
    Z = rng.standard_normal((d, d))
    Om = _qr_haar(Z, "cpu")
    D = np.linspace(-1.0, 1.0, d)
    A = alpha * (Om * D[None, :]) @ Om.T
    return np.ascontiguousarray(0.5 * (A + A.T)), Om, alpha * D


def probe_block(d, seed, n_unit=8, n_gauss=8):
    """V = [e_j1 .. e_j8 | g_1 .. g_8] with j from default_rng(1000+seed).choice(d, 8)
    and g from the same generator's standard_normal((d, 8))."""
    rng = np.random.default_rng(1000 + seed)
    n_unit = min(n_unit, d)
    idx = rng.choice(d, n_unit, replace=False)
    g = rng.standard_normal((d, n_gauss))
    V = np.zeros((d, n_unit + n_gauss))
    V[idx, np.arange(n_unit)] = 1.0
    V[:, n_unit:] = g
    return V, idx


def random_matrix(d, seed, scale=0.5):
    """Generic A = scale G / sqrt(d) for parity sweeps."""
    rng = np.random.default_rng(seed)
    return scale * rng.standard_normal((d, d)) / np.sqrt(max(d, 1))


# OpenBLAS pinned to one thread and to its Haswell kernels: numpy's QR / GEMM then run the same
# instruction sequence on any x86-64 host with AVX2, so a CPU-built A has the same bits here and
# on the GPU box (with 8 threads, or the host's own kernel choice, the bits differ run to run
# across hosts).  Used for the matrices the committed goldens (tests/golden/) were computed on.
REPRO_ENV = {"OPENBLAS_CORETYPE": "Haswell", "OPENBLAS_NUM_THREADS": "1", "OMP_NUM_THREADS": "1",
             "MKL_NUM_THREADS": "1"}


def sha256(a):
    """SHA-256 of an array's bytes (C order) -- identifies the exact A a golden belongs to."""
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cpu_reproducible(name, full=False, **kw):
    """inputs.<name>(device="cpu", **kw) computed in a child process under REPRO_ENV; returns A
    (the first element if the generator returns a tuple), or the whole tuple with full=True.
    cfg3: ~16 s, cfg5: ~190 s."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "r.npz")
        code = ("import sys; sys.path.insert(0, %r); import numpy as np; "
                "from paper_2602_11843_b200 import inputs; r = inputs.%s(**%r); "
                "r = r if isinstance(r, tuple) else (r,); "
                "np.savez(%r, *r)" % (root, name, dict(kw), out))
        subprocess.run([sys.executable, "-c", code], env={**os.environ, **REPRO_ENV}, check=True)
        z = np.load(out)
        r = tuple(z["arr_%d" % i] for i in range(len(z.files)))
        return r if full else r[0]
