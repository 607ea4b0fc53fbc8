"""NEXT-3: desk-scale analog of the paper's LSMS experiment.

PAPER.md:113-119 (§3.2): LSMS computes the Green function by "the LU-based
inversion of the multiple scattering matrix evaluated across a complex energy
contour", on a "semi-circular path using a ~30-point Gaussian quadrature", and
the paper reports "the percent error in the energy-dependent ... integrated
Green function G(z)" for each emulation mode against native FP64 (Fig. 1a).
SPEC.md [MODULE] workload fixes the desk-scale stand-in used here:

  * H: a Hermitian test operator (``synth.hamiltonian``);
  * nodes z_j / weights w_j: Gauss-Legendre on theta in [pi, 0], mapped to the
    upper semicircle z = c + r e^(i theta) between e_bottom and e_fermi
    (weights carry dz/dtheta);
  * G(z_j) = (z_j I - H)^-1 by a right-looking blocked LU with partial
    pivoting: panel factor and triangular solves in native FP64 (cuSOLVER /
    cuBLAS through torch), EVERY trailing-submatrix update through the GEMM
    under test -- native cuBLAS ZGEMM, Ozaki-I (``ozaki_zgemm``, s slices) or
    Ozaki-II (``ozaki2_zgemm``, N moduli);
  * g(z) = trace G(z); percent error 100 |g_mode - g_native| / |g_native|;
    integrated density N_est = -(1/pi) Im sum_j w_j g(z_j) (= the number of
    eigenvalues of H inside (e_bottom, e_fermi) up to quadrature error).

The emulated GEMM is the only place where precision differs between modes, as
in the paper's experiment.
"""
from __future__ import annotations

import math
import time

import numpy as np

from . import colmajor, ozaki2_zgemm, zgemm


# ----------------------------------------------------------------- contour
def contour_nodes(e_bottom: float, e_fermi: float, npts: int = 30):
    """Gauss-Legendre nodes and weights on the upper semicircle from e_bottom to e_fermi."""
    if not e_bottom < e_fermi or npts < 2:
        raise ValueError("need e_bottom < e_fermi and npts >= 2")
    x, w = np.polynomial.legendre.leggauss(npts)     # on [-1, 1]
    c = 0.5 * (e_bottom + e_fermi)
    r = 0.5 * (e_fermi - e_bottom)
    theta = 0.5 * math.pi * (1.0 - x)                # x = -1 -> theta = pi (e_bottom), x = 1 -> 0
    z = c + r * np.exp(1j * theta)
    dz_dtheta = 1j * r * np.exp(1j * theta)
    # d theta = -(pi / 2) dx, path from theta = pi to 0
    wz = w * (-0.5 * math.pi) * dz_dtheta
    return z, wz


# ------------------------------------------------------------------ GEMMs
def gemm_native():
    """C <- alpha A B + beta C with cuBLAS complex128 (the FP64 ground truth of the sweep)."""
    def f(A, B, C, alpha, beta):
        C.mul_(beta).add_(A @ B, alpha=alpha)
    f.label = "native"
    return f


def gemm_ozaki1(s: int):
    def f(A, B, C, alpha, beta):
        zgemm("N", "N", alpha, A, B, beta, C, s)
    f.label = f"ozaki1 s={s} ({8 * s - 1} bits)"
    return f


def gemm_ozaki2(nmod: int):
    def f(A, B, C, alpha, beta):
        ozaki2_zgemm("N", "N", alpha, A, B, beta, C, nmod)
    f.label = f"ozaki2 N={nmod} moduli"
    return f


# --------------------------------------------------------------- blocked LU
def trailing_updates(n: int, nb: int) -> int:
    """Number of trailing-submatrix GEMMs of the right-looking blocked LU."""
    return max(0, (n + nb - 1) // nb - 1)


def timed_gemm(gemm):
    """Wrap a GEMM so its device time (CUDA events) accumulates in ``.ms``."""
    import torch

    def f(A, B, C, alpha, beta):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        gemm(A, B, C, alpha, beta)
        e1.record()
        f.events.append((e0, e1))
    f.events = []
    f.label = gemm.label

    def total_ms():
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in f.events)
    f.total_ms = total_ms
    return f


def blocked_trsm(T, B, nb: int, gemm, lower: bool, unit: bool, stats: dict | None = None):
    """NEXT-4 emulated ZTRSM: solve T X = B in place of B (T triangular n x n, B n x r,
    column-major CUDA/CPU tensors) by blocks of nb rows.  The nb x nb diagonal solves are
    native FP64; every off-diagonal update B_rest -= T_rest,i X_i goes through ``gemm``
    (SURVEY.md §8(f) NEXT-4 "emulated ZTRSM through blocked TRSM with GEMM updates";
    PAPER.md:115 ZGEMM + ZTRSM dominate LSMS)."""
    import torch
    n = T.shape[0]
    order = range(0, n, nb) if lower else reversed(range(0, n, nb))
    updates = 0
    for i0 in order:
        i1 = min(n, i0 + nb)
        B[i0:i1] = torch.linalg.solve_triangular(T[i0:i1, i0:i1], B[i0:i1], upper=not lower,
                                                 unitriangular=unit)
        if lower and i1 < n:
            gemm(T[i1:, i0:i1], B[i0:i1], B[i1:], -1.0, 1.0)
            updates += 1
        if not lower and i0 > 0:
            gemm(T[:i0, i0:i1], B[i0:i1], B[:i0], -1.0, 1.0)
            updates += 1
    if stats is not None:
        stats["trsm_updates"] = stats.get("trsm_updates", 0) + updates
    return B


def blocked_lu_invert(M, nb: int, gemm, stats: dict | None = None, emulated_trsm: bool = False,
                      check: bool = True):
    """Inverse of a square complex128 CUDA tensor by right-looking blocked LU with partial
    pivoting; the trailing updates A22 -= L21 U12 go through ``gemm``.  Returns (Minv,
    residual max|M Minv - I|); with check=False the residual (a native n^3 product) is skipped
    and None is returned in its place, so that timing covers the inversion alone."""
    import torch
    if M.is_cuda:
        torch.backends.cuda.preferred_linalg_library("cusolver")
    n = M.shape[0]
    A = colmajor(M.clone())                         # column-major working copy
    perm = torch.arange(n, device=M.device)
    updates = 0
    for j0 in range(0, n, nb):
        j1 = min(n, j0 + nb)
        LU, piv = torch.linalg.lu_factor(A[j0:, j0:j1])
        # sequential LAPACK row swaps of the panel -> permutation of rows j0..n-1
        p = list(range(n - j0))
        for i, t in enumerate(piv.tolist()):
            t -= 1
            if t != i:
                p[i], p[t] = p[t], p[i]
        if p != list(range(n - j0)):
            idx = torch.tensor(p, device=M.device) + j0
            A[j0:] = A[idx]
            perm[j0:] = perm[idx]
        A[j0:, j0:j1] = LU
        if j1 < n:
            L11 = torch.tril(A[j0:j1, j0:j1], -1) + torch.eye(j1 - j0, dtype=A.dtype, device=A.device)
            A[j0:j1, j1:] = torch.linalg.solve_triangular(L11, A[j0:j1, j1:], upper=False, unitriangular=True)
            gemm(A[j1:, j0:j1], A[j0:j1, j1:], A[j1:, j1:], -1.0, 1.0)    # Schur complement update
            updates += 1
    if stats is not None:
        stats["trailing_updates"] = stats.get("trailing_updates", 0) + updates
    L = torch.tril(A, -1) + torch.eye(n, dtype=A.dtype, device=A.device)
    U = torch.triu(A)
    Pm = torch.zeros((n, n), dtype=A.dtype, device=A.device)
    Pm[torch.arange(n, device=M.device), perm] = 1.0                 # P M = L U
    if emulated_trsm:      # M^-1 = U^-1 (L^-1 P) with blocked TRSMs whose updates use ``gemm``
        L, U = colmajor(L), colmajor(U)
        Y = blocked_trsm(L, colmajor(Pm), nb, gemm, lower=True, unit=True, stats=stats)
        Minv = blocked_trsm(U, Y, nb, gemm, lower=False, unit=False, stats=stats)
    else:
        Y = torch.linalg.solve_triangular(L, Pm, upper=False, unitriangular=True)
        Minv = torch.linalg.solve_triangular(U, Y, upper=True)
    if not check:
        return Minv, None
    return Minv, residual(M, Minv)


def residual(M, Minv) -> float:
    """max |M Minv - I| in native FP64."""
    import torch
    I = torch.eye(M.shape[0], dtype=M.dtype, device=M.device)
    return float((M @ Minv - I).abs().max())


# ------------------------------------------------------------------ sweep
def green_function_sweep(H, e_bottom: float, e_fermi: float, npts: int, gemms, nb: int = 64,
                         device="cuda"):
    """G(z_j) for every node and GEMM mode; the first mode is the reference (native)."""
    import torch
    z, w = contour_nodes(e_bottom, e_fermi, npts)
    Hd = torch.from_numpy(np.ascontiguousarray(H)).to(device)
    n = Hd.shape[0]
    I = torch.eye(n, dtype=torch.complex128, device=device)
    report = {"n": n, "nb": nb, "nodes": npts, "e_bottom": e_bottom, "e_fermi": e_fermi, "modes": {}}
    ref = None
    for gm in gemms:
        g = np.zeros(npts, dtype=np.complex128)
        resid = 0.0
        st = {}
        if Hd.is_cuda:
            torch.cuda.synchronize()
        t0 = time.perf_counter()
        for j, zj in enumerate(z):
            Minv, r = blocked_lu_invert(complex(zj) * I - Hd, nb, gm, st)
            g[j] = complex(torch.trace(Minv))
            resid = max(resid, r)
        if Hd.is_cuda:
            torch.cuda.synchronize()
        secs = time.perf_counter() - t0
        nest = float(-(1.0 / math.pi) * np.imag(np.sum(w * g)))
        rec = {"g": g, "residual_max": resid, "N_est": nest, "seconds": secs,
               "trailing_updates": st.get("trailing_updates", 0)}
        if ref is None:
            ref = g
        pe = 100.0 * np.abs(g - ref) / np.abs(ref)
        rec["percent_error"] = pe
        rec["max_percent_error"] = float(pe.max())
        rec["argmax_node"] = int(np.argmax(pe))
        report["modes"][gm.label] = rec
    report["z"] = z
    return report
