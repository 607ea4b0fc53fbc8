"""NEXT-3 workload (paper_2603_29975_b200/workload.py): SPEC.md [MODULE] workload.

CPU (-m "not gpu"): contour quadrature, the test Hamiltonian, the blocked LU with a
native GEMM (identity, residual, update count closed form), integrated density.
GPU: the G(z) sweep with native / Ozaki-I / Ozaki-II trailing updates -- native
self-error 0, errors ordered by precision (Fig. 1a staircase), N_est = eigenvalue count.
"""
import math

import numpy as np
import pytest
import torch

import synth
from paper_2603_29975_b200 import workload as W


def test_contour_quadrature():
    x, w = np.polynomial.legendre.leggauss(2)          # SPEC: +-1/sqrt(3), weights 1, before mapping
    assert np.allclose(np.sort(x), [-1 / math.sqrt(3), 1 / math.sqrt(3)]) and np.allclose(w, 1.0)
    z, wz = W.contour_nodes(-1.0, 0.5, 30)
    assert (z.imag > 0).all()
    assert abs(wz.sum() - 1.5) < 1e-13                 # path integral of 1 = e_fermi - e_bottom
    assert abs(z[0].real - (-1.0)) < 0.01 and abs(z[-1].real - 0.5) < 0.01
    with pytest.raises(ValueError):
        W.contour_nodes(1.0, 0.0, 10)


def test_hamiltonian():
    H, ev = synth.hamiltonian(3, seed=1, eigs=[-0.5, 0.2, 0.9])
    assert np.abs(H - H.conj().T).max() == 0.0
    assert np.allclose(np.linalg.eigvalsh(H), [-0.5, 0.2, 0.9], atol=1e-12)
    H2, _ = synth.hamiltonian(3, seed=1, eigs=[-0.5, 0.2, 0.9])
    assert (H == H2).all()


def _cpu_native():
    def f(A, B, C, alpha, beta):
        C.mul_(beta).add_(A @ B, alpha=alpha)
    f.label = "native"
    return f


def test_blocked_lu_cpu_native():
    n = 64
    g = np.random.default_rng(3)
    M = g.standard_normal((n, n)) + 1j * g.standard_normal((n, n)) + 20 * np.eye(n)
    Mt = torch.from_numpy(M)
    st = {}
    Minv, r = W.blocked_lu_invert(Mt, 16, _cpu_native(), st)
    assert r <= 1e-12 and st["trailing_updates"] == W.trailing_updates(n, 16) == 3
    # check=False (timed runs): same inverse, no residual; the residual helper gives the same value
    Minv2, r2 = W.blocked_lu_invert(Mt, 16, _cpu_native(), check=False)
    assert r2 is None and torch.equal(Minv2, Minv) and W.residual(Mt, Minv2) == r
    I = torch.eye(8, dtype=torch.complex128)
    Iinv, r = W.blocked_lu_invert(I, 3, _cpu_native())
    assert r == 0.0 and torch.equal(Iinv, I)
    # pivoting path: a matrix that needs row swaps
    P = np.eye(n)[np.random.default_rng(4).permutation(n)] * (1 + 0j)
    Minv, r = W.blocked_lu_invert(torch.from_numpy(P @ M), 16, _cpu_native())
    assert r <= 1e-12
    assert W.trailing_updates(200, 64) == 3 and W.trailing_updates(64, 64) == 0


def test_blocked_trsm_cpu_native():
    n, r, nb = 70, 33, 16
    g = np.random.default_rng(5)
    Tl = np.tril(g.standard_normal((n, n)) + 1j * g.standard_normal((n, n))) + 8 * np.eye(n)
    Tu = np.triu(g.standard_normal((n, n)) + 1j * g.standard_normal((n, n))) + 8 * np.eye(n)
    B = g.standard_normal((n, r)) + 1j * g.standard_normal((n, r))
    for T, lower, unit in ((Tl, True, False), (Tu, False, False), (0.05 * np.tril(Tl, -1) + np.eye(n), True, True)):
        X = W.blocked_trsm(torch.from_numpy(T), torch.from_numpy(B.copy()), nb, _cpu_native(), lower, unit)
        assert np.abs(T @ X.numpy() - B).max() < 1e-12
    Mt = torch.from_numpy(Tl @ Tu)
    st = {}
    Minv, res = W.blocked_lu_invert(Mt, nb, _cpu_native(), st, emulated_trsm=True)
    assert res < 1e-12 and st["trsm_updates"] == 2 * W.trailing_updates(n, nb)


def test_integrated_density_cpu():
    H, ev = synth.hamiltonian(3, seed=1, eigs=[-0.5, 0.2, 0.9])
    rep = W.green_function_sweep(H, -1.0, 0.5, 30, [_cpu_native()], nb=2, device="cpu")
    assert abs(rep["modes"]["native"]["N_est"] - 2.0) < 1e-6
    rep = W.green_function_sweep(H, 1.0, 1.5, 30, [_cpu_native()], nb=2, device="cpu")   # empty window
    assert abs(rep["modes"]["native"]["N_est"]) < 1e-8


@pytest.mark.gpu
def test_green_function_sweep_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n, nodes = 256, 30
    eb, ef = -0.8, 0.4
    g = np.random.default_rng(7)
    eigs = []
    while len(eigs) < n:                       # keep poles >= 0.1 from the contour endpoints
        x = g.uniform(-1.0, 1.0)
        if abs(x - eb) >= 0.1 and abs(x - ef) >= 0.1:
            eigs.append(x)
    H, ev = synth.hamiltonian(n, seed=7, eigs=eigs)
    count = int(((ev > eb) & (ev < ef)).sum())
    modes = [W.gemm_native()] + [W.gemm_ozaki1(s) for s in (3, 4, 5, 6, 7, 8)] + \
            [W.gemm_ozaki2(m) for m in (8, 10, 12, 14, 16, 18)]
    rep = W.green_function_sweep(H, eb, ef, nodes, modes, nb=64)
    R = rep["modes"]
    assert R["native"]["max_percent_error"] == 0.0
    assert abs(R["native"]["N_est"] - count) < 0.05          # 30-point quadrature error
    assert R["native"]["trailing_updates"] == nodes * W.trailing_updates(n, 64)
    e1 = [R[W.gemm_ozaki1(s).label]["max_percent_error"] for s in (3, 4, 5, 6, 7, 8)]
    e2 = [R[W.gemm_ozaki2(m).label]["max_percent_error"] for m in (8, 10, 12, 14, 16, 18)]
    # precision staircase (Fig. 1a): more slices / moduli never worse, and strictly better at the low end
    assert all(b <= a * 1.5 + 1e-13 for a, b in zip(e1, e1[1:])) and e1[0] > 100 * e1[3]
    assert all(b <= a * 1.5 + 1e-13 for a, b in zip(e2, e2[1:])) and e2[1] > e2[4]
    for lab, rec in R.items():
        assert rec["residual_max"] < 1e-4, lab            # 23-bit mode: ~5e-6
        # the contour integral suppresses the per-node emulation error
        assert abs(rec["N_est"] - R["native"]["N_est"]) < 1e-5, lab
    for lab in (W.gemm_ozaki1(7).label, W.gemm_ozaki2(16).label):
        assert R[lab]["residual_max"] < 1e-12, lab         # FP64-level modes


@pytest.mark.gpu
def test_emulated_trsm_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n, nb = 300, 64
    H, _ = synth.hamiltonian(n, seed=9)
    M = torch.from_numpy(np.ascontiguousarray(H)).cuda() - (0.1 + 0.2j) * torch.eye(n, dtype=torch.complex128,
                                                                                       device="cuda")
    ref, _ = W.blocked_lu_invert(M, nb, W.gemm_native())
    errs = []
    for s in (4, 6, 8):
        st = {}
        Minv, res = W.blocked_lu_invert(M, nb, W.gemm_ozaki1(s), st, emulated_trsm=True)
        assert st["trsm_updates"] == 2 * W.trailing_updates(n, nb)
        errs.append(float((Minv - ref).abs().max() / ref.abs().max()))
    assert errs[0] > errs[1] > errs[2] and errs[2] < 1e-13, errs
