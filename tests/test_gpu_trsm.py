"""Emulated TRSM (reading R23, NEXT-4c; "ZGEMM and ZTRSM"): ozaki_dtrsm /
ozaki_ztrsm through the C ABI vs the oracle's blocked TRSM (oracle.trsm: the same R23 block
order, the R23 substitution in C, the oracle's emulated GEMM for the updates) -- bit for bit
for every side / uplo / transa / diag, ragged block counts, alpha != 1, host pointers."""
import itertools

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_29975_b200 as oz  # noqa: E402


def dev(x):
    return oz.colmajor(torch.from_numpy(np.asfortranarray(x)).to("cuda"))


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if np.iscomplexobj(a) or np.iscomplexobj(b):
        return same(a.real, b.real) and same(a.imag, b.imag)
    na, nb = np.isnan(a), np.isnan(b)
    return a.shape == b.shape and bool((na == nb).all() and ((a == b) | na).all())


def system(dim, nrhs, side, uplo, seed, cplx):
    A = synth.spread(dim, dim, seed, phi=1.0, complex_=cplx) * 0.25 + np.eye(dim) * 2.0
    A[np.triu_indices(dim, 1) if uplo == "L" else np.tril_indices(dim, -1)] = np.nan   # never read
    B = synth.uniform(dim, nrhs, seed + 1, complex_=cplx) if side == "L" else \
        synth.uniform(nrhs, dim, seed + 1, complex_=cplx)
    return A, B


@pytest.mark.parametrize("side,uplo,transa,diag", list(itertools.product("LR", "LU", "NT", "NU")))
def test_dtrsm_all_modes(orc, side, uplo, transa, diag):
    dim, nrhs, s, nb = 300, 70, 7, 128          # 3 blocks, ragged last
    A, B = system(dim, nrhs, side, uplo, 10, False)
    if diag == "U":
        np.fill_diagonal(A, np.nan)
    Bd = dev(B)
    oz.dtrsm(side, uplo, transa, diag, -0.5, dev(A), Bd, s)
    want = orc.trsm(side, uplo, transa, diag, -0.5, np.nan_to_num(A, nan=0.0), B, s, nb=nb)
    assert same(Bd.cpu().numpy(), want)


@pytest.mark.parametrize("side,uplo,transa,diag", list(itertools.product("LR", "LU", "NTC", "NU")))
def test_ztrsm_all_modes(orc, side, uplo, transa, diag):
    dim, nrhs, s = 200, 33, 6
    A, B = system(dim, nrhs, side, uplo, 20, True)
    if diag == "U":
        np.fill_diagonal(A, np.nan)
    oz.set_trsm_block(64)
    try:
        Bd = dev(B)
        oz.ztrsm(side, uplo, transa, diag, 0.5 + 0.25j, dev(A), Bd, s)
    finally:
        oz.set_trsm_block(128)
    want = orc.trsm(side, uplo, transa, diag, 0.5 + 0.25j, np.nan_to_num(A, nan=0.0), B, s, nb=64)
    assert same(Bd.cpu().numpy(), want)


@pytest.mark.parametrize("nb", [1, 5, 32, 1000])
def test_trsm_block_sizes(orc, nb):
    dim, nrhs, s = 77, 9, 5
    A, B = system(dim, nrhs, "L", "U", 30, False)
    oz.set_trsm_block(nb)
    try:
        Bd = dev(B)
        oz.dtrsm("L", "U", "N", "N", 1.0, dev(A), Bd, s)
    finally:
        oz.set_trsm_block(128)
    assert same(Bd.cpu().numpy(), orc.trsm("L", "U", "N", "N", 1.0, np.nan_to_num(A, nan=0.0), B, s, nb=nb))


def test_trsm_subviews_host_and_alpha0(orc):
    """Sub-blocks of larger arrays (lda, ldb > rows), host pointers, alpha = 0 (B not read)."""
    dim, nrhs, s = 150, 40, 7
    A, B = system(dim, nrhs, "R", "L", 40, True)
    bigA = np.full((dim + 13, dim + 3), np.nan + 0j)
    bigA[:dim, :dim] = A
    bigB = np.full((nrhs + 7, dim + 2), 9.0 + 0j)
    bigB[:nrhs, :dim] = B
    Ad = dev(bigA)[:dim, :dim]
    Bdd = dev(bigB)
    oz.ztrsm("R", "L", "C", "N", 1.0, Ad, Bdd[:nrhs, :dim], s)
    want = orc.trsm("R", "L", "C", "N", 1.0, np.nan_to_num(A, nan=0.0), B, s, nb=128)
    got = Bdd.cpu().numpy()
    assert same(got[:nrhs, :dim], want)
    assert (got[nrhs:, :] == 9.0).all() and (got[:, dim:] == 9.0).all()
    # host pointers (staged), pageable memory
    hA = torch.from_numpy(np.asfortranarray(np.nan_to_num(A, nan=0.0)))
    hB = torch.from_numpy(np.asfortranarray(B))
    oz.ztrsm("R", "L", "C", "N", 1.0, hA, hB, s)
    assert same(hB.numpy(), want)
    # alpha = 0: B = 0 without reading B (NaN-safe), A not read
    Bn = dev(np.full((nrhs, dim), np.nan + 0j))
    oz.ztrsm("R", "L", "C", "N", 0.0, Ad, Bn, s)
    assert (Bn.cpu().numpy() == 0).all()


def test_trsm_inverse_workload(orc):
    """The G(z) use: X = L^-1 B with a unit lower factor, then U^-1 -- the two solves of an LU
    inverse -- bitwise vs the oracle, and the residual of the composed solve is small."""
    n, s = 256, 7
    M = synth.uniform(n, n, 5, complex_=True) * 0.1 + np.eye(n) * 3.0
    L = np.tril(M, -1) + np.eye(n)
    U = np.triu(M)
    B = np.eye(n, dtype=complex)
    Bd = dev(B)
    oz.ztrsm("L", "L", "N", "U", 1.0, dev(L), Bd, s)
    oz.ztrsm("L", "U", "N", "N", 1.0, dev(U), Bd, s)
    X1 = orc.trsm("L", "L", "N", "U", 1.0, L, B, s)
    X2 = orc.trsm("L", "U", "N", "N", 1.0, U, X1, s)
    got = Bd.cpu().numpy()
    assert same(got, X2)
    assert np.max(np.abs(L @ U @ got - np.eye(n))) < 1e-12
