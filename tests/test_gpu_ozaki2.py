"""GPU parity of Ozaki-II (CRT, NEXT-1) through the C ABI vs oracle/ozaki2.py.

Bar: bit-exact FP64 C (the GPU reconstructs the exact integer product and
rounds once, readings R16..R20), NaN where the oracle has NaN.
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_29975_b200 as oz  # noqa: E402
from oracle import ozaki2 as o2  # noqa: E402


def dev(x):
    return oz.colmajor(torch.from_numpy(np.asfortranarray(x)).to("cuda"))


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if np.iscomplexobj(a) or np.iscomplexobj(b):
        return same(np.real(a), np.real(b)) and same(np.imag(a), np.imag(b))
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    return bool((na == nb).all() and ((a == b) | na).all())


def _op_shape(t, rows, cols):
    return (rows, cols) if t == "N" else (cols, rows)


@pytest.mark.parametrize("nmod", [6, 10, 14, 16, 18, 20])
@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
def test_dgemm_bitexact(nmod, ta, tb):
    m, n, k = 77, 301, 133                        # ragged in every dimension, 2 column tiles
    g = np.random.default_rng(nmod * 7 + ord(ta) + 3 * ord(tb))
    A = synth.spread(*_op_shape(ta, m, k), seed=int(g.integers(1 << 30)), phi=2.0)
    B = synth.spread(*_op_shape(tb, k, n), seed=int(g.integers(1 << 30)), phi=2.0)
    C = synth.uniform(m, n, seed=int(g.integers(1 << 30)))
    for al, be in ((1.0, 0.0), (-1.5, 0.25)):
        ref = o2.dgemm(ta, tb, al, A, B, be, C, nmod)
        Cd = dev(C)
        oz.ozaki2_dgemm(ta, tb, al, dev(A), dev(B), be, Cd, nmod)
        assert same(Cd.cpu().numpy(), ref), (nmod, ta, tb, al, be)


@pytest.mark.parametrize("shape", [(1, 1, 1), (3, 5, 2), (256, 256, 32), (257, 255, 33), (520, 130, 700)])
def test_dgemm_shapes(shape):
    m, n, k = shape
    A = synth.uniform(m, k, seed=m + 1)
    B = synth.spread(k, n, seed=n + 2, phi=1.0)
    ref = o2.dgemm("N", "N", 1.0, A, B, 0.0, None, 16)
    C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    oz.ozaki2_dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, 16)
    assert same(C.cpu().numpy(), ref), shape


def test_dgemm_integer_exact_and_nonfinite():
    A = synth.integer(40, 60, seed=1, bits=12)
    B = synth.integer(60, 30, seed=2, bits=12)
    C = torch.zeros((30, 40), dtype=torch.float64, device="cuda").t()
    oz.ozaki2_dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, 10)
    assert (C.cpu().numpy() == A @ B).all()
    A = synth.uniform(20, 33, seed=3)
    B = synth.uniform(33, 17, seed=4)
    A[5, 7] = np.inf
    B[2, 3] = np.nan
    ref = o2.dgemm("N", "N", 1.0, A, B, 0.0, None, 12)
    C = torch.zeros((17, 20), dtype=torch.float64, device="cuda").t()
    oz.ozaki2_dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, 12)
    out = C.cpu().numpy()
    assert np.isnan(out[5]).all() and np.isnan(out[:, 3]).all() and same(out, ref)


@pytest.mark.parametrize("nmod", [8, 12, 16, 18])
@pytest.mark.parametrize("ta", ["N", "C"])
def test_zgemm_bitexact(nmod, ta):
    m, n, k = 70, 45, 97
    A = synth.make("kkr", *_op_shape(ta, m, k), seed=nmod, complex_=True, gamma=1.0)
    B = synth.make("spread", k, n, seed=nmod + 1, complex_=True, phi=1.0)
    C = synth.make("uniform", m, n, seed=nmod + 2, complex_=True)
    for al, be in ((1.0, 0.0), (0.5 - 2j, 0.25 + 1j)):
        ref = o2.zgemm(ta, "N", al, A, B, be, C, nmod)
        Cd = dev(C)
        oz.ozaki2_zgemm(ta, "N", al, dev(A), dev(B), be, Cd, nmod)
        assert same(Cd.cpu().numpy(), ref), (nmod, ta, al)


def test_batched_real_and_complex():
    batch, m, n, k = 3, 90, 140, 64
    A = [synth.uniform(m, k, seed=10 + i) for i in range(batch)]
    B = [synth.spread(k, n, seed=20 + i, phi=2.0) for i in range(batch)]
    At = torch.stack([dev(a) for a in A])
    Bt = torch.stack([dev(b) for b in B])
    At = oz.colmajor(At)
    Bt = oz.colmajor(Bt)
    C = oz.colmajor(torch.zeros((batch, m, n), dtype=torch.float64, device="cuda"))
    oz.ozaki2_dgemm_strided_batched("N", "N", 1.0, At, Bt, 0.0, C, 14)
    for i in range(batch):
        assert same(C[i].cpu().numpy(), o2.dgemm("N", "N", 1.0, A[i], B[i], 0.0, None, 14)), i
    ZA = [synth.make("kkr", 64, 64, seed=30 + i, complex_=True, gamma=3.0) for i in range(batch)]
    ZB = [synth.make("kkr", 64, 64, seed=40 + i, complex_=True, gamma=3.0) for i in range(batch)]
    ZAt = oz.colmajor(torch.stack([dev(a) for a in ZA]))
    ZBt = oz.colmajor(torch.stack([dev(b) for b in ZB]))
    ZC = oz.colmajor(torch.zeros((batch, 64, 64), dtype=torch.complex128, device="cuda"))
    oz.ozaki2_zgemm_strided_batched("N", "N", 1.0, ZAt, ZBt, 0.0, ZC, 16)
    for i in range(batch):
        assert same(ZC[i].cpu().numpy(), o2.zgemm("N", "N", 1.0, ZA[i], ZB[i], 0.0, None, 16)), i


def test_host_offload_and_errors():
    A = synth.uniform(50, 40, seed=5)
    B = synth.uniform(40, 30, seed=6)
    Ah = torch.from_numpy(np.asfortranarray(A))
    Bh = torch.from_numpy(np.asfortranarray(B))
    Ch = oz.colmajor(torch.zeros((50, 30), dtype=torch.float64))
    oz.ozaki2_dgemm("N", "N", 1.0, oz.colmajor(Ah), oz.colmajor(Bh), 0.0, Ch, 12)
    assert same(Ch.numpy(), o2.dgemm("N", "N", 1.0, A, B, 0.0, None, 12))
    C = torch.zeros((30, 50), dtype=torch.float64, device="cuda").t()
    with pytest.raises(oz.OzakiError) as ei:     # 1 modulus cannot hold a k = 40 product
        oz.ozaki2_dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, 1)
    assert ei.value.args[0] == 4 or "nu" in str(ei.value)
    with pytest.raises(oz.OzakiError):
        oz.ozaki2_dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, 21)
    # alpha = 0: C = beta C without touching A, B
    C.fill_(2.0)
    oz.ozaki2_dgemm("N", "N", 0.0, dev(A), dev(B), 0.5, C, 12)
    assert (C.cpu().numpy() == 1.0).all()


def test_more_moduli_more_accurate():
    import oracle
    A = synth.uniform(64, 256, seed=7)
    B = synth.uniform(256, 64, seed=8)
    T = oracle.exact_product(A, B)
    errs = []
    for nmod in (8, 10, 12, 14, 16):
        C = torch.zeros((64, 64), dtype=torch.float64, device="cuda").t()
        oz.ozaki2_dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, nmod)
        errs.append(float(np.max(np.abs(C.cpu().numpy() - T) / (np.abs(A) @ np.abs(B)))))
    assert all(b <= a for a, b in zip(errs, errs[1:])) and errs[-1] < 1e-15, errs


@pytest.mark.parametrize("nmod", [6, 12, 14, 20])
@pytest.mark.parametrize("shape", [(40, 36, 5000), (33, 17, 8192)])
def test_dgemm_long_rows_cluster_split(nmod, shape):
    """Long real rows (k > 2048) take the single-read cluster split (split_cluster.cuh, residues
    emitted from shared memory): NN and TT layouts, a padded leading dimension, a non-finite
    row found in a middle K chunk; bit-exact vs the oracle and vs the two-kernel form."""
    import os
    m, n, k = shape
    A = synth.spread(m, k, seed=nmod + k, phi=2.0)
    B = synth.uniform(k, n, seed=nmod + k + 1)
    A[3, k // 2 + 7] = np.inf
    ref = o2.dgemm("N", "N", 1.0, A, B, 0.0, None, nmod)
    got = dev(np.zeros((m, n)))
    oz.ozaki2_dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, got, nmod)
    assert same(got.cpu().numpy(), ref)
    assert np.isnan(got.cpu().numpy()[3]).all()
    got_t = dev(np.zeros((m, n)))
    oz.ozaki2_dgemm("T", "T", 1.0, dev(A.T.copy()), dev(B.T.copy()), 0.0, got_t, nmod)
    assert same(got_t.cpu().numpy(), ref)
    big = np.full((m + 1, k), 3.0)
    big[:m] = A
    got_p = dev(np.zeros((m, n)))
    oz.ozaki2_dgemm("N", "N", 1.0, dev(big)[:m], dev(B), 0.0, got_p, nmod)
    assert same(got_p.cpu().numpy(), ref)
    os.environ["OZAKI_SPLIT_CLUSTER"] = "0"
    try:
        two = dev(np.zeros((m, n)))
        oz.ozaki2_dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, two, nmod)
    finally:
        del os.environ["OZAKI_SPLIT_CLUSTER"]
    assert same(two.cpu().numpy(), ref)


@pytest.mark.parametrize("nw", ["1", "2"])
@pytest.mark.parametrize("shape", [(300, 700, 200), (257, 1030, 4200)])
def test_residue_gemm_tile_widths(nw, shape):
    """Residue-GEMM tiles of 256 x 256 (double-buffered accumulators) and 256 x 512 (each A tile
    feeds two MMAs; the default when K spans >= 128 k-blocks), forced both ways on a short-K and a
    long-K shape with ragged columns: bit-exact vs the oracle."""
    import os
    m, n, k = shape
    A = synth.spread(m, k, seed=m + k, phi=1.0)
    B = synth.uniform(k, n, seed=n + k)
    ref = o2.dgemm("N", "N", 1.0, A, B, 0.0, None, 12)
    os.environ["OZAKI_CRT_NW"] = nw
    try:
        C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
        oz.ozaki2_dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, 12)
        Z = synth.kkr(m // 2, k // 2, seed=5, gamma=1.0)
        W = synth.kkr(k // 2, n // 2, seed=6, gamma=1.0)
        Cz = torch.zeros((n // 2, m // 2), dtype=torch.complex128, device="cuda").t()
        oz.ozaki2_zgemm("N", "N", 1.0, dev(Z), dev(W), 0.0, Cz, 10)
    finally:
        del os.environ["OZAKI_CRT_NW"]
    assert same(C.cpu().numpy(), ref)
    assert same(Cz.cpu().numpy(), o2.zgemm("N", "N", 1.0, Z, W, 0.0, None, 10))
