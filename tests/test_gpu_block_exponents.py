"""GPU parity of the NEXT-4 per-block exponent variant (reading R22) vs the oracle, bit for bit."""
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
        return same(np.real(a), np.real(b)) and same(np.imag(a), np.imag(b))
    na, nb = np.isnan(a), np.isnan(b)
    return a.shape == b.shape and bool((na == nb).all() and ((a == b) | na).all())


@pytest.fixture
def kblock():
    def set_(kb):
        oz.set_exponent_block(kb)
    try:
        yield set_
    finally:
        oz.set_exponent_block(0)


@pytest.mark.parametrize("kb", [32, 64, 100, 1000])
@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "T")])
def test_dgemm_blocked(orc, kblock, kb, ta, tb):
    m, n, k, s = 130, 90, 257, 5
    A = synth.spread(m, k, seed=kb, phi=2.0)
    B = synth.spread(k, n, seed=kb + 1, phi=2.0)
    C = synth.uniform(m, n, seed=kb + 2)
    Aop = A if ta == "N" else np.asfortranarray(A.T)
    Bop = B if tb == "N" else np.asfortranarray(B.T)
    kblock(kb)
    for al, be in ((1.0, 0.0), (-1.5, 0.25)):
        ref = orc.dgemm_blocked(ta, tb, al, Aop, Bop, be, C, s, kb)
        Cd = dev(C)
        oz.dgemm(ta, tb, al, dev(Aop), dev(Bop), be, Cd, s)
        assert same(Cd.cpu().numpy(), ref), (kb, ta, al)


@pytest.mark.parametrize("method", ["4m", "3m"])
def test_zgemm_blocked(orc, kblock, method):
    m, n, k, s, kb = 60, 45, 150, 6, 64
    A = synth.make("kkr", m, k, seed=5, complex_=True, gamma=1.0)
    B = synth.make("spread", k, n, seed=6, complex_=True, phi=1.0)
    C = synth.make("uniform", m, n, seed=7, complex_=True)
    kblock(kb)
    ref = orc.zgemm_blocked("N", "N", 0.5 - 1j, A, B, 2.0, C, s, kb, method=method)
    Cd = dev(C)
    (oz.zgemm if method == "4m" else oz.zgemm3m)("N", "N", 0.5 - 1j, dev(A), dev(B), 2.0, Cd, s)
    assert same(Cd.cpu().numpy(), ref)


def test_blocked_batched_and_accuracy(orc, kblock):
    g = np.random.default_rng(8)
    m, k, n, kb, s = 96, 256, 80, 64, 4
    A = g.uniform(-1, 1, (m, k))
    A[:, 64:128] *= 2.0 ** -40
    B = g.uniform(-1, 1, (k, n))
    B[64:128] *= 2.0 ** 40
    T = orc.exact_product(A, B)
    w = np.abs(A) @ np.abs(B)
    C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, s)
    e_row = np.max(np.abs(C.cpu().numpy() - T) / w)
    kblock(kb)
    oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, s)
    e_blk = np.max(np.abs(C.cpu().numpy() - T) / w)
    assert e_row > 0.1 and e_blk < 1e-9, (e_row, e_blk)
    assert same(C.cpu().numpy(), orc.dgemm_blocked("N", "N", 1.0, A, B, 0.0, None, s, kb))
    # batched: every entry blocked independently
    batch = 3
    As = [synth.spread(40, 100, seed=20 + i, phi=2.0) for i in range(batch)]
    Bs = [synth.spread(100, 30, seed=30 + i, phi=2.0) for i in range(batch)]
    At = oz.colmajor(torch.stack([dev(a) for a in As]))
    Bt = oz.colmajor(torch.stack([dev(b) for b in Bs]))
    Ct = oz.colmajor(torch.zeros((batch, 40, 30), dtype=torch.float64, device="cuda"))
    kblock(32)
    oz.dgemm_strided_batched("N", "N", 1.0, At, Bt, 0.0, Ct, 6)
    for i in range(batch):
        assert same(Ct[i].cpu().numpy(), orc.dgemm_blocked("N", "N", 1.0, As[i], Bs[i], 0.0, None, 6, 32))
