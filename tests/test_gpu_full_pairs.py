"""GPU parity of the NEXT-4 full pair-set variant (reading R21) vs the oracle, bit for bit."""
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
def full_pairs():
    oz.set_pair_set("full")
    try:
        yield
    finally:
        oz.set_pair_set("triangular")


@pytest.mark.parametrize("s", [1, 3, 5, 8])
def test_level_sums_full(orc, full_pairs, s):
    A = synth.spread(70, 90, seed=s, phi=2.0)
    B = synth.spread(90, 45, seed=s + 1, phi=2.0)
    S = oz.debug_level_sums("N", "N", dev(A), dev(B), s).cpu().numpy()
    DA, _, _ = orc.split_rows(A, s)
    DB, _, _ = orc.split_rows(np.ascontiguousarray(B.T), s)
    ref = orc.level_sums_full(DA, DB, s)
    assert S.shape[0] == 2 * s - 1 and (S == ref).all()


@pytest.mark.parametrize("s", [1, 2, 3, 4, 5, 6, 7, 8])
def test_dgemm_full_bitexact(orc, full_pairs, s):
    m, n, k = 259, 140, 77
    A = synth.spread(m, k, seed=10 * s, phi=2.0)
    B = synth.spread(k, n, seed=10 * s + 1, phi=2.0)
    C = synth.uniform(m, n, seed=10 * s + 2)
    for ta, tb, al, be in (("N", "N", 1.0, 0.0), ("T", "N", -1.5, 0.25)):
        Aop = A if ta == "N" else np.asfortranarray(A.T)
        ref = orc.dgemm(ta, tb, al, Aop, B, be, C, s, pairs="full")
        Cd = dev(C)
        oz.dgemm(ta, tb, al, dev(Aop), dev(B), be, Cd, s)
        assert same(Cd.cpu().numpy(), ref), (s, ta)


@pytest.mark.parametrize("method", ["4m", "3m"])
def test_zgemm_full_bitexact(orc, full_pairs, method):
    m, n, k, s = 70, 45, 97, 6
    A = synth.make("kkr", m, k, seed=3, complex_=True, gamma=1.0)
    B = synth.make("spread", k, n, seed=4, complex_=True, phi=1.0)
    ref = orc.zgemm("N", "N", 1.0, A, B, 0.0, None, s, method=method, pairs="full")
    C = oz.colmajor(torch.zeros((n, m), dtype=torch.complex128, device="cuda").t())
    fn = oz.zgemm if method == "4m" else oz.zgemm3m
    fn("N", "N", 1.0, dev(A), dev(B), 0.0, C, s)
    assert same(C.cpu().numpy(), ref)


def test_full_pairs_limits_and_accuracy(orc, full_pairs):
    A = synth.uniform(64, 64, seed=5)
    B = synth.uniform(64, 64, seed=6)
    C = torch.zeros((64, 64), dtype=torch.float64, device="cuda").t()
    with pytest.raises(oz.OzakiError):
        oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, 9)       # 17 levels do not fit 4 passes
    T = orc.exact_product(A, B)
    oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, 4)
    ef = np.max(np.abs(C.cpu().numpy() - T))
    oz.set_pair_set("triangular")
    oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, 4)
    et = np.max(np.abs(C.cpu().numpy() - T))
    assert ef < et
