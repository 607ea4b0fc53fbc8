"""GPU parity of k_split_fast (split_fast.cuh), the production K1, on the inputs where its
shortcuts could go wrong, vs the CPU oracle bit for bit:

- the exponent scan decides R3 from IEEE high words and rescans rows with the exact 64-bit
  max only when the high word is not enough: the 127-rule tie (max = (1 + 63/64) 2^E with
  and without low fraction bits), subnormal maxima, maxima whose leading bit sits in the
  low word, zero rows;
- rows longer than one SMEM window (real k > 1024, complex k > 512) and ragged tails;
- conjugated operands (4M A side via -scale, B side via swapped +-Im targets; 3M Im');
- the two-kernel LONG form (exponents by k_split_exps, one CTA per (row group, window));
- the generic kernel (OZAKI_SPLIT=generic) gives the same bits.
The GEMM result (and the INT32 level sums) are bit-exact only if every exponent and digit is.
"""
import os

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_29975_b200 as oz  # noqa: E402

TIE = 1.0 + 63.0 / 64.0                      # fraction field exactly 63 * 2^46: no bump
TIE_UP = np.nextafter(TIE, 2.0)              # one low fraction bit more: bump (R3)
TIE_HI_ONLY = TIE + 2.0 ** -30               # decided by the high word alone


def dev(x):
    return oz.colmajor(torch.from_numpy(np.asfortranarray(x)).to("cuda"))


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if np.iscomplexobj(a) or np.iscomplexobj(b):
        return same(np.real(a), np.real(b)) and same(np.imag(a), np.imag(b))
    na, nb = np.isnan(a), np.isnan(b)
    return a.shape == b.shape and bool((na == nb).all() and ((a == b) | na).all())


def tricky_real(rows, k, seed):
    """Rows (of op(A) / columns of op(B)) exercising every exponent branch."""
    X = synth.uniform(rows, k, seed=seed) * 0.5
    X[:3, :] *= 2.0 ** -12                   # rows 0-2: the planted value is the row max
    X[0, 3] = TIE * 2.0 ** 5
    X[1, k - 1] = -TIE_UP * 2.0 ** -7
    X[2, k // 2] = TIE_HI_ONLY
    X[3, :] = synth.uniform(1, k, seed=seed + 1)[0] * 2.0 ** -1040        # subnormal row, hi-word lead
    X[4, :] = synth.uniform(1, k, seed=seed + 2)[0] * 2.0 ** -1060        # leading bit in the low word
    X[5, :] = 0.0
    X[6, :] = 0.0
    X[6, ::7] = 2.0 ** -1074
    X[7, :] *= 2.0 ** -1040
    X[7, 0] = TIE * 2.0 ** -1022                                          # normal min-exponent tie
    return X


@pytest.fixture(params=["auto", "0", "1"])
def split_long(request):
    """The single-kernel form, the two-kernel LONG form (k_split_exps + one CTA per window), or
    the automatic choice (LONG from 3 windows)."""
    if request.param != "auto":
        os.environ["OZAKI_SPLIT_LONG"] = request.param
    yield request.param
    os.environ.pop("OZAKI_SPLIT_LONG", None)


def with_generic(fn):
    os.environ["OZAKI_SPLIT"] = "generic"
    try:
        return fn()
    finally:
        del os.environ["OZAKI_SPLIT"]


@pytest.mark.parametrize("s", [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12])
@pytest.mark.parametrize("shape", [(70, 50, 40), (130, 70, 1500)])
def test_dgemm_fast_split_exponent_branches(orc, s, shape, split_long):
    m, n, k = shape
    A = tricky_real(m, k, seed=11 * s)
    B = tricky_real(n, k, seed=13 * s).T.copy()      # columns of B carry the tricky rows
    want = orc.dgemm("N", "N", 1.0, A, B, 0.0, None, s)
    got = dev(np.zeros((m, n)))
    oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, got, s)
    assert same(got.cpu().numpy(), want)
    # transposed storage: op(A) rows become column-contiguous (the RCONTIG load path flips)
    got_t = dev(np.zeros((m, n)))
    oz.dgemm("T", "T", 1.0, dev(A.T.copy()), dev(B.T.copy()), 0.0, got_t, s)
    assert same(got_t.cpu().numpy(), want)
    gen = dev(np.zeros((m, n)))
    with_generic(lambda: oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, gen, s))
    assert same(gen.cpu().numpy(), want)


@pytest.mark.parametrize("s", [2, 5, 7, 8, 9, 12])
def test_level_sums_fast_split_multiwindow(orc, s, split_long):
    m, n, k = 65, 130, 2100                          # 3 real windows, ragged tail
    A = tricky_real(m, k, seed=s)
    B = synth.spread(k, n, seed=50 + s, phi=2.0)
    S = oz.debug_level_sums("N", "N", dev(A), dev(B), s).cpu().numpy()
    DA, _, _ = orc.split_rows(np.ascontiguousarray(A), s)
    DB, _, _ = orc.split_rows(np.ascontiguousarray(B.T), s)
    assert (S.astype(np.int64) == orc.level_sums(DA, DB, s)).all()


@pytest.mark.parametrize("s", [1, 3, 4, 7, 8, 9, 12])
@pytest.mark.parametrize("method", ["4m", "3m"])
@pytest.mark.parametrize("trans", [("N", "N"), ("C", "C"), ("T", "C"), ("C", "N")])
@pytest.mark.parametrize("k", [45, 700, 1100])
def test_zgemm_fast_split_conj_windows(orc, s, method, trans, k, split_long):
    ta, tb = trans
    m, n = 40, 36
    seed = (s * 131 + k) % 9973
    A = synth.kkr(*((m, k) if ta == "N" else (k, m)), seed=seed, gamma=3.0)
    B = synth.spread(*((k, n) if tb == "N" else (n, k)), seed=seed + 1, phi=1.5, complex_=True)
    # exponent-branch rows on the complex side too (max over |Re|, |Im|; 3M: Re, Im, Re+Im)
    if ta == "N":
        A[1, 2] = complex(0.1, -TIE_UP * 4)
        A[2, :] = A[2, :] * 2.0 ** -1060
        A[3, :] = 0.0
    else:
        A[2, 1] = complex(TIE * 8, 0.5)
        A[:, 4] = A[:, 4] * 2.0 ** -1045
    C = synth.uniform(m, n, seed=seed + 2, complex_=True)
    al, be = complex(0.75, -1.25), complex(0.5, 0.25)
    want = orc.zgemm(ta, tb, al, A, B, be, C, s, method)
    fn = oz.zgemm if method == "4m" else oz.zgemm3m
    got = dev(C)
    fn(ta, tb, al, dev(A), dev(B), be, got, s)
    assert same(got.cpu().numpy(), want)
    gen = dev(C)
    with_generic(lambda: fn(ta, tb, al, dev(A), dev(B), be, gen, s))
    assert same(gen.cpu().numpy(), want)
