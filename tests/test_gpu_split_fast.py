"""GPU parity of k_split_fast (split_fast.cuh), the production K1, on the inputs where its
shortcuts could go wrong, vs the CPU oracle bit for bit:

- the exponent scan decides R3 from IEEE high words and rescans rows with the exact 64-bit
  max only when the high word is not enough: the 127-rule tie (max = (1 + 63/64) 2^E with
  and without low fraction bits), subnormal maxima, maxima whose leading bit sits in the
  low word, zero rows;
- rows longer than one SMEM window (real k > 1024, complex k > 512) and ragged tails;
- conjugated operands (4M A side via -scale, B side via swapped +-Im targets; 3M Im');
- the two-kernel LONG form (exponents by k_split_exps, one CTA per (row group, window));
- the single-read cluster form for long real rows (split_cluster.cuh: a cluster of up to 16
  CTAs per 16-row group, partial maxima exchanged through distributed shared memory), with
  aligned / misaligned leading dimensions, ragged K, partial row groups, batches, non-finite
  rows and the fallback beyond 16 chunks;
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


@pytest.fixture(params=["auto", "0", "1", "1-nocluster"])
def split_long(request):
    """The single-kernel form, the long-row forms (real: the cluster kernel; else / with
    OZAKI_SPLIT_CLUSTER=0 the two-kernel form, k_split_exps + one CTA per window), or the
    automatic choice (long from 3 windows)."""
    if request.param != "auto":
        os.environ["OZAKI_SPLIT_LONG"] = request.param[0]
    if request.param.endswith("nocluster"):
        os.environ["OZAKI_SPLIT_CLUSTER"] = "0"
    yield request.param
    os.environ.pop("OZAKI_SPLIT_LONG", None)
    os.environ.pop("OZAKI_SPLIT_CLUSTER", None)


def with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


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


# ------------------------------------------------------------ single-read cluster split
def padded(X, extra_rows):
    """Column-major device view of X inside a taller array (leading dimension rows + extra)."""
    r, c = X.shape
    big = np.full((r + extra_rows, c), 7.0)
    big[:r] = X
    return dev(big)[:r]


@pytest.mark.parametrize("s", [1, 3, 7, 9, 12])
@pytest.mark.parametrize("shape", [(70, 50, 8192), (130, 40, 5000), (33, 17, 2049)])
@pytest.mark.parametrize("rg", ["8", "16"])
def test_dgemm_cluster_split(orc, s, shape, rg):
    """Long real rows through k_split_cluster: 8- or 16-row groups (70 / 130 / 33 rows: partial
    last group), K chunks of <= 512 over clusters of 5..16 CTAs, ragged depth (5000, 2049), NN
    (rows of op(A) adjacent in memory, op(B) rows contiguous) and TT (the layouts flip); bit-exact
    vs the oracle and vs the two-kernel form."""
    m, n, k = shape
    A = tricky_real(m, k, seed=7 * s + k)
    B = tricky_real(n, k, seed=5 * s + k).T.copy()
    want = orc.dgemm("N", "N", 1.0, A, B, 0.0, None, s)
    got = dev(np.zeros((m, n)))
    with_env({"OZAKI_SPLIT_RG": rg}, lambda: oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, got, s))
    assert same(got.cpu().numpy(), want)
    got_t = dev(np.zeros((m, n)))
    with_env({"OZAKI_SPLIT_RG": rg},
             lambda: oz.dgemm("T", "T", 1.0, dev(A.T.copy()), dev(B.T.copy()), 0.0, got_t, s))
    assert same(got_t.cpu().numpy(), want)
    two = dev(np.zeros((m, n)))
    with_env({"OZAKI_SPLIT_CLUSTER": "0"}, lambda: oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, two, s))
    assert same(two.cpu().numpy(), want)


@pytest.mark.parametrize("s", [4, 7])
@pytest.mark.parametrize("extra", [1, 2, 3])
def test_dgemm_cluster_split_leading_dims(orc, s, extra):
    """Odd / even padded leading dimensions: the 16-B cp.async pieces apply only when the row
    group (NN A side) or each row (B side) starts 16-B aligned, else 8-B copies."""
    m, n, k = 48, 40, 3000
    A = tricky_real(m, k, seed=90 + extra)
    B = synth.spread(k, n, seed=91 + extra, phi=2.0)
    C = synth.uniform(m, n, seed=92)
    want = orc.dgemm("N", "N", -1.0, A, B, 1.0, C, s)
    got = padded(C, 0)
    oz.dgemm("N", "N", -1.0, padded(A, extra), padded(B, extra), 1.0, got, s)
    assert same(got.cpu().numpy(), want)
    want_t = orc.dgemm("T", "N", 0.5, A.T.copy(), B, 0.0, None, s)
    got_t = dev(np.zeros((m, n)))
    oz.dgemm("T", "N", 0.5, padded(A.T.copy(), extra), padded(B, extra), 0.0, got_t, s)
    assert same(got_t.cpu().numpy(), want_t)


@pytest.mark.parametrize("kc", ["256", "512", "1024"])
def test_dgemm_cluster_split_chunk_sizes(orc, kc):
    """OZAKI_SPLIT_KC moves the chunk (and so the cluster size: 2..16) without changing bits;
    depths needing more than 16 chunks fall back to the two-kernel form."""
    s = 6
    for m, n, k in ((40, 36, 2200), (20, 24, 4100), (24, 20, 9000)):
        A = tricky_real(m, k, seed=k)
        B = synth.uniform(k, n, seed=k + 1)
        want = orc.dgemm("N", "N", 1.0, A, B, 0.0, None, s)
        got = dev(np.zeros((m, n)))
        with_env({"OZAKI_SPLIT_KC": kc}, lambda: oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, got, s))
        assert same(got.cpu().numpy(), want)


def test_dgemm_cluster_split_batched_nonfinite(orc):
    """Batched entries (blockIdx.y) and non-finite rows / columns (R10) found in a middle chunk:
    NaN rows / columns, the nonfinite counter, finite entries bit-exact."""
    s, batch, m, n, k = 5, 3, 40, 34, 6000
    As = [synth.spread(m, k, seed=300 + i, phi=1.0) for i in range(batch)]
    Bs = [synth.uniform(k, n, seed=310 + i) for i in range(batch)]
    As[1][5, 2600] = np.inf
    Bs[2][3100, 7] = np.nan
    tA = torch.stack([dev(a) for a in As]).transpose(1, 2).contiguous().transpose(1, 2)
    tB = torch.stack([dev(b) for b in Bs]).transpose(1, 2).contiguous().transpose(1, 2)
    tC = torch.zeros((batch, n, m), dtype=torch.float64, device="cuda").transpose(1, 2)
    oz.reset_stats()
    oz.dgemm_strided_batched("N", "N", 1.0, tA, tB, 0.0, tC, s)
    got = tC.cpu().numpy()
    assert oz.get_stats()["nonfinite_rows"] == 2
    for i in range(batch):
        assert same(got[i], orc.dgemm("N", "N", 1.0, As[i], Bs[i], 0.0, None, s))
    assert np.isnan(got[1][5]).all() and np.isnan(got[2][:, 7]).all()
