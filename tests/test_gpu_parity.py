"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit for bit.

Bars: exponents, INT8 slices and INT32 level sums bit-exact;
final FP64 C bit-exact (the GPU executes the oracle's FP64 operation sequence,
readings R6/R7), NaN where the oracle has NaN.
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_29975_b200 as oz  # noqa: E402


def dev(x):
    """numpy (Fortran-order) -> column-major CUDA tensor."""
    t = torch.from_numpy(np.asfortranarray(x)).to("cuda")
    return oz.colmajor(t)


def host(t):
    return t.cpu().numpy()


def same(a, b):
    """Bitwise-equal up to the sign of zero; NaN matches NaN."""
    a = np.asarray(a)
    b = np.asarray(b)
    if np.iscomplexobj(a) or np.iscomplexobj(b):
        return same(np.real(a), np.real(b)) and same(np.imag(a), np.imag(b))
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    return bool((na == nb).all() and ((a == b) | na).all())


# ------------------------------------------------------------------ K1 split
def _oracle_rows(orc, X, side, trans, kind):
    """Rows the oracle splits for this operand (op(A) rows / op(B) columns)."""
    opX = orc.op(X, trans)
    rows = opX if side == "A" else opX.T
    return np.ascontiguousarray(rows)


@pytest.mark.parametrize("side", ["A", "B"])
@pytest.mark.parametrize("trans", ["N", "T"])
@pytest.mark.parametrize("s", [1, 3, 7, 8, 9, 16])
def test_split_real_bitexact(orc, side, trans, s):
    g = synth.rng(s)
    for fam, shape in (("spread", (37, 53)), ("uniform", (130, 70)), ("integer", (5, 300))):
        X = synth.make(fam, *shape, seed=int(g.integers(1 << 30)))
        if fam == "spread":
            X[3, 5] = 2.0 ** -1074 * 7      # subnormal
            X[4, :] = 0.0                   # zero row / column
            X[0, 0] = 1.5e300
        sl, ex = oz.debug_split(side, "d", trans, dev(X), s)
        rows = _oracle_rows(orc, X, side, trans, "d")
        D, e, nf = orc.split_rows(rows, s)
        assert (host(ex) == e).all()
        assert (host(sl) == D).all()


@pytest.mark.parametrize("side", ["A", "B"])
@pytest.mark.parametrize("trans", ["N", "T", "C"])
@pytest.mark.parametrize("s", [2, 7, 11])
def test_split_complex_bitexact(orc, side, trans, s):
    X = synth.kkr(45, 39, seed=s, gamma=3.0)
    opX = orc.op(X, trans)
    rows = opX if side == "A" else opX.T       # complex rows x k
    k = rows.shape[1]
    # 3M operands
    for kind, val in (("r", rows.real), ("i", rows.imag), ("s", rows.real + rows.imag)):
        sl, ex = oz.debug_split(side, kind, trans, dev(X), s)
        D, e, nf = orc.split_rows(np.ascontiguousarray(val), s)
        assert (host(ex) == e).all(), kind
        assert (host(sl) == D).all(), kind
    # 4M embedding (R9, N side): A rows r = [Re | Im]; B columns 2j = [Re ; -Im],
    # 2j+1 = [Im ; Re]; halves start at 0 and kh = round_up(k, 32)
    sl, ex = oz.debug_split(side, "z", trans, dev(X), s)
    sl, ex = host(sl), host(ex)
    kh = (k + 31) // 32 * 32

    def check_halves(got, src):
        assert (got[:, :k] == src[:, :k]).all()
        assert (got[:, kh:kh + k] == src[:, k:]).all()
        assert not got[:, k:kh].any() and not got[:, kh + k:].any()

    if side == "A":
        D, e, _ = orc.split_rows(np.ascontiguousarray(np.hstack([rows.real, rows.imag])), s)
        assert (ex == e).all()
        for r in range(rows.shape[0]):
            check_halves(sl[:, r, :], D[:, r, :])
    else:
        nn = rows.shape[0]
        D, e, _ = orc.split_rows(np.ascontiguousarray(np.vstack([np.hstack([rows.real, -rows.imag]),
                                                                 np.hstack([rows.imag, rows.real])])), s)
        for r in range(nn):
            check_halves(sl[:, 2 * r, :], D[:, r, :])
            check_halves(sl[:, 2 * r + 1, :], D[:, nn + r, :])
            assert ex[2 * r] == e[r] == ex[2 * r + 1] == e[nn + r]


# ------------------------------------------------------------ level sums
@pytest.mark.parametrize("s", [1, 2, 5, 8, 9, 13])
@pytest.mark.parametrize("shape", [(64, 64, 64), (200, 150, 97), (129, 65, 33)])
def test_level_sums_bitexact(orc, s, shape):
    m, n, k = shape
    A = synth.spread(m, k, seed=s, phi=1.5)
    B = synth.uniform(k, n, seed=100 + s)
    S = host(oz.debug_level_sums("N", "N", dev(A), dev(B), s))
    DA, _, _ = orc.split_rows(np.ascontiguousarray(A), s)
    DB, _, _ = orc.split_rows(np.ascontiguousarray(B.T), s)
    So = orc.level_sums(DA, DB, s)
    assert np.abs(So).max() < 2 ** 31
    assert (S.astype(np.int64) == So).all()


# ---------------------------------------------------------------- DGEMM
CASES_D = [
    # (m, n, k, transa, transb, alpha, beta, family)
    (64, 64, 64, "N", "N", 1.0, 0.0, "uniform"),
    (37, 53, 71, "T", "N", -1.5, 0.25, "spread"),
    (300, 200, 150, "N", "T", 1.0, 1.0, "uniform"),
    (129, 65, 33, "T", "T", 0.5, -2.0, "spread"),
    (1, 1, 1, "N", "N", 1.0, 0.0, "uniform"),
    (256, 128, 1, "N", "N", 3.0, 0.0, "integer"),
    (17, 300, 260, "C", "C", 1.0, 0.5, "uniform"),
]


@pytest.mark.parametrize("case", CASES_D)
@pytest.mark.parametrize("s", [1, 3, 4, 6, 7, 8, 9, 16])
def test_dgemm_bitexact(orc, case, s):
    m, n, k, ta, tb, al, be, fam = case
    seed = hash((m, n, k, ta, tb, s)) % (1 << 30)
    A = synth.make(fam, *((m, k) if ta == "N" else (k, m)), seed=seed)
    B = synth.make(fam, *((k, n) if tb == "N" else (n, k)), seed=seed + 1)
    C = synth.uniform(m, n, seed=seed + 2)
    want = orc.dgemm(ta, tb, al, A, B, be, C, s)
    Cd = dev(C)
    oz.dgemm(ta, tb, al, dev(A), dev(B), be, Cd, s)
    assert same(host(Cd), want)


def test_dgemm_leading_dims_and_views(orc):
    """lda/ldb/ldc larger than the rows: operate on sub-views of bigger buffers."""
    s = 6
    bigA = synth.uniform(90, 70, seed=1)
    bigB = synth.uniform(80, 60, seed=2)
    bigC = synth.uniform(100, 50, seed=3)
    A, B, C = bigA[5:55, 3:43], bigB[7:47, 2:32], bigC[10:60, 4:34]
    want = orc.dgemm("N", "N", 1.25, A, B, 0.5, C, s)
    tA, tB, tC = dev(bigA), dev(bigB), dev(bigC)
    vC = tC[10:60, 4:34]
    oz.dgemm("N", "N", 1.25, tA[5:55, 3:43], tB[7:47, 2:32], 0.5, vC, s)
    assert same(host(vC), want)
    out = host(tC)
    untouched = np.ones_like(out, bool)
    untouched[10:60, 4:34] = False
    assert (out[untouched] == bigC[untouched]).all()


def test_dgemm_edge_cases(orc):
    s = 5
    A = synth.spread(40, 30, seed=4, phi=3.0)
    B = synth.spread(30, 20, seed=5, phi=3.0)
    # non-finite rows/cols -> NaN rows/cols (R10)
    A2, B2 = A.copy(), B.copy()
    A2[3, 7] = np.inf
    B2[11, 4] = np.nan
    want = orc.dgemm("N", "N", 1.0, A2, B2, 0.0, None, s)
    C = torch.zeros((40, 20), dtype=torch.float64, device="cuda").t().contiguous().t()
    oz.reset_stats()
    oz.dgemm("N", "N", 1.0, dev(A2), dev(B2), 0.0, C, s)
    got = host(C)
    assert same(got, want)
    assert np.isnan(got[3]).all() and np.isnan(got[:, 4]).all()
    assert oz.get_stats()["nonfinite_rows"] == 2
    # beta == 0: C is never read (NaN in C does not leak)
    Cn = dev(np.full((40, 20), np.nan))
    oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, Cn, s)
    assert same(host(Cn), orc.dgemm("N", "N", 1.0, A, B, 0.0, None, s))
    # alpha == 0 quick return: C = beta C, and beta == 0 gives zeros without reading
    C0 = synth.uniform(40, 20, seed=6)
    Cd = dev(C0)
    oz.dgemm("N", "N", 0.0, dev(A), dev(B), -3.0, Cd, s)
    assert same(host(Cd), orc.dgemm("N", "N", 0.0, A, B, -3.0, C0, s))
    Cd = dev(np.full((40, 20), np.nan))
    oz.dgemm("N", "N", 0.0, dev(A), dev(B), 0.0, Cd, s)
    assert (host(Cd) == 0).all()
    # k == 0
    Cd = dev(C0)
    oz.dgemm("N", "N", 1.0, dev(np.zeros((40, 0))), dev(np.zeros((0, 20))), 2.0, Cd, s)
    assert same(host(Cd), 2.0 * C0)
    # extreme exponents: huge, tiny, subnormal outputs
    A3 = A * 1e300
    B3 = B * 1e-300
    A4 = A * 2.0 ** -540
    B4 = B * 2.0 ** -540
    for a, b in ((A3, B3), (A4, B4), (A * 2.0 ** 500, B * 2.0 ** 500)):
        want = orc.dgemm("N", "N", 1.0, a, b, 0.0, None, s)
        Cd = dev(np.zeros((40, 20)))
        oz.dgemm("N", "N", 1.0, dev(a), dev(b), 0.0, Cd, s)
        assert same(host(Cd), want)


def test_dgemm_large_k_chunked(orc):
    """s * k > 131071 (reading R8): K is chunked with exact partial level sums."""
    s = 8
    A = synth.uniform(40, 17000, seed=11)
    B = synth.spread(17000, 36, seed=12, phi=1.0)
    want = orc.dgemm("N", "N", 1.0, A, B, 0.0, None, s)
    C = dev(np.zeros((40, 36)))
    oz.reset_stats()
    oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, s)
    assert same(host(C), want)
    assert oz.get_stats()["k_chunks"] == 2


@pytest.fixture
def force_chunks(monkeypatch):
    monkeypatch.setenv("OZAKI_KCHUNK_KB", "3")
    monkeypatch.setenv("OZAKI_PANEL_COLS", "128")
    yield


@pytest.mark.parametrize("s", [3, 7, 9])
def test_forced_kchunks_and_panels_bitexact(orc, force_chunks, s):
    """Multi-chunk (first / middle / last) and multi-panel paths on small shapes."""
    m, n, k = 150, 300, 260          # KB = 9 -> 3 chunks; 3 panels of 128 columns
    A = synth.spread(m, k, seed=s, phi=1.5)
    B = synth.uniform(k, n, seed=s + 1)
    C = synth.uniform(m, n, seed=s + 2)
    want = orc.dgemm("N", "N", -0.75, A, B, 0.5, C, s)
    Cd = dev(C)
    oz.dgemm("N", "N", -0.75, dev(A), dev(B), 0.5, Cd, s)
    assert same(host(Cd), want)
    Z = synth.kkr(70, 90, seed=s, gamma=1.0)
    W = synth.kkr(90, 130, seed=s + 5, gamma=1.0)
    for method, fn in (("4m", oz.zgemm), ("3m", oz.zgemm3m)):
        Zc = dev(np.zeros((70, 130), np.complex128))
        fn("N", "C", 1.0 + 0.5j, dev(Z), dev(np.conj(W.T).copy()), 0.0, Zc, s)
        assert same(host(Zc), orc.zgemm("N", "N", 1.0 + 0.5j, Z, W, 0.0, None, s, method))
    # batched entries through the chunked driver
    batch = 3
    As = [synth.uniform(m, k, seed=20 + i) for i in range(batch)]
    Bs = [synth.uniform(k, n, seed=30 + i) for i in range(batch)]
    tA = torch.stack([dev(a) for a in As]).transpose(1, 2).contiguous().transpose(1, 2)
    tB = torch.stack([dev(b) for b in Bs]).transpose(1, 2).contiguous().transpose(1, 2)
    tC = torch.zeros((batch, n, m), dtype=torch.float64, device="cuda").transpose(1, 2)
    oz.dgemm_strided_batched("N", "N", 1.0, tA, tB, 0.0, tC, s)
    got = host(tC)
    for i in range(batch):
        assert same(got[i], orc.dgemm("N", "N", 1.0, As[i], Bs[i], 0.0, None, s))


# ---------------------------------------------------------------- ZGEMM
CASES_Z = [
    (48, 40, 36, "N", "N", 1.0, 0.0),
    (70, 33, 65, "C", "N", 0.5 - 1.25j, -0.75 + 0.5j),
    (129, 64, 100, "N", "C", 1j, 1.0),
    (20, 150, 40, "T", "T", -1.0, 0.0),
]


@pytest.mark.parametrize("case", CASES_Z)
@pytest.mark.parametrize("s", [2, 4, 7, 8, 10])
@pytest.mark.parametrize("method", ["4m", "3m"])
def test_zgemm_bitexact(orc, case, s, method):
    m, n, k, ta, tb, al, be = case
    seed = hash((m, n, k, ta, tb, s, method)) % (1 << 30)
    A = synth.kkr(*((m, k) if ta == "N" else (k, m)), seed=seed, gamma=1.0)
    B = synth.spread(*((k, n) if tb == "N" else (n, k)), seed=seed + 1, phi=1.0, complex_=True)
    C = synth.uniform(m, n, seed=seed + 2, complex_=True)
    want = orc.zgemm(ta, tb, al, A, B, be, C, s, method)
    Cd = dev(C)
    fn = oz.zgemm if method == "4m" else oz.zgemm3m
    fn(ta, tb, al, dev(A), dev(B), be, Cd, s)
    assert same(host(Cd), want)


# ------------------------------------------------------------ batched
@pytest.mark.parametrize("s", [3, 8])
def test_batched_bitexact(orc, s):
    batch, m, n, k = 5, 70, 90, 50
    As = [synth.uniform(m, k, seed=10 + i) for i in range(batch)]
    Bs = [synth.spread(k, n, seed=20 + i, phi=1.0) for i in range(batch)]
    Cs = [synth.uniform(m, n, seed=30 + i) for i in range(batch)]
    tA = torch.stack([dev(a) for a in As]).transpose(1, 2).contiguous().transpose(1, 2)
    tB = torch.stack([dev(b) for b in Bs]).transpose(1, 2).contiguous().transpose(1, 2)
    tC = torch.stack([dev(c) for c in Cs]).transpose(1, 2).contiguous().transpose(1, 2)
    oz.dgemm_strided_batched("N", "N", 2.0, tA, tB, -1.0, tC, s)
    got = host(tC)
    for i in range(batch):
        assert same(got[i], orc.dgemm("N", "N", 2.0, As[i], Bs[i], -1.0, Cs[i], s))
    zA = [synth.kkr(m, k, seed=40 + i) for i in range(batch)]
    zB = [synth.kkr(k, n, seed=50 + i) for i in range(batch)]
    for method, fn in (("4m", oz.zgemm_strided_batched), ("3m", oz.zgemm3m_strided_batched)):
        tA = torch.stack([dev(a) for a in zA]).transpose(1, 2).contiguous().transpose(1, 2)
        tB = torch.stack([dev(b) for b in zB]).transpose(1, 2).contiguous().transpose(1, 2)
        tC = torch.zeros((batch, n, m), dtype=torch.complex128, device="cuda").transpose(1, 2)
        fn("N", "N", 1.0, tA, tB, 0.0, tC, s)
        got = host(tC)
        for i in range(batch):
            assert same(got[i], orc.zgemm("N", "N", 1.0, zA[i], zB[i], 0.0, None, s, method))


def test_stats_closed_forms():
    oz.reset_stats()
    A = dev(synth.uniform(32, 32, seed=1))
    C = dev(np.zeros((32, 32)))
    oz.dgemm("N", "N", 1.0, A, A, 0.0, C, 5)
    Z = dev(synth.uniform(16, 16, seed=2, complex_=True))
    Zc = dev(np.zeros((16, 16), np.complex128))
    oz.zgemm("N", "N", 1.0, Z, Z, 0.0, Zc, 5)
    oz.zgemm3m("N", "N", 1.0, Z, Z, 0.0, Zc, 5)
    st = oz.get_stats()
    # s(s+1)/2 per real product, x4 (4M), x3 (3M)
    assert st["int8_gemm_equiv"] == 15 + 4 * 15 + 3 * 15
    assert st["dgemm_calls"] == 1 and st["zgemm_calls"] == 1 and st["zgemm3m_calls"] == 1
    # dgemm: 1 split launch (both operands) + 1 GEMM; zgemm 4M: same; zgemm3m: 1 split launch
    # (both operands, Re/Im/Sum) + ONE GEMM launch over the three products + the combine
    assert st["kernel_launches"] == 2 + 2 + (1 + 1 + 1)


_VARIANT_SNIPPET = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import oracle, synth, paper_2603_29975_b200 as oz
def dev(x): return oz.colmajor(torch.from_numpy(np.asfortranarray(x)).cuda())
bad = 0
for s in {slices}:
    A = synth.spread(130, 75, seed=s, phi=1.5); B = synth.uniform(75, 140, seed=s + 1)
    C = synth.uniform(130, 140, seed=s + 2)
    Cd = dev(C); oz.dgemm("N", "T", 1.5, dev(A), dev(B.T.copy()), -0.5, Cd, s)
    bad += int(not (Cd.cpu().numpy() == oracle.dgemm("N", "T", 1.5, A, B.T.copy(), -0.5, C, s)).all())
    Z = synth.kkr(66, 50, seed=s); Wm = synth.kkr(50, 70, seed=s + 3)
    for method, fn in (("4m", oz.zgemm), ("3m", oz.zgemm3m)):
        Zc = dev(np.zeros((66, 70), np.complex128)); fn("N", "N", 1j, dev(Z), dev(Wm), 0.0, Zc, s)
        w = oracle.zgemm("N", "N", 1j, Z, Wm, 0.0, None, s, method); g = Zc.cpu().numpy()
        bad += int(not ((g.real == w.real).all() and (g.imag == w.imag).all()))
print("BAD", bad)
"""


@pytest.mark.parametrize("variant,slices", [("lv1", [2, 7, 12]), ("flat", [1, 6, 13, 16])])
def test_kernel_variants_bitexact(variant, slices):
    """The 1-CTA level-pass kernel and the flat kernel (OZAKI_KERNEL) are bit-exact too."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, OZAKI_KERNEL=variant)
    res = subprocess.run([sys.executable, "-c", _VARIANT_SNIPPET.format(root=root, slices=slices)],
                         env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    assert "BAD 0" in res.stdout, res.stdout + res.stderr[-2000:]


@pytest.mark.parametrize("pinned", [True, False])
def test_host_offload_bitexact(orc, pinned):
    """Host operands: pipelined H2D / GEMM / D2H inside the library, bit-exact."""
    batch, m, n, k, s = 7, 90, 70, 60, 7
    zA = [synth.kkr(m, k, seed=60 + i) for i in range(batch)]
    zB = [synth.kkr(k, n, seed=70 + i) for i in range(batch)]
    zC = [synth.uniform(m, n, seed=80 + i, complex_=True) for i in range(batch)]

    def host3(lst):
        t = torch.from_numpy(np.stack([np.asfortranarray(x).T for x in lst])).contiguous()
        t = t.pin_memory() if pinned else t
        return t.transpose(1, 2)      # (batch, rows, cols) column-major per entry, CPU

    for method, fn in (("4m", oz.zgemm_strided_batched), ("3m", oz.zgemm3m_strided_batched)):
        tC = host3(zC)
        fn("N", "N", 0.5 - 1j, host3(zA), host3(zB), -0.25, tC, s)
        got = tC.numpy()
        for i in range(batch):
            assert same(got[i], orc.zgemm("N", "N", 0.5 - 1j, zA[i], zB[i], -0.25, zC[i], s, method))
    # real, non-batched
    A = synth.uniform(64, 50, seed=1)
    B = synth.uniform(50, 40, seed=2)
    C = torch.zeros((40, 64), dtype=torch.float64).t()
    oz.dgemm("N", "N", 1.0, torch.from_numpy(np.asfortranarray(A)), torch.from_numpy(np.asfortranarray(B)),
             0.0, C, s)
    assert same(C.numpy(), orc.dgemm("N", "N", 1.0, A, B, 0.0, None, s))
    # mixed host/device operands are refused
    with pytest.raises(oz.OzakiError):
        oz.dgemm("N", "N", 1.0, dev(A), torch.from_numpy(np.asfortranarray(B)), 0.0, C, s)


def test_disjoint_views_of_one_matrix(orc):
    """LAPACK-style Schur update C = A22 - L21 U12 on sub-blocks of ONE column-major array:
    the byte spans interleave but the elements are disjoint, so it must run (and match the
    oracle); truly overlapping views are still rejected (OZAKI_ERR_ALIAS)."""
    n, nb = 200, 48
    X = synth.make("uniform", n, n, seed=77, complex_=True)
    Xd = dev(X)
    L21, U12, A22 = Xd[nb:, :nb], Xd[:nb, nb:], Xd[nb:, nb:]
    want = orc.zgemm("N", "N", -1.0, X[nb:, :nb], X[:nb, nb:], 1.0, X[nb:, nb:], 7)
    oz.zgemm("N", "N", -1.0, L21, U12, 1.0, A22, 7)
    assert same(A22.cpu().numpy(), want)
    assert same(Xd[:nb].cpu().numpy(), X[:nb]) and same(Xd[:, :nb].cpu().numpy(), X[:, :nb])
    with pytest.raises(oz.OzakiError) as ei:
        oz.zgemm("N", "N", 1.0, Xd[10:60, 10:60], Xd[10:60, 10:60], 0.0, Xd[40:90, 40:90], 7)
    assert ei.value.code == 5


def test_host_offload_ldc_padding_and_quick_return(orc):
    """Host offload moves C as m x n with pitch ldc: the rows m..ldc-1 of the caller's array
    are never written, also with beta = 0; alpha = 0 / k = 0 with host pointers is
    the BLAS quick return C = beta C (beta = 1: untouched; beta = 0: zeros, C not read)."""
    m, n, k, ld, s = 70, 45, 33, 101, 6
    A = synth.uniform(m, k, seed=3)
    B = synth.uniform(k, n, seed=4)
    C0 = synth.uniform(m, n, seed=5)
    for beta in (0.0, -0.75):
        big = torch.full((n, ld), 12345.0, dtype=torch.float64).pin_memory()   # column-major ld x n
        big.t()[:m, :] = torch.from_numpy(C0)
        Cv = big.t()[:m, :]
        oz.dgemm("N", "N", 1.25, torch.from_numpy(np.asfortranarray(A)), torch.from_numpy(np.asfortranarray(B)),
                 beta, Cv, s)
        assert same(Cv.numpy(), orc.dgemm("N", "N", 1.25, A, B, beta, C0, s))
        assert (big.t()[m:, :] == 12345.0).all(), beta
    # quick returns on host pointers
    for alpha, kk, beta in ((0.0, k, 0.5), (0.0, k, 0.0), (2.0, 0, -2.0), (0.0, k, 1.0)):
        big = torch.full((n, ld), 7.0, dtype=torch.float64)
        big.t()[:m, :] = torch.from_numpy(C0)
        if beta == 0.0:
            big.t()[:m, :] = float("nan")
        Cv = big.t()[:m, :]
        Ah = torch.from_numpy(np.asfortranarray(A[:, :kk]))
        Bh = torch.from_numpy(np.asfortranarray(B[:kk, :]))
        oz.dgemm("N", "N", alpha, Ah, Bh, beta, Cv, s)
        want = orc.dgemm("N", "N", alpha, A[:, :kk], B[:kk, :], beta, None if beta == 0.0 else C0, s)
        assert same(Cv.numpy(), want), (alpha, kk, beta)
        assert (big.t()[m:, :] == 7.0).all()
    # complex, batched, quick return with a complex beta on pinned host memory
    Z0 = [synth.uniform(m, n, seed=20 + i, complex_=True) for i in range(3)]
    tZ = torch.from_numpy(np.stack([np.asfortranarray(z).T for z in Z0])).contiguous().pin_memory().transpose(1, 2)
    zA = torch.zeros((3, k, m), dtype=torch.complex128).transpose(1, 2)
    zB = torch.zeros((3, n, k), dtype=torch.complex128).transpose(1, 2)
    oz.zgemm_strided_batched("N", "N", 0.0, zA, zB, 0.5 - 0.25j, tZ, s)
    for i in range(3):
        assert same(tZ[i].numpy(), orc.zgemm("N", "N", 0.0, np.zeros((m, k), complex), np.zeros((k, n), complex),
                                            0.5 - 0.25j, Z0[i], s))


def test_lazy_conj_views(orc):
    """torch keeps A.mH / A.conj() as a conj bit over unconjugated storage: the binding
    resolves A and B before the call and refuses a conj-view C."""
    A = synth.uniform(40, 30, seed=1, complex_=True)     # op(A) = A^H is 30 x 40
    B = synth.uniform(40, 20, seed=2, complex_=True)
    Ad = torch.from_numpy(A).to("cuda")                   # row-major: .mH is a column-major view
    Bd = dev(B)
    C = dev(np.zeros((30, 20), complex))
    oz.zgemm("N", "N", 1.0, Ad.mH, Bd, 0.0, C, 7)
    assert same(C.cpu().numpy(), orc.zgemm("C", "N", 1.0, A, B, 0.0, None, 7))
    oz.zgemm("N", "N", 1.0, Ad.mH, Bd.conj(), 0.0, C, 7)
    assert same(C.cpu().numpy(), orc.zgemm("C", "N", 1.0, A, np.conj(B), 0.0, None, 7))
    with pytest.raises(ValueError):
        oz.zgemm("N", "N", 1.0, Ad.mH, Bd, 0.0, C.conj(), 7)


@pytest.mark.parametrize("rows,cols", [(None, "128"), ("100", "128"), ("64", "1000")])
@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "T"), ("N", "C")])
def test_host_offload_column_panels(orc, ta, tb, rows, cols, monkeypatch):
    """One large GEMM on host pointers moves in 2-D blocks (row panels of op(A), column panels of
    op(B), C blocks; H2D / GEMM / D2H overlapped): forced block sizes (ragged last blocks),
    transposes, beta != 0 and ldc > m -- bitwise equal to the oracle, padding rows untouched."""
    monkeypatch.setenv("OZAKI_OFFLOAD_PANEL_COLS", cols)
    if rows:
        monkeypatch.setenv("OZAKI_OFFLOAD_PANEL_ROWS", rows)
    m, n, k, ld, s = 300, 700, 90, 333, 6
    Aop = synth.uniform(m, k, seed=31, complex_=True)
    Bop = synth.spread(k, n, seed=32, phi=1.0, complex_=True)
    C0 = synth.uniform(m, n, seed=33, complex_=True)
    A = Aop if ta == "N" else (Aop.T.copy() if ta == "T" else np.conj(Aop.T).copy())
    B = Bop if tb == "N" else (Bop.T.copy() if tb == "T" else np.conj(Bop.T).copy())
    big = torch.full((n, ld), 5.0 + 0j, dtype=torch.complex128).pin_memory()
    big.t()[:m, :] = torch.from_numpy(C0)
    Cv = big.t()[:m, :]
    hA = torch.from_numpy(np.ascontiguousarray(A.T)).t()
    hB = torch.from_numpy(np.ascontiguousarray(B.T)).t()
    oz.zgemm(ta, tb, 0.5 + 0.25j, hA, hB, -1.0, Cv, s)
    assert same(Cv.numpy(), orc.zgemm("N", "N", 0.5 + 0.25j, Aop, Bop, -1.0, C0, s))
    assert (big.t()[m:, :] == 5.0).all()
    # real DGEMM, beta = 0 (C not read), Ozaki-II through the same panels
    Ar, Br = Aop.real.copy(), Bop.real.copy()
    Cr = torch.full((n, m), float("nan"), dtype=torch.float64).t()
    oz.dgemm("N", "N", 1.0, torch.from_numpy(np.asfortranarray(Ar)), torch.from_numpy(np.asfortranarray(Br)),
             0.0, Cr, s)
    assert same(Cr.numpy(), orc.dgemm("N", "N", 1.0, Ar, Br, 0.0, None, s))
    from oracle import ozaki2 as o2
    oz.ozaki2_dgemm("N", "N", 1.0, torch.from_numpy(np.asfortranarray(Ar)), torch.from_numpy(np.asfortranarray(Br)),
                    0.0, Cr, 14)
    assert same(Cr.numpy()[:40], o2.dgemm("N", "N", 1.0, Ar[:40], Br, 0.0, None, 14))


@pytest.mark.parametrize("alpha", [-1.0, 1.0, -1.0 + 0.5j])
@pytest.mark.parametrize("method", ["4m", "3m"])
def test_zgemm_lu_update_signed_zeros(orc, alpha, method):
    """beta = 1 with alpha = -1 / +1 (the LU trailing update; the epilogue reduces R7's FMA
    shapes to one DADD per component plus exact signed-zero terms) -- bitwise vs the oracle
    INCLUDING the sign of zero, with +-0, +-Inf and NaN entries in C and zero / non-finite rows
    in A (P = +0 / NaN)."""
    m, n, k, s = 140, 96, 70, 6
    A = synth.uniform(m, k, 3, complex_=True)
    A[5, :] = 0.0                      # P row = +0
    A[9, 3] = np.inf                   # P row = NaN (R10)
    B = synth.uniform(k, n, 4, complex_=True)
    B[:, 7] = 0.0
    C0 = synth.uniform(m, n, 5, complex_=True)
    specials = [complex(-0.0, -0.0), complex(0.0, -0.0), complex(-0.0, 0.0), complex(np.inf, 1.0),
                complex(1.0, -np.inf), complex(np.nan, 0.0), complex(-0.0, 2.0), complex(3.0, -0.0)]
    g = np.random.default_rng(9)
    for idx, z in enumerate(specials * 6):
        C0[g.integers(m), g.integers(n)] = z
    C0[5, :8] = np.array(specials)     # zero P meets every special C
    C0[10:18, 7] = np.array(specials)
    C = dev(C0)
    (oz.zgemm if method == "4m" else oz.zgemm3m)("N", "N", alpha, dev(A), dev(B), 1.0, C, s)
    got = host(C)
    want = orc.zgemm("N", "N", alpha, A, B, 1.0, C0, s, method)
    assert same(got, want)
    for part in (np.real, np.imag):
        g_, w_ = part(got), part(want)
        z = (g_ == 0) & (w_ == 0)
        assert (np.signbit(g_[z]) == np.signbit(w_[z])).all()


def test_batch_above_grid_limit(orc):
    """More than 65535 batch entries (the kernels index entries with blockIdx.y / z): the call
    runs as consecutive sub-batches; entries on both sides of the 65535 boundary bit-exact."""
    s, batch, m, n, k = 3, 65540, 8, 6, 5
    rng = np.random.default_rng(7)
    A = rng.uniform(-1, 1, (batch, m, k))
    B = rng.uniform(-1, 1, (batch, k, n))
    tA = torch.from_numpy(A).cuda().transpose(1, 2).contiguous().transpose(1, 2)
    tB = torch.from_numpy(B).cuda().transpose(1, 2).contiguous().transpose(1, 2)
    tC = torch.full((batch, n, m), np.nan, dtype=torch.float64, device="cuda").transpose(1, 2)
    oz.dgemm_strided_batched("N", "N", 1.0, tA, tB, 0.0, tC, s)
    got = tC.cpu().numpy()
    for i in (0, 65534, 65535, 65536, batch - 1):
        assert same(got[i], orc.dgemm("N", "N", 1.0, A[i], B[i], 0.0, None, s)), i
    Z = (A[:, :4, :4] + 1j * A[:, 4:, :4]).copy()
    tZ = torch.from_numpy(Z).cuda().transpose(1, 2).contiguous().transpose(1, 2)
    tW = torch.zeros((batch, 4, 4), dtype=torch.complex128, device="cuda").transpose(1, 2)
    oz.zgemm_strided_batched("N", "C", 0.5 - 0.25j, tZ, tZ, 0.0, tW, s)
    gz = tW.cpu().numpy()
    for i in (0, 65535, batch - 1):
        assert same(gz[i], orc.zgemm("N", "C", 0.5 - 0.25j, Z[i], Z[i], 0.0, None, s, "4m")), i
