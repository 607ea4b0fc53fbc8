"""Parity of the persistent schedule when every CTA pair owns SEVERAL tiles.

The pair GEMM launches min(tiles, SMs/2) = 74 CTA pairs and loops over (batch, tile); the
mbarrier phases, TMEM level slots and pass plan are carried from one tile to the next.  The
shapes below have >= 148 super-tiles (>= 2 per pair) with ragged last tiles, and every sampled
entry -- tile edges, the last row / column -- must equal the oracle bit for bit, at every slice
count (triangular s = 1..12, the flat fallback s = 13..16), the full pair set s = 1..8, the
general alpha/beta epilogue and Ozaki-II at several moduli counts.  The oracle sees FULL rows of
op(A) and FULL columns of op(B), so its exponents are those of the whole problem.
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2603_29975_b200 as oz  # noqa: E402

M, N, K = 2300, 4700, 100        # Ozaki-I: 9 x 37 = 333 super-tiles of 256 x 128 (4.5 per pair)


def dev(x):
    return oz.colmajor(torch.from_numpy(np.asfortranarray(x)).to("cuda"))


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if np.iscomplexobj(a) or np.iscomplexobj(b):
        return same(a.real, b.real) and same(a.imag, b.imag)
    na, nb = np.isnan(a), np.isnan(b)
    return a.shape == b.shape and bool((na == nb).all() and ((a == b) | na).all())


def sample(n, tile, seed):
    g = np.random.default_rng(seed)
    edges = [0, 1, tile - 1, tile, 2 * tile - 1, 2 * tile, n // 2, n - tile, n - 2, n - 1]
    return np.unique(np.clip(np.r_[edges, g.integers(0, n, 14)], 0, n - 1))


def gather(Cd, r, c):
    rr, cc = torch.from_numpy(r).cuda(), torch.from_numpy(c).cuda()
    return Cd[rr][:, cc].cpu().numpy()


@pytest.fixture(scope="module")
def real_inputs():
    A = synth.spread(M, K, 11, phi=1.0)
    B = synth.uniform(K, N, 12)
    C0 = synth.uniform(M, N, 13)
    return A, B, C0, dev(A), dev(B), dev(C0)


@pytest.mark.parametrize("s", list(range(1, 17)))
def test_dgemm_multitile_every_s(orc, real_inputs, s):
    A, B, C0, Ad, Bd, _ = real_inputs
    C = torch.empty((N, M), dtype=torch.float64, device="cuda").t()
    C.fill_(float("nan"))                   # beta = 0: C must not be read
    oz.dgemm("N", "N", 1.0, Ad, Bd, 0.0, C, s)
    r, c = sample(M, 128, s), sample(N, 128, 100 + s)
    want = orc.dgemm("N", "N", 1.0, A[r], B[:, c], 0.0, None, s)
    assert same(gather(C, r, c), want), s


@pytest.mark.parametrize("s", [3, 7, 9, 12])
@pytest.mark.parametrize("ta,tb", [("T", "N"), ("N", "T")])
def test_dgemm_multitile_general_ab_trans(orc, real_inputs, s, ta, tb):
    """alpha = -1, beta = 1 (the LU trailing update) and transposed operands, multi-tile."""
    A, B, C0, _, _, C0d = real_inputs
    Aop = A if ta == "N" else np.asfortranarray(A.T)
    Bop = B if tb == "N" else np.asfortranarray(B.T)
    C = C0d.clone()
    oz.dgemm(ta, tb, -1.0, dev(Aop), dev(Bop), 1.0, C, s)
    r, c = sample(M, 128, 7 * s), sample(N, 128, 9 * s)
    want = orc.dgemm("N", "N", -1.0, A[r], B[:, c], 1.0, C0[np.ix_(r, c)], s)
    assert same(gather(C, r, c), want)


@pytest.mark.parametrize("s", list(range(1, 9)))
def test_dgemm_multitile_full_pairs(orc, real_inputs, s):
    A, B, C0, Ad, Bd, C0d = real_inputs
    C = C0d.clone()
    oz.set_pair_set("full")
    try:
        oz.dgemm("N", "N", 0.75, Ad, Bd, -0.5, C, s)
    finally:
        oz.set_pair_set("triangular")
    r, c = sample(M, 128, 20 + s), sample(N, 128, 30 + s)
    want = orc.dgemm("N", "N", 0.75, A[r], B[:, c], -0.5, C0[np.ix_(r, c)], s, pairs="full")
    assert same(gather(C, r, c), want)


@pytest.mark.parametrize("nmod", [6, 10, 14, 18, 20])
def test_ozaki2_multitile(real_inputs, nmod):
    """Ozaki-II residue GEMM uses 256 x 256 super-tiles: 9 x 19 = 171 on 74 pairs."""
    from oracle import ozaki2 as o2
    A, B, C0, Ad, Bd, C0d = real_inputs
    C = C0d.clone()
    oz.ozaki2_dgemm("N", "N", 1.0, Ad, Bd, 0.25, C, nmod)
    r, c = sample(M, 256, nmod), sample(N, 256, 50 + nmod)
    want = o2.dgemm("N", "N", 1.0, A[r], B[:, c], 0.25, C0[np.ix_(r, c)], nmod)
    assert same(gather(C, r, c), want), nmod


@pytest.fixture(scope="module")
def c2_inputs():
    import bench
    batch, n = 30, 512
    A_h, B_h = bench.make_inputs(batch, n, 3.0, 1000)
    A = bench.to_dev_batched(torch, A_h, torch.device("cuda"))
    B = bench.to_dev_batched(torch, B_h, torch.device("cuda"))
    return A_h, B_h, A, B


@pytest.mark.parametrize("s", list(range(1, 13)))
@pytest.mark.parametrize("method", ["4m", "3m"])
def test_c2x30_entries_0_and_29_every_s(orc, c2_inputs, s, method):
    """C2 x 30 (480 super-tiles, 6.5 per pair for 4M; 3 x 30 entries for 3M), every s."""
    A_h, B_h, A, B = c2_inputs
    batch, n = A.shape[0], A.shape[1]
    C = oz.colmajor(torch.zeros((batch, n, n), dtype=torch.complex128, device="cuda"))
    fn = oz.zgemm_strided_batched if method == "4m" else oz.zgemm3m_strided_batched
    fn("N", "N", 1.0, A, B, 0.0, C, s)
    r, c = sample(n, 128, s), sample(n, 64, 40 + s)
    for e in (0, batch - 1):
        want = orc.zgemm("N", "N", 1.0, A_h[e][r], B_h[e][:, c], 0.0, None, s, method)
        got = C[e].cpu().numpy()[np.ix_(r, c)]
        assert same(got, want), (method, s, e)


# ---------------------------------------- complex quick returns with a complex beta (R7)
@pytest.mark.parametrize("fn_name,method", [("zgemm", "4m"), ("zgemm3m", "3m")])
@pytest.mark.parametrize("case", ["alpha0", "k0"])
def test_complex_quick_return_complex_beta(orc, fn_name, method, case):
    m, n, k = 70, 50, (0 if case == "k0" else 30)
    A = synth.uniform(m, k, 1, complex_=True)
    B = synth.uniform(k, n, 2, complex_=True)
    C0 = synth.uniform(m, n, 3, complex_=True)
    alpha = 0.0 if case == "alpha0" else 1.5 - 0.5j
    for beta in (0.5 - 0.75j, -1.25 + 0.375j, 0.0):
        C = dev(C0)
        if beta == 0.0:
            C.fill_(complex(float("nan"), float("nan")))
        getattr(oz, fn_name)("N", "N", alpha, dev(A), dev(B), beta, C, 7)
        want = orc.zgemm("N", "N", alpha, A, B, beta, C0, 7, method)
        assert same(C.cpu().numpy(), want), (beta, case)


@pytest.mark.parametrize("fn_name", ["zgemm_strided_batched", "zgemm3m_strided_batched"])
def test_complex_quick_return_batched(orc, fn_name):
    batch, m, n = 3, 40, 33
    C0 = [synth.uniform(m, n, 10 + i, complex_=True) for i in range(batch)]
    Cd = oz.colmajor(torch.stack([dev(x) for x in C0]))
    A = oz.colmajor(torch.zeros((batch, m, 0), dtype=torch.complex128, device="cuda"))
    B = oz.colmajor(torch.zeros((batch, 0, n), dtype=torch.complex128, device="cuda"))
    beta = 0.25 + 1.5j
    getattr(oz, fn_name)("N", "N", 2.0 + 1.0j, A, B, beta, Cd, 5)
    for i in range(batch):
        want = orc.zgemm("N", "N", 2.0 + 1.0j, np.zeros((m, 0), complex), np.zeros((0, n), complex),
                         beta, C0[i], 5)
        assert same(Cd[i].cpu().numpy(), want), i


# ------------------------------------------------ R9 hand-derived golden on the GPU
def test_complex_embedding_golden_gpu():
    import os
    gold = os.path.join(os.path.dirname(__file__), "golden", "complex_embedding.txt")
    for ln in open(gold):
        if not ln.strip() or ln.startswith("#"):
            continue
        meth, s_s, a_s, b_s, want_s, _ = [x.strip() for x in ln.split("|")]
        ar, ai = (float.fromhex(x) for x in a_s.split())
        br, bi = (float.fromhex(x) for x in b_s.split())
        wr, wi = (float.fromhex(x) for x in want_s.split())
        A = dev(np.array([[complex(ar, ai)]]))
        B = dev(np.array([[complex(br, bi)]]))
        C = dev(np.zeros((1, 1), complex))
        (oz.zgemm if meth == "4m" else oz.zgemm3m)("N", "N", 1.0, A, B, 0.0, C, int(s_s))
        got = C.cpu().numpy()[0, 0]
        assert got.real == wr and got.imag == wi, (ln, got)
