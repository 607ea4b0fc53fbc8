"""Split-K for small problems: when the super-tiles leave more than half of
the CTA pairs idle, each tile runs as S units over equal shares of the k-blocks, every unit
writes its EXACT integer partials (the int64 prefix of the first pass's levels, the int32 sums
of the later levels) and k_splitk_combine adds them and runs the unchanged FP64 combine and
store.  Integer sums are order-free, so the result must equal the oracle bit for bit for every
S.  OZAKI_SPLITK=n forces S (read per call)."""
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


@pytest.mark.parametrize("S", [2, 3, 4, 7])
@pytest.mark.parametrize("s", [1, 2, 3, 4, 5, 7, 8, 9, 12])
def test_dgemm_forced_splitk(orc, monkeypatch, S, s):
    monkeypatch.setenv("OZAKI_SPLITK", str(S))
    m, n, k = 300, 200, 37 * 32 + 11          # KB = 38 k-blocks: uneven shares, ragged K
    A = synth.spread(m, k, 100 + s, phi=1.5)
    B = synth.uniform(k, n, 200 + s)
    C0 = synth.uniform(m, n, 300 + s)
    C = dev(C0)
    oz.dgemm("N", "N", -1.0, dev(A), dev(B), 0.5, C, s)
    assert same(C.cpu().numpy(), orc.dgemm("N", "N", -1.0, A, B, 0.5, C0, s)), (S, s)


@pytest.mark.parametrize("S", [2, 5])
@pytest.mark.parametrize("ta,tb", [("T", "N"), ("N", "T"), ("T", "T")])
def test_dgemm_forced_splitk_trans_beta0(orc, monkeypatch, S, ta, tb):
    monkeypatch.setenv("OZAKI_SPLITK", str(S))
    m, n, k, s = 129, 257, 700, 7
    A = synth.uniform(m, k, 1) if ta == "N" else synth.uniform(k, m, 1)
    B = synth.spread(k, n, 2, phi=2.0) if tb == "N" else synth.spread(n, k, 2, phi=2.0)
    C = torch.full((n, m), float("nan"), dtype=torch.float64, device="cuda").t()
    oz.dgemm(ta, tb, 1.0, dev(A), dev(B), 0.0, C, s)
    assert same(C.cpu().numpy(), orc.dgemm(ta, tb, 1.0, A, B, 0.0, None, s))


@pytest.mark.parametrize("S", [2, 4])
@pytest.mark.parametrize("method", ["4m", "3m"])
def test_zgemm_forced_splitk(orc, monkeypatch, S, method):
    monkeypatch.setenv("OZAKI_SPLITK", str(S))
    m, n, k, s = 200, 150, 333, 6
    A = synth.kkr(m, k, seed=5, gamma=1.0)
    B = synth.kkr(k, n, seed=6, gamma=1.0)
    C0 = synth.uniform(m, n, 7, complex_=True)
    C = dev(C0)
    fn = oz.zgemm if method == "4m" else oz.zgemm3m
    fn("N", "C", 0.5 - 0.25j, dev(A), dev(np.conj(B.T).copy()), 1.0 + 0.5j, C, s)
    assert same(C.cpu().numpy(), orc.zgemm("N", "N", 0.5 - 0.25j, A, B, 1.0 + 0.5j, C0, s, method))


@pytest.mark.parametrize("S", [2, 3])
@pytest.mark.parametrize("s", [2, 5, 8])
def test_full_pairs_forced_splitk(orc, monkeypatch, S, s):
    monkeypatch.setenv("OZAKI_SPLITK", str(S))
    m, n, k = 140, 90, 400
    A = synth.spread(m, k, 8, phi=1.0)
    B = synth.uniform(k, n, 9)
    C = dev(np.zeros((m, n)))
    oz.set_pair_set("full")
    try:
        oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, s)
    finally:
        oz.set_pair_set("triangular")
    assert same(C.cpu().numpy(), orc.dgemm("N", "N", 1.0, A, B, 0.0, None, s, pairs="full"))


def test_batched_forced_splitk(orc, monkeypatch):
    monkeypatch.setenv("OZAKI_SPLITK", "3")
    batch, m, n, k, s = 3, 100, 70, 300, 7
    As = [synth.kkr(m, k, seed=10 + i, gamma=1.0) for i in range(batch)]
    Bs = [synth.kkr(k, n, seed=20 + i, gamma=1.0) for i in range(batch)]
    A = oz.colmajor(torch.stack([dev(x) for x in As]))
    B = oz.colmajor(torch.stack([dev(x) for x in Bs]))
    C = oz.colmajor(torch.zeros((batch, m, n), dtype=torch.complex128, device="cuda"))
    oz.zgemm_strided_batched("N", "N", 1.0, A, B, 0.0, C, s)
    for i in range(batch):
        assert same(C[i].cpu().numpy(), orc.zgemm("N", "N", 1.0, As[i], Bs[i], 0.0, None, s)), i


def test_auto_splitk_c2_single_block(orc):
    """configs[1] single block (ZGEMM 512^3, 16 super-tiles on 74 pairs): split-K is chosen by
    the planner; sampled entries (tile edges, last row / column) bit-exact vs the oracle."""
    import bench
    n, s = 512, 7
    A_h, B_h = bench.make_inputs(1, n, 3.0, 1000)
    A, B = dev(A_h[0]), dev(B_h[0])
    C = dev(np.zeros((n, n), complex))
    st0 = oz.get_stats()
    oz.zgemm("N", "N", 1.0, A, B, 0.0, C, s)
    st1 = oz.get_stats()
    assert st1["kernel_launches"] - st0["kernel_launches"] == 3      # split, GEMM units, combine
    r = np.unique(np.r_[0, 1, 127, 128, 255, 256, 383, 384, 510, 511, np.arange(7, n, 53)])
    c = np.unique(np.r_[0, 63, 64, 127, 128, 255, 256, 511, np.arange(5, n, 47)])
    want = orc.zgemm("N", "N", 1.0, A_h[0][r], B_h[0][:, c], 0.0, None, s)
    assert same(C.cpu().numpy()[np.ix_(r, c)], want)


def test_splitk_with_overlap_sequence(orc):
    """Cross-call overlap with split-K calls in the sequence (the stream's last kernel is the
    combine): bitwise identical to the results without overlap."""
    g = synth.rng(3)
    shapes = [(256, 256, 512), (300, 100, 900), (128, 640, 256)]
    ins = [(synth.uniform(m, k, int(g.integers(1 << 20))), synth.uniform(k, n, int(g.integers(1 << 20))))
           for m, n, k in shapes]
    outs = {}
    for ov in (False, True):
        oz.set_overlap(ov)
        try:
            res = []
            for (A, B), (m, n, k) in zip(ins, shapes):
                C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
                oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, 6)
                res.append(C)
            torch.cuda.synchronize()
            outs[ov] = [x.cpu().numpy() for x in res]
        finally:
            oz.set_overlap(False)
    for a, b, (A, B) in zip(outs[False], outs[True], ins):
        assert same(a, b)
        assert same(a, orc.dgemm("N", "N", 1.0, A, B, 0.0, None, 6))
