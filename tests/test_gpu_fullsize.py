"""Parity at BASELINE.json's FULL sizes, in the launch configuration bench.py times
(strided-batched 4M for C2/C4, one DGEMM for C3/C5), on sampled outputs the oracle computes
row by row: the oracle sees FULL rows of op(A) and FULL columns of op(B), so its exponents are
the ones of the whole problem, and each sampled C entry must match bit for bit.  Samples
include tile edges (rows 127/128/255/256, columns 63/64/127/128) and the last row / column.
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
    return oz.colmajor(torch.from_numpy(np.asfortranarray(x)).to("cuda"))


def stack_dev(blocks):
    return oz.colmajor(torch.stack([dev(b) for b in blocks]))


def rows_sample(n):
    return np.unique(np.clip(np.r_[0, 1, 127, 128, 255, 256, 511, 512, n // 2, n - 2, n - 1], 0, n - 1))


def cols_sample(n):
    return np.unique(np.clip(np.r_[0, 63, 64, 127, 128, 129, 1000, n // 3, n - 1], 0, n - 1))


def test_c2_bench_workload_full_entries(orc):
    """bench.py default: 30 x ZGEMM 512^3 KKR(gamma=3), 4M, s=7 -- entries 0 and 29 in full."""
    import bench
    batch, n, s = 30, 512, 7
    A_h, B_h = bench.make_inputs(batch, n, 3.0, 1000)
    A = bench.to_dev_batched(torch, A_h, torch.device("cuda"))
    B = bench.to_dev_batched(torch, B_h, torch.device("cuda"))
    C = torch.zeros((batch, n, n), dtype=torch.complex128, device="cuda").transpose(1, 2)
    oz.zgemm_strided_batched("N", "N", 1.0, A, B, 0.0, C, s)
    for e in (0, batch - 1):
        want = orc.zgemm("N", "N", 1.0, np.asfortranarray(A_h[e]), np.asfortranarray(B_h[e]), 0.0, None, s)
        got = C[e].cpu().numpy()
        assert (got.real == want.real).all() and (got.imag == want.imag).all(), e


def test_c3_dgemm_8192(orc):
    n, s = 8192, 7
    A = synth.uniform(n, n, 1)
    B = synth.uniform(n, n, 2)
    C = torch.zeros((n, n), dtype=torch.float64, device="cuda").t()
    oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, s)
    r, c = rows_sample(n), cols_sample(n)
    got = C.cpu().numpy()[np.ix_(r, c)]
    want = orc.dgemm("N", "N", 1.0, A[r], B[:, c], 0.0, None, s)
    assert (got == want).all()
    # Ozaki-II on the same full problem, N = 16
    from oracle import ozaki2 as o2
    oz.ozaki2_dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, 16)
    got = C.cpu().numpy()[np.ix_(r[:8], c[:8])]
    want = o2.dgemm("N", "N", 1.0, A[r[:8]], B[:, c[:8]], 0.0, None, 16)
    assert (got == want).all()


@pytest.mark.parametrize("s", [3, 9])
def test_c3_dgemm_8192_other_slices(orc, s):
    """The C3 sweep's ends at full size: s = 3 (one-pass plan, 54-KB stages of three k-blocks)
    and s = 9 (three passes, 128-bit fixed point in the split); both through the single-read
    cluster split.  Plus Ozaki-II N = 12 (256 x 512 residue tiles) on the same problem."""
    n = 8192
    A = synth.spread(n, n, 3, phi=1.0)
    B = synth.spread(n, n, 4, phi=1.0)
    C = torch.zeros((n, n), dtype=torch.float64, device="cuda").t()
    oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, s)
    r, c = rows_sample(n), cols_sample(n)
    got = C.cpu().numpy()[np.ix_(r, c)]
    want = orc.dgemm("N", "N", 1.0, A[r], B[:, c], 0.0, None, s)
    assert (got == want).all()
    if s == 3:
        from oracle import ozaki2 as o2
        oz.ozaki2_dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, 12)
        got = C.cpu().numpy()[np.ix_(r[:8], c[:8])]
        want = o2.dgemm("N", "N", 1.0, A[r[:8]], B[:, c[:8]], 0.0, None, 12)
        assert (got == want).all()


def test_c4_batched_256_zgemm_1024(orc):
    """256 x ZGEMM 1024^3 KKR(gamma=1), s=7, one strided-batched call (8 distinct blocks tiled,
    as bench.py --workload c4)."""
    n, batch, s, distinct = 1024, 256, 7, 8
    As = [synth.kkr(n, n, seed=10 + i, gamma=1.0) for i in range(distinct)]
    Bs = [synth.kkr(n, n, seed=50 + i, gamma=1.0) for i in range(distinct)]
    Ad, Bd = stack_dev(As), stack_dev(Bs)
    A = oz.colmajor(torch.stack([Ad[i % distinct] for i in range(batch)]))
    B = oz.colmajor(torch.stack([Bd[i % distinct] for i in range(batch)]))
    del Ad, Bd
    C = oz.colmajor(torch.zeros((batch, n, n), dtype=torch.complex128, device="cuda"))
    oz.zgemm_strided_batched("N", "N", 1.0, A, B, 0.0, C, s)
    r, c = rows_sample(n), cols_sample(n)
    for e in (0, 131, batch - 1):
        got = C[e].cpu().numpy()[np.ix_(r, c)]
        want = orc.zgemm("N", "N", 1.0, As[e % distinct][r], Bs[e % distinct][:, c], 0.0, None, s)
        assert (got.real == want.real).all() and (got.imag == want.imag).all(), e


def test_c5_dgemm_32768x32768x4096(orc):
    m, n, k, s = 32768, 32768, 4096, 7
    A = synth.spread(m, k, 1, phi=4.0)
    B = synth.spread(k, n, 2, phi=4.0)
    C = torch.zeros((n, m), dtype=torch.float64, device="cuda").t()
    oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, s)
    r, c = rows_sample(m), cols_sample(n)
    got = C[torch.from_numpy(r).cuda()][:, torch.from_numpy(c).cuda()].cpu().numpy()
    want = orc.dgemm("N", "N", 1.0, A[r], B[:, c], 0.0, None, s)
    assert (got == want).all()
