"""GPU: cross-call overlap (ozaki_set_overlap) -- consecutive Ozaki-I calls on one stream with the
split of call i+1 launched under call i's GEMM (PDL).  Results must be bitwise those of the
same calls without overlap, including: C reused call after call (write-after-write with the GEMM
still running), the previous call's C as the next call's A or B (the split must wait), calls of
other kinds in between (3M, Ozaki-II, quick returns), workspace growth between calls, and
host-pointer (offload) calls."""
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


def batched(xs):
    return torch.stack([dev(x) for x in xs]).transpose(1, 2).contiguous().transpose(1, 2)


def run_sequence(overlap):
    """A fixed sequence of calls; returns every result (host copies) in order."""
    oz.set_overlap(overlap)
    try:
        out = []
        s = 7
        zA = batched([synth.kkr(160, 150, seed=i, gamma=3.0) for i in range(6)])
        zB = batched([synth.kkr(150, 140, seed=20 + i, gamma=1.0) for i in range(6)])
        zC = torch.zeros((6, 140, 160), dtype=torch.complex128, device="cuda").transpose(1, 2)
        for rep in range(4):          # same C every call: WAW with the previous GEMM in flight
            oz.zgemm_strided_batched("N", "N", 1.0 - 0.25j * rep, zA, zB, 0.0, zC, s)
        out.append(zC.cpu().numpy())
        A = dev(synth.spread(200, 200, seed=3, phi=1.0))
        B = dev(synth.uniform(200, 200, seed=4))
        C1 = dev(np.zeros((200, 200)))
        C2 = dev(np.zeros((200, 200)))
        oz.dgemm("N", "N", 1.0, A, B, 0.0, C1, s)
        oz.dgemm("N", "N", 1.0, C1, B, 0.0, C2, s)      # previous C is this call's A: must wait
        oz.dgemm("T", "N", 0.5, B, C2, 0.0, C1, s)      # previous C is this call's B
        out += [C2.cpu().numpy(), C1.cpu().numpy()]
        # other kinds in between, then Ozaki-I again on the same C
        oz.zgemm3m_strided_batched("N", "N", 1.0, zA, zB, 0.0, zC, s)
        oz.dgemm("N", "N", 0.0, A, B, 2.0, C1, s)       # quick return (alpha = 0)
        oz.ozaki2_dgemm("N", "N", 1.0, A, C1, 0.0, C2, 12)
        oz.dgemm("N", "N", 1.0, C2, A, 0.5, C1, s)
        out += [zC.cpu().numpy(), C2.cpu().numpy(), C1.cpu().numpy()]
        # workspace growth (bigger call after smaller ones), then a small one again
        Ab = dev(synth.uniform(700, 900, seed=7))
        Bb = dev(synth.spread(900, 650, seed=8, phi=2.0))
        Cb = dev(np.zeros((700, 650)))
        oz.dgemm("N", "N", 1.0, Ab, Bb, 0.0, Cb, 5)
        oz.dgemm("N", "N", 1.0, A, B, 0.0, C1, 5)
        out += [Cb.cpu().numpy(), C1.cpu().numpy()]
        # host pointers (offload path) in between
        hA = torch.from_numpy(np.asfortranarray(synth.uniform(96, 80, seed=9))).t().contiguous().t().pin_memory()
        hB = torch.from_numpy(np.asfortranarray(synth.uniform(80, 64, seed=10))).t().contiguous().t().pin_memory()
        hC = torch.zeros((64, 96), dtype=torch.float64).t().pin_memory()
        oz.dgemm("N", "N", 1.0, hA, hB, 0.0, hC, s)
        oz.dgemm("N", "N", 1.0, C1, B[:, :200], 0.0, C2, s)
        out += [hC.numpy().copy(), C2.cpu().numpy()]
        # long real rows (k > 2048: the single-read cluster split, PDL-launched after the GEMM):
        # repeated C, then the previous C as the next call's A
        Al = dev(synth.uniform(96, 3000, seed=11))
        Bl = dev(synth.spread(3000, 3000, seed=12, phi=1.0))
        Cl = dev(np.zeros((96, 3000)))
        Cm = dev(np.zeros((96, 3000)))
        for _ in range(2):
            oz.dgemm("N", "N", 1.0, Al, Bl, 0.0, Cl, 6)
        oz.dgemm("N", "N", 1.0, Cl, Bl, 0.0, Cm, 6)
        out += [Cl.cpu().numpy(), Cm.cpu().numpy()]
        torch.cuda.synchronize()
        return out
    finally:
        oz.set_overlap(False)


def test_overlap_sequence_bitwise():
    ref = run_sequence(False)
    for _ in range(2):
        got = run_sequence(True)
        for i, (g, r) in enumerate(zip(got, ref)):
            assert np.array_equal(g, r), f"result {i} differs with overlap on"


def test_overlap_flag_thread_local_default_off():
    assert oz.get_overlap() is False
    oz.set_overlap(True)
    assert oz.get_overlap() is True
    oz.set_overlap(False)
    assert oz.get_overlap() is False


def test_overlap_two_streams_interleaved():
    """Calls alternating between two streams (per-stream overlap state and workspaces), each
    stream's C reused: bitwise equal to the same calls without overlap."""
    s = 6
    A = [dev(synth.uniform(300, 260, seed=30 + i)) for i in range(2)]
    B = [dev(synth.spread(260, 280, seed=40 + i, phi=1.5)) for i in range(2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]

    def run(overlap):
        oz.set_overlap(overlap)
        try:
            C = [dev(np.zeros((300, 280))) for _ in range(2)]
            torch.cuda.synchronize()
            for rep in range(5):
                for i in (0, 1):
                    with torch.cuda.stream(streams[i]):
                        oz.dgemm("N", "N", 1.0 + rep, A[i], B[i], 0.5, C[i], s)
            torch.cuda.synchronize()
            return [c.cpu().numpy() for c in C]
        finally:
            oz.set_overlap(False)

    ref = run(False)
    got = run(True)
    for g, r in zip(got, ref):
        assert np.array_equal(g, r)
