"""Small invocations of every kernel path, for compute-sanitizer runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_2603_29975_b200 as oz

def dev(x):
    return oz.colmajor(torch.from_numpy(np.asfortranarray(x)).cuda())

A = synth.spread(200, 70, seed=1); B = synth.uniform(70, 150, seed=2)
C = dev(np.zeros((200, 150)))
for s in (3, 7, 13):
    oz.dgemm("N", "T", 1.0, dev(A), dev(B.T.copy()), 0.0, C, s)
Z = synth.kkr(100, 60, seed=3); W = synth.kkr(60, 90, seed=4)
Zc = dev(np.zeros((100, 90), np.complex128))
oz.zgemm("N", "N", 1.0, dev(Z), dev(W), 0.5, Zc, 7)
oz.zgemm3m("C", "N", 1.0, dev(np.conj(Z.T).copy()), dev(W), 0.0, Zc, 5)
os.environ["OZAKI_KCHUNK_KB"] = "1"
oz.dgemm("N", "N", 1.0, dev(A), dev(synth.uniform(70, 150, seed=5)), 0.0, C, 6)
del os.environ["OZAKI_KCHUNK_KB"]
oz.debug_split("B", "z", "N", dev(W), 8)
oz.debug_level_sums("N", "N", dev(A), dev(synth.uniform(70, 150, seed=5)), 4)
# Ozaki-II: split variant, residue GEMM, CRT (real and 4M, ragged)
oz.ozaki2_dgemm("N", "T", 1.0, dev(A), dev(B.T.copy()), 0.0, C, 14)
oz.ozaki2_zgemm("N", "N", 1.0, dev(Z), dev(W), 0.5, Zc, 12)
# NEXT-4: full pair set, per-block exponents
oz.set_pair_set("full")
oz.dgemm("N", "N", 1.0, dev(A), dev(synth.uniform(70, 150, seed=6)), 0.0, C, 5)
oz.set_pair_set("triangular")
oz.set_exponent_block(32)
oz.zgemm("N", "N", 1.0, dev(Z), dev(W), 0.0, Zc, 6)
oz.set_exponent_block(0)
# round-1 additions: long-row split (exponent kernel + per-window digits), s = 9..12 fast split,
# Ozaki-II through the fast split (both operands, conj), cross-call overlap (PDL split after GEMM)
os.environ["OZAKI_SPLIT_LONG"] = "1"
oz.dgemm("N", "N", 1.0, dev(synth.uniform(90, 700, seed=7)), dev(synth.uniform(700, 60, seed=8)), 0.0,
         dev(np.zeros((90, 60))), 7)
oz.zgemm("N", "C", 1.0, dev(synth.kkr(40, 600, seed=9)), dev(synth.kkr(50, 600, seed=10)), 0.0,
         dev(np.zeros((40, 50), np.complex128)), 6)
oz.ozaki2_dgemm("T", "N", 1.0, dev(synth.uniform(700, 50, seed=11)), dev(synth.uniform(700, 40, seed=12)), 0.0,
                dev(np.zeros((50, 40))), 10)
del os.environ["OZAKI_SPLIT_LONG"]
oz.dgemm("N", "N", 1.0, dev(A), dev(synth.uniform(70, 150, seed=13)), 0.0, C, 11)
oz.ozaki2_zgemm("C", "N", 1.0, dev(np.conj(Z.T).copy()), dev(W), 0.0, Zc, 16)
oz.set_overlap(True)
Zd, Wd = dev(Z), dev(W)
for _ in range(3):
    oz.zgemm("N", "N", 1.0, Zd, Wd, 0.0, Zc, 7)
Cd = dev(np.zeros((200, 150)))
oz.dgemm("N", "N", 1.0, dev(A), dev(synth.uniform(70, 150, seed=14)), 0.0, Cd, 7)
oz.dgemm("N", "N", 1.0, Cd, dev(synth.uniform(150, 150, seed=15)), 0.0, C, 7)
oz.set_overlap(False)
# round-2 additions: split-K (forced S = 3, real / 4M / 3M / full pairs, and a split-K call under
# cross-call overlap), the general alpha / beta (GAB) store, the emulated TRSM (all sides, real
# and complex, host pointers), the 2-D block host offload
os.environ["OZAKI_SPLITK"] = "3"
oz.dgemm("N", "N", -1.0, dev(synth.uniform(130, 400, seed=16)), dev(synth.uniform(400, 90, seed=17)), 1.0,
         dev(synth.uniform(130, 90, seed=18)), 7)
oz.zgemm("N", "C", 0.5 - 0.5j, dev(synth.kkr(70, 300, seed=19)), dev(synth.kkr(60, 300, seed=20)), 1.0,
         dev(synth.uniform(70, 60, seed=21, complex_=True)), 6)
oz.zgemm3m("N", "N", 1.0, dev(synth.kkr(70, 300, seed=22)), dev(synth.kkr(300, 60, seed=23)), 0.0,
           dev(np.zeros((70, 60), np.complex128)), 5)
oz.set_pair_set("full")
oz.dgemm("N", "N", 1.0, dev(synth.uniform(130, 400, seed=24)), dev(synth.uniform(400, 90, seed=25)), 0.0,
         dev(np.zeros((130, 90))), 4)
oz.set_pair_set("triangular")
oz.set_overlap(True)
for _ in range(2):
    oz.dgemm("N", "N", 1.0, dev(synth.uniform(130, 400, seed=26)), dev(synth.uniform(400, 90, seed=27)), 0.0,
             dev(np.zeros((130, 90))), 6)
oz.set_overlap(False)
del os.environ["OZAKI_SPLITK"]
oz.set_trsm_block(32)
for side, uplo, ta in (("L", "L", "N"), ("L", "U", "T"), ("R", "U", "N"), ("R", "L", "C")):
    Tm = np.tril(synth.uniform(70, 70, seed=28, complex_=True)) * 0.2 + 2 * np.eye(70)
    Tm = Tm if uplo == "L" else Tm.T.copy()
    Bm = synth.uniform(70, 40, seed=29, complex_=True) if side == "L" else synth.uniform(40, 70, seed=29, complex_=True)
    oz.ztrsm(side, uplo, ta, "N", 0.5 + 0.5j, dev(Tm), dev(Bm), 6)
    oz.dtrsm(side, uplo, "T" if ta == "C" else ta, "U", 1.0, dev(Tm.real.copy()), dev(Bm.real.copy()), 6)
hT = torch.from_numpy(np.asfortranarray(np.tril(synth.uniform(50, 50, seed=30)) + 2 * np.eye(50)))
hB = torch.from_numpy(np.asfortranarray(synth.uniform(50, 20, seed=31)))
oz.dtrsm("L", "L", "N", "N", 1.0, hT, hB, 7)
oz.set_trsm_block(128)
os.environ["OZAKI_OFFLOAD_PANEL_COLS"] = "64"
os.environ["OZAKI_OFFLOAD_PANEL_ROWS"] = "96"
hA = torch.from_numpy(np.asfortranarray(synth.uniform(200, 90, seed=32)))
hBB = torch.from_numpy(np.asfortranarray(synth.uniform(90, 150, seed=33)))
hC = torch.from_numpy(np.asfortranarray(synth.uniform(200, 150, seed=34)))
oz.dgemm("N", "N", 1.0, hA, hBB, 0.5, hC, 7)
del os.environ["OZAKI_OFFLOAD_PANEL_COLS"], os.environ["OZAKI_OFFLOAD_PANEL_ROWS"]
# round-2 session-3 additions: the single-read cluster split (k_split_cluster: DSMEM pushes of the
# partial row maxima, Ozaki-I digits and Ozaki-II residues, 8- and 16-row groups, padded leading
# dimensions, TT layouts, a batch, and a PDL launch under cross-call overlap)
Ak = synth.uniform(40, 3000, seed=35)
Bk = synth.spread(3000, 36, seed=36, phi=1.0)
Ck = dev(np.zeros((40, 36)))
oz.dgemm("N", "N", 1.0, dev(Ak), dev(Bk), 0.0, Ck, 7)
oz.dgemm("T", "T", 1.0, dev(Ak.T.copy()), dev(Bk.T.copy()), 0.0, Ck, 4)
os.environ["OZAKI_SPLIT_RG"] = "16"
big = np.zeros((41, 3000)); big[:40] = Ak
oz.dgemm("N", "N", 1.0, dev(big)[:40], dev(Bk), 0.0, Ck, 9)
del os.environ["OZAKI_SPLIT_RG"]
oz.dgemm("N", "N", 1.0, dev(synth.uniform(20, 8192, seed=37)), dev(synth.uniform(8192, 24, seed=38)), 0.0,
         dev(np.zeros((20, 24))), 5)
oz.ozaki2_dgemm("N", "N", 1.0, dev(Ak), dev(Bk), 0.0, Ck, 14)
tAk = torch.stack([dev(Ak), dev(Ak)]).transpose(1, 2).contiguous().transpose(1, 2)
tBk = torch.stack([dev(Bk), dev(Bk)]).transpose(1, 2).contiguous().transpose(1, 2)
tCk = torch.zeros((2, 36, 40), dtype=torch.float64, device="cuda").transpose(1, 2)
oz.dgemm_strided_batched("N", "N", 1.0, tAk, tBk, 0.0, tCk, 6)
oz.set_overlap(True)
Akd, Bkd = dev(Ak), dev(Bk)
for _ in range(3):
    oz.dgemm("N", "N", 1.0, Akd, Bkd, 0.0, Ck, 7)
oz.set_overlap(False)
torch.cuda.synchronize()
print("sanitize_check done")
