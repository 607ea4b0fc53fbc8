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
torch.cuda.synchronize()
print("sanitize_check done")
