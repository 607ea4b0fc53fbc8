"""One small call per case (after warm-up) for ncu source-level captures of the pair GEMM.
usage: python tools/ncu_small.py {c1|c2}"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2603_29975_b200 as oz  # noqa: E402


def dev(x):
    return oz.colmajor(torch.from_numpy(np.asfortranarray(x)).cuda())


case = sys.argv[1] if len(sys.argv) > 1 else "c1"
if case == "c1":
    A, B, C = dev(synth.uniform(64, 64, 1)), dev(synth.uniform(64, 64, 2)), dev(np.zeros((64, 64)))
    fn = lambda: oz.dgemm("N", "N", 1.0, A, B, 0.0, C, 7)   # noqa: E731
else:
    A, B = dev(synth.kkr(512, 512, seed=1, gamma=3.0)), dev(synth.kkr(512, 512, seed=2, gamma=3.0))
    C = dev(np.zeros((512, 512), complex))
    fn = lambda: oz.zgemm("N", "N", 1.0, A, B, 0.0, C, 7)   # noqa: E731
for _ in range(4):
    fn()
torch.cuda.synchronize()
