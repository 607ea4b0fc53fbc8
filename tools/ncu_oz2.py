"""One Ozaki-II C3 call (N moduli) after warm-up, for ncu captures of the CRT split / CRT kernels.
usage: ncu ... python tools/ncu_oz2.py [N]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_29975_b200 as oz  # noqa: E402

nmod = int(sys.argv[1]) if len(sys.argv) > 1 else 14
A_h, B_h = bench.c3_inputs(8192, "U")
A = oz.colmajor(torch.from_numpy(A_h).cuda())
B = oz.colmajor(torch.from_numpy(B_h).cuda())
C = torch.zeros((8192, 8192), dtype=torch.float64, device="cuda").t()
for _ in range(3):
    oz.ozaki2_dgemm("N", "N", 1.0, A, B, 0.0, C, nmod)
torch.cuda.synchronize()
