"""One C3 DGEMM 8192^3 call per requested s (after warm-up calls) for ncu captures of the slice
GEMM: `ncu -k regex:k_gemm_lv2 -s <warmups> -c 1 ... python tools/ncu_c3.py --s 7`.
The inputs are bench.py's (c3_inputs, family U)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_29975_b200 as oz  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--s", type=int, nargs="+", default=[7])
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--warm", type=int, default=2)
ap.add_argument("--fam", default="U")
ap.add_argument("--alpha", type=float, default=1.0)
ap.add_argument("--beta", type=float, default=0.0)
a = ap.parse_args()
A_h, B_h = bench.c3_inputs(a.n, a.fam)
A = oz.colmajor(torch.from_numpy(A_h).cuda())
B = oz.colmajor(torch.from_numpy(B_h).cuda())
C = torch.zeros((a.n, a.n), dtype=torch.float64, device="cuda").t()
for s in a.s:
    for _ in range(a.warm + 1):
        oz.dgemm("N", "N", a.alpha, A, B, a.beta, C, s)
    torch.cuda.synchronize()
print("done", a.s)
