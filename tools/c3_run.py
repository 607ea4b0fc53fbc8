"""Runs Ozaki-I DGEMM 8192^3 (C3) a few times (profiling target for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_29975_b200 as oz  # noqa: E402

s = int(os.environ.get("SLICES", "7"))
n = 8192
g = torch.Generator(device="cuda").manual_seed(5)
A = (torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
B = (torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
C = torch.zeros((n, n), dtype=torch.float64, device="cuda").t()
for _ in range(3):
    oz.dgemm("N", "N", 1.0, A, B, 0.0, C, s)
torch.cuda.synchronize()
print("done")
