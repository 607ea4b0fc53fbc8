"""A/B timing of library builds (experiment aid): C2x30 (4M s=7) and C3 DGEMM 8192^3 s=7 with
the library at paper_2603_29975_b200/<lib>.  usage: python tools/ab_libs.py libozaki.so ..."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2603_29975_b200 as oz  # noqa: E402

oz.LIB_PATH = os.path.join(ROOT, "paper_2603_29975_b200", sys.argv[1])
import bench  # noqa: E402

st = torch.cuda.current_stream()
A_h, B_h = bench.make_inputs(30, 512, 3.0, 1000)
Az, Bz = bench.to_dev_batched(torch, A_h, "cuda"), bench.to_dev_batched(torch, B_h, "cuda")
Cz = torch.zeros((30, 512, 512), dtype=torch.complex128, device="cuda").transpose(1, 2)
res = {"lib": sys.argv[1]}
for s in (5, 7):
    call = lambda s=s: oz.zgemm_strided_batched("N", "N", 1.0, Az, Bz, 0.0, Cz, s)   # noqa: E731
    for _ in range(5):
        call()
    ms, clk = bench.timed(torch, st, call, 50, 0)
    res[f"c2x30_s{s}"] = {"ms": round(ms, 4), "mhz": clk.get("sm_mhz")}
if len(sys.argv) > 2 and sys.argv[2] == "c3":        # C3 DGEMM 8192^3: step and GEMM kernel time
    A_h, B_h = bench.c3_inputs(8192, "U")
    A = oz.colmajor(torch.from_numpy(A_h).cuda())
    B = oz.colmajor(torch.from_numpy(B_h).cuda())
    C = torch.zeros((8192, 8192), dtype=torch.float64, device="cuda").t()
    for s in (4, 7):
        call = lambda s=s: oz.dgemm("N", "N", 1.0, A, B, 0.0, C, s)   # noqa: E731
        for _ in range(2):
            call()
        ms, clk = bench.timed(torch, st, call, 5, 0)
        _, g, ph, clk2 = bench.profiled(torch, oz, st, call, 3, 0)
        res[f"c3_s{s}"] = {"ms": round(ms, 4), "mhz": clk.get("sm_mhz"), "gemm": round(g, 4), "mhz2": clk2.get("sm_mhz")}
if len(sys.argv) > 2 and sys.argv[2] == "oz2":       # Ozaki-II C3 phases
    A_h, B_h = bench.c3_inputs(8192, "U")
    A = oz.colmajor(torch.from_numpy(A_h).cuda())
    B = oz.colmajor(torch.from_numpy(B_h).cuda())
    C = torch.zeros((8192, 8192), dtype=torch.float64, device="cuda").t()
    for nmod in (12, 14):
        call = lambda nmod=nmod: oz.ozaki2_dgemm("N", "N", 1.0, A, B, 0.0, C, nmod)   # noqa: E731
        for _ in range(2):
            call()
        _, g, ph, clk = bench.profiled(torch, oz, st, call, 3, 0)
        res[f"c3_oz2_N{nmod}"] = {"split": ph.get("k1_slice"), "crt": ph.get("other"), "gemm": round(g, 4),
                                  "mhz": clk.get("sm_mhz")}
print(json.dumps(res), flush=True)
