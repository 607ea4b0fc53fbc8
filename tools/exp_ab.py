"""Experiment: C2x30 (4M) and DGEMM 4096^3 s=7 with alpha = 1, beta = 0 vs the LU update
alpha = -1, beta = 1, production library or libozaki_exp.so.  usage: exp_ab.py {prod|exp}"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2603_29975_b200 as oz  # noqa: E402

if sys.argv[1] == "exp":
    oz.LIB_PATH = os.path.join(ROOT, "paper_2603_29975_b200", "libozaki_exp.so")
import bench  # noqa: E402
import synth  # noqa: E402

st = torch.cuda.current_stream()
res = {"lib": sys.argv[1]}
A_h, B_h = bench.make_inputs(30, 512, 3.0, 1000)
Az, Bz = bench.to_dev_batched(torch, A_h, "cuda"), bench.to_dev_batched(torch, B_h, "cuda")
Cz = torch.zeros((30, 512, 512), dtype=torch.complex128, device="cuda").transpose(1, 2)
n = int(os.environ.get("EXP_N", "4096"))
A = oz.colmajor(torch.from_numpy(synth.uniform(n, n, 1)).cuda())
B = oz.colmajor(torch.from_numpy(synth.uniform(n, n, 2)).cuda())
C = torch.zeros((n, n), dtype=torch.float64, device="cuda").t()
for s in [int(x) for x in os.environ.get("EXP_S", "7").split(",")]:
    for name, (al, be) in (("unit", (1.0, 0.0)), ("lu", (-1.0, 1.0))):
        call = lambda al=al, be=be: oz.zgemm_strided_batched("N", "N", al, Az, Bz, be, Cz, s)   # noqa: E731
        for _ in range(3):
            call()
        ms, clk = bench.timed(torch, st, call, 30, 0)
        res[f"c2x30_s{s}_{name}"] = {"ms": round(ms, 4), "mhz": clk.get("sm_mhz")}
        call = lambda al=al, be=be: oz.dgemm("N", "N", al, A, B, be, C, s)   # noqa: E731
        for _ in range(3):
            call()
        ms, clk = bench.timed(torch, st, call, 10, 0)
        res[f"d{n}_s{s}_{name}"] = {"ms": round(ms, 4), "mhz": clk.get("sm_mhz")}
print(json.dumps(res))
