"""A/B of the Ozaki-II residue-GEMM tile width (OZAKI_CRT_NW = 1: 256 x 256 tiles, double-buffered
accumulators; 2: 256 x 512, each A tile feeding two MMAs) on C3 (DGEMM 8192^3) and C2x30-shaped
ZGEMMs: residue GEMM ms per launch (phase profiler), call ms, clock, bitwise equality."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_29975_b200 as oz  # noqa: E402

st = torch.cuda.current_stream()
n = 8192
A_h, B_h = bench.c3_inputs(n, "U")
A = oz.colmajor(torch.from_numpy(A_h).cuda())
B = oz.colmajor(torch.from_numpy(B_h).cuda())
C = torch.zeros((n, n), dtype=torch.float64, device="cuda").t()
res = {}
for rep in range(2):
    for nmod in (12, 14, 16):
        for nw in ("1", "2"):
            os.environ["OZAKI_CRT_NW"] = nw
            call = lambda nmod=nmod: oz.ozaki2_dgemm("N", "N", 1.0, A, B, 0.0, C, nmod)   # noqa: E731
            for _ in range(2):
                call()
            ms, g, ph, clk = bench.profiled(torch, oz, st, call, 4, 0)
            key = f"c3_N{nmod}_nw{nw}_r{rep}"
            res[key] = {"gemm_ms": round(g, 4), "call_ms": round(ms, 4), "mhz": clk.get("sm_mhz"),
                        "tops": round(2 * nmod * n ** 3 / g / 1e9, 1), "sum": float(C.sum())}
            print(key, res[key], flush=True)
del A, B, C
torch.cuda.empty_cache()
A_h, B_h = bench.make_inputs(30, 512, 3.0, 1000)
Az, Bz = bench.to_dev_batched(torch, A_h, "cuda"), bench.to_dev_batched(torch, B_h, "cuda")
Cz = torch.zeros((30, 512, 512), dtype=torch.complex128, device="cuda").transpose(1, 2)
ref = None
for nw in ("1", "2"):
    os.environ["OZAKI_CRT_NW"] = nw
    call = lambda: oz.ozaki2_zgemm_strided_batched("N", "N", 1.0, Az, Bz, 0.0, Cz, 16)   # noqa: E731
    for _ in range(3):
        call()
    ms, g, ph, clk = bench.profiled(torch, oz, st, call, 10, 0)
    c = Cz.clone()
    ref = c if ref is None else ref
    res[f"c2x30_N16_nw{nw}"] = {"gemm_ms": round(g, 4), "call_ms": round(ms, 4), "mhz": clk.get("sm_mhz"),
                                "bitwise_equal": bool(torch.equal(c, ref))}
    print(f"c2x30_N16_nw{nw}", res[f"c2x30_N16_nw{nw}"], flush=True)
os.environ.pop("OZAKI_CRT_NW", None)
print(json.dumps(res))
