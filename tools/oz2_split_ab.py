"""A/B of the Ozaki-II long-row split on C3 (DGEMM 8192^3): the single-read cluster kernel vs the
two-kernel form (OZAKI_SPLIT_CLUSTER=0), per moduli count: split / residue GEMM / CRT ms per call
(phase profiler) and whether C is bitwise equal.  usage: python tools/oz2_split_ab.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_29975_b200 as oz  # noqa: E402

n = 8192
st = torch.cuda.current_stream()
A_h, B_h = bench.c3_inputs(n, "U")
A = oz.colmajor(torch.from_numpy(A_h).cuda())
B = oz.colmajor(torch.from_numpy(B_h).cuda())
C = torch.zeros((n, n), dtype=torch.float64, device="cuda").t()
res = {}
for nmod in (12, 14, 16):
    ref = None
    for name, env in (("cluster", {}), ("two_kernel", {"OZAKI_SPLIT_CLUSTER": "0"})):
        os.environ.pop("OZAKI_SPLIT_CLUSTER", None)
        os.environ.update(env)
        call = lambda nmod=nmod: oz.ozaki2_dgemm("N", "N", 1.0, A, B, 0.0, C, nmod)   # noqa: E731
        for _ in range(2):
            call()
        ms, g, ph, clk = bench.profiled(torch, oz, st, call, 5, 0)
        c = C.clone()
        ref = c if ref is None else ref
        res[f"N{nmod}_{name}"] = {"split": round(ph.get("k1_exponent", 0) + ph.get("k1_slice", 0), 4),
                                 "gemm": round(g, 4), "crt": ph.get("other"), "step_ms": round(ms, 4),
                                 "tflops": round(2 * n ** 3 / ms / 1e9, 1), "mhz": clk.get("sm_mhz"),
                                 "bitwise_equal": bool(torch.equal(c, ref))}
        print(name, nmod, res[f"N{nmod}_{name}"], flush=True)
os.environ.pop("OZAKI_SPLIT_CLUSTER", None)
print(json.dumps(res))
