"""A/B of the pair GEMM's pipeline shape (OZAKI_STAGE_KB: minimum stage size, OZAKI_STAGES_MAX:
stage count cap) on C3 (DGEMM 8192^3) at several s and on C2x30: GEMM kernel ms per launch
(phase profiler), call ms, SM clock, bitwise equality with the default."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_29975_b200 as oz  # noqa: E402

KEYS = ("OZAKI_STAGE_KB", "OZAKI_STAGES_MAX")
variants = [("default", {}), ("stages12", {"OZAKI_STAGES_MAX": "12"}), ("stage36k", {"OZAKI_STAGE_KB": "36"}),
            ("stage54k", {"OZAKI_STAGE_KB": "54"}), ("stage36k_12", {"OZAKI_STAGE_KB": "36", "OZAKI_STAGES_MAX": "12"})]
st = torch.cuda.current_stream()
n = 8192
A_h, B_h = bench.c3_inputs(n, "U")
A = oz.colmajor(torch.from_numpy(A_h).cuda())
B = oz.colmajor(torch.from_numpy(B_h).cuda())
C = torch.zeros((n, n), dtype=torch.float64, device="cuda").t()
out = {}
for s in (3, 4, 5, 7):
    ref = None
    for name, env in variants:
        for k in KEYS:
            os.environ.pop(k, None)
        os.environ.update(env)
        call = lambda s=s: oz.dgemm("N", "N", 1.0, A, B, 0.0, C, s)   # noqa: E731
        for _ in range(2):
            call()
        ms, g, ph, clk = bench.profiled(torch, oz, st, call, 4, 0)
        c = C.clone()
        ref = c if ref is None else ref
        out[f"c3_s{s}_{name}"] = {"gemm_ms": round(g, 4), "call_ms": round(ms, 4), "mhz": clk.get("sm_mhz"),
                                  "tops": round(s * (s + 1) * n ** 3 / g / 1e9, 1),
                                  "bitwise_equal": bool(torch.equal(c, ref))}
        print(f"c3 s{s}", name, out[f"c3_s{s}_{name}"], flush=True)
del A, B, C
torch.cuda.empty_cache()
A_h, B_h = bench.make_inputs(30, 512, 3.0, 1000)
Az, Bz = bench.to_dev_batched(torch, A_h, "cuda"), bench.to_dev_batched(torch, B_h, "cuda")
Cz = torch.zeros((30, 512, 512), dtype=torch.complex128, device="cuda").transpose(1, 2)
for s in (4, 7):
    ref = None
    for name, env in variants:
        for k in KEYS:
            os.environ.pop(k, None)
        os.environ.update(env)
        call = lambda s=s: oz.zgemm_strided_batched("N", "N", 1.0, Az, Bz, 0.0, Cz, s)   # noqa: E731
        for _ in range(3):
            call()
        ms, g, ph, clk = bench.profiled(torch, oz, st, call, 20, 0)
        c = Cz.clone()
        ref = c if ref is None else ref
        out[f"c2x30_s{s}_{name}"] = {"gemm_ms": round(g, 4), "call_ms": round(ms, 4), "mhz": clk.get("sm_mhz"),
                                     "bitwise_equal": bool(torch.equal(c, ref))}
        print(f"c2x30 s{s}", name, out[f"c2x30_s{s}_{name}"], flush=True)
for k in KEYS:
    os.environ.pop(k, None)
print(json.dumps(out))
