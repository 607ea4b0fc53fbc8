"""A/B of the long-row split forms on C3 (DGEMM 8192^3) and C5-depth (k = 4096) operands:
the single-read cluster kernel (chunk OZAKI_SPLIT_KC) vs the two-kernel form
(OZAKI_SPLIT_CLUSTER=0).  Prints per variant the split ms per call (phase profiler, CUDA events
on the launch stream), its HBM fraction on algorithmic bytes and whether C is bitwise equal to
the first variant's.  usage: python tools/split_cluster_ab.py [n] [k]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_29975_b200 as oz  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
k = int(sys.argv[2]) if len(sys.argv) > 2 else n
peak = bench.hbm_peak()[0]
g = torch.Generator().manual_seed(1)
A = oz.colmajor((torch.rand((n, k), generator=g, dtype=torch.float64) * 2 - 1).cuda())
B = oz.colmajor((torch.rand((k, n), generator=g, dtype=torch.float64) * 2 - 1).cuda())
C = torch.zeros((n, n), dtype=torch.float64, device="cuda").t()
st = torch.cuda.current_stream()
variants = [("rg8_kc512", {}), ("rg16_kc512", {"OZAKI_SPLIT_RG": "16"}),
            ("rg8_kc1024", {"OZAKI_SPLIT_RG": "8", "OZAKI_SPLIT_KC": "1024"}),
            ("two_kernel", {"OZAKI_SPLIT_CLUSTER": "0"})]
KEYS = ("OZAKI_SPLIT_KC", "OZAKI_SPLIT_CLUSTER", "OZAKI_SPLIT_RG", "OZAKI_SPLIT_PERSIST")
out = {"n": n, "k": k, "peak_gbs": peak}
for s in (3, 7):
    ref = None
    for name, env in variants:
        for key in KEYS:
            os.environ.pop(key, None)
        os.environ.update(env)
        call = lambda s=s: oz.dgemm("N", "N", 1.0, A, B, 0.0, C, s)   # noqa: E731
        for _ in range(3):
            call()
        ms, gemm_ms, ph, clk = bench.profiled(torch, oz, st, call, 10, 0)
        split = ph.get("k1_exponent", 0.0) + ph.get("k1_slice", 0.0)
        byts = 8 * n * k * 2 + s * n * k * 2 + 8 * n
        c = C.clone()
        if ref is None:
            ref = c
        out[f"s{s}_{name}"] = {"split_ms": round(split, 4), "phase": ph, "step_ms": round(ms, 4),
                               "gbs": round(byts / split / 1e6, 1), "frac": round(byts / split / 1e6 / peak, 3),
                               "bitwise_equal": bool(torch.equal(c, ref)), "mhz": clk.get("sm_mhz")}
        print(name, s, out[f"s{s}_{name}"], flush=True)
for key in KEYS:
    os.environ.pop(key, None)
print(json.dumps(out))
