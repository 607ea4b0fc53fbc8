"""A/B of the one-GEMM host offload (C3 e2e: DGEMM 8192^3, s=7, pinned host A, B, C) over panel
sizes (OZAKI_OFFLOAD_PANEL_ROWS / _COLS): ms per call (CUDA events, 3 calls after 1 warm-up),
SM clock, bitwise equality with the first variant."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_29975_b200 as oz  # noqa: E402

n, s = 8192, 7
A_h, B_h = bench.c3_inputs(n, "U")
Ap = torch.from_numpy(np.ascontiguousarray(A_h.T)).pin_memory().t()
Bp = torch.from_numpy(np.ascontiguousarray(B_h.T)).pin_memory().t()
Cp = torch.empty((n, n), dtype=torch.float64).pin_memory().t()
st = torch.cuda.current_stream()
variants = [("default", {}), ("r1024_c2048", {"OZAKI_OFFLOAD_PANEL_ROWS": "1024"}),
            ("r2048_c8192", {"OZAKI_OFFLOAD_PANEL_COLS": "8192"}),
            ("r1024_c8192", {"OZAKI_OFFLOAD_PANEL_ROWS": "1024", "OZAKI_OFFLOAD_PANEL_COLS": "8192"}),
            ("r512_c8192", {"OZAKI_OFFLOAD_PANEL_ROWS": "512", "OZAKI_OFFLOAD_PANEL_COLS": "8192"}),
            ("r4096_c1024", {"OZAKI_OFFLOAD_PANEL_ROWS": "4096", "OZAKI_OFFLOAD_PANEL_COLS": "1024"})]
res, ref = {}, None
for name, env in variants:
    for k in ("OZAKI_OFFLOAD_PANEL_ROWS", "OZAKI_OFFLOAD_PANEL_COLS"):
        os.environ.pop(k, None)
    os.environ.update(env)
    call = lambda: oz.dgemm("N", "N", 1.0, Ap, Bp, 0.0, Cp, s)   # noqa: E731
    call()
    ms, clk = bench.timed(torch, st, call, 3, 0)
    c = Cp.clone()
    ref = c if ref is None else ref
    res[name] = {"ms": round(ms, 3), "tflops": round(2 * n ** 3 / ms / 1e9, 2), "mhz": clk.get("sm_mhz"),
                 "bitwise_equal": bool(torch.equal(c, ref))}
    print(name, res[name], flush=True)
print(json.dumps(res))
