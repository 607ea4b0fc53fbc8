"""Per-role timers of the GEMM kernel on the bench workload (debug aid)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_29975_b200 as oz
import bench

def run(n=512, batch=30, s=7, method="4m", kind="z"):
    dev = torch.device("cuda", 0)
    if kind == "z":
        A_h, B_h = bench.make_inputs(batch, n, 3.0, 1000)
        A = bench.to_dev_batched(torch, A_h, dev); B = bench.to_dev_batched(torch, B_h, dev)
        C = torch.zeros((batch, n, n), dtype=torch.complex128, device=dev).transpose(1, 2)
        fn = oz.zgemm_strided_batched if method == "4m" else oz.zgemm3m_strided_batched
        call = lambda: fn("N", "N", 1.0, A, B, 0.0, C, s)
    else:
        A = torch.rand((n, n), dtype=torch.float64, device=dev).t(); B = torch.rand((n, n), dtype=torch.float64, device=dev).t()
        C = torch.zeros((n, n), dtype=torch.float64, device=dev).t()
        call = lambda: oz.dgemm("N", "N", 1.0, A, B, 0.0, C, s)
    for _ in range(3): call()
    torch.cuda.synchronize()
    oz.debug_timing(True); oz.debug_timing(True, read=True)
    oz.profile_enable(True); oz.profile_read()
    reps = 5
    for _ in range(reps): call()
    torch.cuda.synchronize()
    t = oz.debug_timing(False, read=True)
    pr = oz.profile_read(); oz.profile_enable(False)
    ctas = 148 * reps
    out = {k: round(v / ctas / 1.9e3, 1) for k, v in t.items()}   # us per CTA per launch at ~1.9 GHz
    out["gemm_ms"] = round(pr["k2_gemm"]["ms"] / max(1, pr["k2_gemm"]["launches"]), 4)
    out["config"] = f"{kind} n={n} batch={batch} s={s} {method}"
    print(json.dumps(out))

if __name__ == "__main__":
    run()
    run(s=4)
    run(s=8)
    run(n=8192, batch=1, s=7, kind="d")
