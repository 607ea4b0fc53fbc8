"""Ozaki-I (slices s) vs Ozaki-II (moduli N) on the bench workloads: FP64-eq TFLOP/s,
per-phase device ms (library profiler), GEMM INT8 TOPS, and accuracy on a sample vs the
exact product.  Writes gpurun_out/method_compare.json (summarised into profiles/)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import bench
import oracle
import paper_2603_29975_b200 as oz
import synth


def timed(fn, reps=5, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    oz.profile_enable(True)
    oz.profile_read()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    pr = oz.profile_read()
    oz.profile_enable(False)
    ms = e0.elapsed_time(e1) / reps
    return ms, {k: round(v["ms"] / reps, 4) for k, v in pr.items()}


def err_sample(got, A, B, rows, cols, cplx):
    if cplx:
        T = oracle.exact_zproduct(A[rows], B[:, cols])
    else:
        T = oracle.exact_product(A[rows], B[:, cols])
    absab = np.abs(A[rows]) @ np.abs(B[:, cols])
    return float(np.max(np.abs(got[np.ix_(rows, cols)] - T) / absab))


def c2(out):
    batch, n = 30, 512
    A_h, B_h = bench.make_inputs(batch, n, 3.0, 1000)
    dv = torch.device("cuda", 0)
    A = bench.to_dev_batched(torch, A_h, dv)
    B = bench.to_dev_batched(torch, B_h, dv)
    C = torch.zeros((batch, n, n), dtype=torch.complex128, device=dv).transpose(1, 2)
    flops = bench.fp64_equiv_flops(batch, n)
    rows = np.r_[0:n:37]
    cols = np.r_[0:n:41]
    A0, B0 = np.asfortranarray(A_h[0]), np.asfortranarray(B_h[0])
    res = {}
    for s in (4, 5, 6, 7, 8):
        ms, ph = timed(lambda: oz.zgemm_strided_batched("N", "N", 1.0, A, B, 0.0, C, s))
        ops = bench.int8_ops(batch, n, s, "4m")
        res[f"ozaki1_s{s}"] = dict(tf=round(flops / ms / 1e9, 2), ms=round(ms, 4), phases=ph,
                                   gemm_tops=round(ops / ph["k2_gemm"] / 1e9, 1),
                                   err=err_sample(C[0].cpu().numpy(), A0, B0, rows, cols, True))
    for N in (10, 12, 14, 16, 18):
        ms, ph = timed(lambda: oz.ozaki2_zgemm_strided_batched("N", "N", 1.0, A, B, 0.0, C, N))
        ops = 2 * N * n * (2 * n) * (2 * n) * batch        # one INT8 GEMM per modulus of m x 2k x 2n
        res[f"ozaki2_N{N}"] = dict(tf=round(flops / ms / 1e9, 2), ms=round(ms, 4), phases=ph,
                                   gemm_tops=round(ops / ph["k2_gemm"] / 1e9, 1),
                                   err=err_sample(C[0].cpu().numpy(), A0, B0, rows, cols, True))
    out["c2x30_zgemm512_kkr3"] = res


def c3(out):
    n = 8192
    g = torch.Generator(device="cuda").manual_seed(5)
    A = (torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    B = (torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    C = torch.zeros((n, n), dtype=torch.float64, device="cuda").t()
    flops = 2 * n ** 3
    rows = np.r_[0:n:997]
    cols = np.r_[0:n:1009]
    Ah = A.cpu().numpy()
    Bh = B.cpu().numpy()
    res = {}
    for s in (4, 6, 7, 8):
        ms, ph = timed(lambda: oz.dgemm("N", "N", 1.0, A, B, 0.0, C, s), reps=3, warm=2)
        ops = 2 * (s * (s + 1) // 2) * n ** 3
        res[f"ozaki1_s{s}"] = dict(tf=round(flops / ms / 1e9, 2), ms=round(ms, 3), phases=ph,
                                   gemm_tops=round(ops / ph["k2_gemm"] / 1e9, 1),
                                   err=err_sample(C.cpu().numpy(), Ah, Bh, rows, cols, False))
    for N in (10, 12, 14, 16, 18):
        ms, ph = timed(lambda: oz.ozaki2_dgemm("N", "N", 1.0, A, B, 0.0, C, N), reps=3, warm=2)
        ops = 2 * N * n ** 3
        res[f"ozaki2_N{N}"] = dict(tf=round(flops / ms / 1e9, 2), ms=round(ms, 3), phases=ph,
                                   gemm_tops=round(ops / ph["k2_gemm"] / 1e9, 1),
                                   err=err_sample(C.cpu().numpy(), Ah, Bh, rows, cols, False))
    out["c3_dgemm8192_uniform"] = res


if __name__ == "__main__":
    out = {}
    c2(out)
    c3(out)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/method_compare.json", "w") as fh:
        json.dump(out, fh, indent=1)
    for wl, res in out.items():
        print(wl)
        for k, v in res.items():
            print(f"  {k:12s} {v['tf']:8.2f} TF-eq  {v['ms']:9.4f} ms  gemm {v['gemm_tops']:7.1f} TOPS  "
                  f"err {v['err']:.2e}  {v['phases']}")
