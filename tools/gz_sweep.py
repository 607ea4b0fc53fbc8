"""NEXT-3 driver: the Fig. 1a analog -- max percent error of
g(z) = Tr (zI - H)^-1 over a 30-point semicircle contour for every emulation mode vs
native FP64, integrated density, and the wall time of the blocked-LU inversions with
the trailing updates on native cuBLAS ZGEMM vs the Ozaki GEMMs.  Writes
gpurun_out/gz_sweep.json."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2603_29975_b200 import workload as W


def gapped_spectrum(n, seed, eb, ef, gap=0.1):
    """U[-1, 1) eigenvalues kept >= gap away from the contour endpoints (SPEC workload)."""
    g = np.random.default_rng(seed)
    ev = []
    while len(ev) < n:
        x = g.uniform(-1.0, 1.0)
        if abs(x - eb) >= gap and abs(x - ef) >= gap:
            ev.append(x)
    return np.sort(ev)


def accuracy(n=512, nodes=30, nb=64):
    eb, ef = -0.8, 0.4
    H, ev = synth.hamiltonian(n, seed=11, eigs=gapped_spectrum(n, 11, eb, ef))
    count = int(((ev > eb) & (ev < ef)).sum())
    modes = [W.gemm_native()] + [W.gemm_ozaki1(s) for s in (3, 4, 5, 6, 7, 8)] + \
            [W.gemm_ozaki2(m) for m in (8, 10, 12, 14, 16, 18)]
    rep = W.green_function_sweep(H, eb, ef, nodes, modes, nb=nb)
    out = {"n": n, "nodes": nodes, "nb": nb, "window": [eb, ef], "eigenvalues_in_window": count, "modes": {}}
    for lab, r in rep["modes"].items():
        out["modes"][lab] = {"max_percent_error": r["max_percent_error"], "argmax_node": r["argmax_node"],
                             "N_est": r["N_est"], "N_est_error": abs(r["N_est"] - count),
                             "N_est_vs_native": abs(r["N_est"] - rep["modes"]["native"]["N_est"]),
                             "residual_max": r["residual_max"]}
    return out


def timing(n=4096, nb=512, reps=2, emulated_trsm=False):
    H, ev = synth.hamiltonian(n, seed=12)
    Hd = torch.from_numpy(np.ascontiguousarray(H)).cuda()
    I = torch.eye(n, dtype=torch.complex128, device="cuda")
    M = complex(-0.2 + 0.05j) * I - Hd
    res = {}
    for base in (W.gemm_native(), W.gemm_ozaki1(4), W.gemm_ozaki1(7), W.gemm_ozaki2(12), W.gemm_ozaki2(16)):
        W.blocked_lu_invert(M, nb, base, emulated_trsm=emulated_trsm)          # warm-up
        gm = W.timed_gemm(base)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):   # the inversion alone: the residual check runs after the timed loop
            Minv, _ = W.blocked_lu_invert(M, nb, gm, emulated_trsm=emulated_trsm, check=False)
        torch.cuda.synchronize()
        secs = (time.perf_counter() - t0) / reps
        r = W.residual(M, Minv)
        gms = gm.total_ms() / reps
        # LU trailing updates: sum over panels of 8 (n - j1)^2 nb real flops (complex MACs x 8);
        # emulated TRSM adds the two block sweeps' updates, each sum_i 8 (rows_left) nb n
        flops = sum(8.0 * (n - j1) ** 2 * nb for j1 in range(nb, n, nb))
        if emulated_trsm:
            flops += 2 * sum(8.0 * (n - j1) * nb * n for j1 in range(nb, n, nb))
        res[gm.label] = {"seconds_per_inversion": secs, "trailing_update_ms": gms,
                         "trailing_update_tflops": flops / (gms * 1e-3) / 1e12, "residual_max": r}
    nat = res.get("native", {}).get("seconds_per_inversion")
    for lab, r in res.items():
        if nat:
            r["speedup_vs_native"] = nat / r["seconds_per_inversion"]
    return {"n": n, "nb": nb, "emulated_trsm": emulated_trsm, "timed": "inversion only (residual after)",
            "modes": res}


if __name__ == "__main__":
    out = {"accuracy": accuracy(), "timing": timing(), "timing_emulated_trsm": timing(emulated_trsm=True)}
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/gz_sweep.json", "w") as fh:
        json.dump(out, fh, indent=1)
    a = out["accuracy"]
    print(f"G(z) sweep: n={a['n']} nodes={a['nodes']} window={a['window']} eigenvalues inside={a['eigenvalues_in_window']}")
    for lab, r in a["modes"].items():
        print(f"  {lab:28s} max % err {r['max_percent_error']:.3e} (node {r['argmax_node']:2d})  "
              f"N_est err {r['N_est_error']:.2e} (vs native {r['N_est_vs_native']:.1e})  resid {r['residual_max']:.1e}")
    for key in ("timing", "timing_emulated_trsm"):
      t = out[key]
      print(f"inversion n={t['n']} nb={t['nb']} emulated_trsm={t['emulated_trsm']}:")
      for lab, r in t["modes"].items():
        print(f"  {lab:28s} {r['seconds_per_inversion'] * 1e3:9.2f} ms total, emulated-GEMM updates "
              f"{r['trailing_update_ms']:8.2f} ms ({r['trailing_update_tflops']:6.1f} TF/s FP64-eq)  "
              f"resid {r['residual_max']:.1e}  x{r.get('speedup_vs_native', 0):.2f} vs native")
