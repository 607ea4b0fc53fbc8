"""Accuracy / speed studies of SURVEY §8(d) beyond the bench headline (round 2):

* configs[1] families: ZGEMM 512^3 with KKR(gamma=1), KKR(gamma=3), Phi(2); op(B) = B ('N') and
  B^H ('C'); 4M vs 3M; s = 4..8.  Timing: one strided-batched call over 30 blocks; error: entry 0,
  32 x 32 sampled entries vs the oracle's exact product (both c-13 definitions).
* configs[4] on one GPU: DGEMM 32768 x 32768 x 4096 with Phi(4) ("large dynamic range") and a
  cancellation variant: 32 columns c_j of B are replaced by b - t (a_r . b / a_r . a_r) a_r^T for a
  row r_j of A, with 1 - t = 10^-x, x in [4, 12], so (AB)_{r_j c_j} is 10^-x of |A||B|; the kappa =
  (|A||B|)_ij / |(AB)_ij| distribution of the sample and the error per s = 4..9 show which s reaches
  FP64-level error.

Writes profiles/r2_accuracy.json and prints a markdown table.  The oracle (oracle/) supplies the
exact products -- this is a measurement tool, like bench.py's cpu_baseline leg.
usage: python tools/accuracy_configs.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2603_29975_b200 as oz  # noqa: E402


def errs(got, truth, absab):
    nz = truth != 0
    return {"rel": float(np.max(np.abs(got - truth)[nz] / np.abs(truth[nz]))),
            "comp": float(np.max(np.abs(got - truth) / absab))}


def c2_study(st):
    out = {}
    n, batch = 512, 30
    fams = {"kkr_g1": lambda sd: synth.kkr(n, n, seed=sd, gamma=1.0),
            "kkr_g3": lambda sd: synth.kkr(n, n, seed=sd, gamma=3.0),
            "phi2": lambda sd: synth.spread(n, n, sd, phi=2.0, complex_=True)}
    rows, cols = bench.c3_sample_idx(n)
    for fam, gen in fams.items():
        A_h = np.stack([gen(2000 + 2 * i) for i in range(batch)])
        B_h = np.stack([gen(2001 + 2 * i) for i in range(batch)])
        A = bench.to_dev_batched(torch, A_h, "cuda")
        for tb in ("N", "C"):
            Bop0 = B_h[0]                                  # op(B) is the same matrix for 'N' and 'C'
            Bstore = B_h if tb == "N" else np.conj(np.transpose(B_h, (0, 2, 1)))   # stored B: op(B) = B^H
            B = bench.to_dev_batched(torch, np.ascontiguousarray(Bstore), "cuda")
            truth = oracle.exact_zproduct(A_h[0][rows], Bop0[:, cols])
            absab = np.abs(A_h[0][rows]) @ np.abs(Bop0[:, cols])
            C = torch.zeros((batch, n, n), dtype=torch.complex128, device="cuda").transpose(1, 2)
            for method, fn in (("4m", oz.zgemm_strided_batched), ("3m", oz.zgemm3m_strided_batched)):
                for s in (4, 5, 6, 7, 8):
                    call = lambda: fn("N", tb, 1.0, A, B, 0.0, C, s)   # noqa: E731
                    for _ in range(2):
                        call()
                    ms, clk = bench.timed(torch, st, call, 5, 0)
                    got = C[0].cpu().numpy()[np.ix_(rows, cols)]
                    out[f"{fam}/{tb}/{method}/s{s}"] = {
                        "tflops": round(8.0 * n ** 3 * batch / (ms * 1e-3) / 1e12, 2), "sm_mhz": clk.get("sm_mhz"),
                        **errs(got, truth, absab)}
            del B, C
        del A
    return out


def c5_study(st):
    m = n = 32768
    k = 4096
    out = {}
    t0 = time.time()
    A_h = np.asfortranarray(synth.spread(m, k, 1, phi=4.0))
    B_h = np.asfortranarray(synth.spread(k, n, 2, phi=4.0))
    g = np.random.default_rng(7)
    rows = np.sort(g.choice(m, 32, replace=False))
    cols = np.sort(g.choice(n, 32, replace=False))
    variants = {"phi4": B_h}
    Bc = B_h.copy(order="F")
    xs = np.linspace(4, 12, 32)
    for r, c, x in zip(rows, cols, xs):          # cancellation on the sample's diagonal pairs
        a = A_h[r, :]
        b = Bc[:, c]
        t = 1.0 - 10.0 ** (-x)
        Bc[:, c] = b - t * (a @ b) / (a @ a) * a
    variants["cancel"] = Bc
    out["gen_seconds"] = round(time.time() - t0, 1)
    A = oz.colmajor(torch.from_numpy(A_h).cuda())
    C = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
    rr, cc = torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda()
    for name, Bv in variants.items():
        B = oz.colmajor(torch.from_numpy(Bv).cuda())
        truth = oracle.exact_product(np.ascontiguousarray(A_h[rows]), np.asfortranarray(Bv[:, cols]))
        absab = np.abs(A_h[rows]) @ np.abs(Bv[:, cols])
        kappa = absab / np.maximum(np.abs(truth), 1e-300)
        out[f"{name}/kappa_percentiles"] = {q: float(np.percentile(kappa, q)) for q in (50, 90, 99, 100)}
        out[f"{name}/kappa_diag"] = [float(x) for x in np.diag(kappa)]
        nat = oracle.fp64_product(np.ascontiguousarray(A_h[rows]), np.asfortranarray(Bv[:, cols]))
        out[f"{name}/native_fp64"] = errs(nat, truth, absab)
        for s in (4, 5, 6, 7, 8, 9):
            call = lambda: oz.dgemm("N", "N", 1.0, A, B, 0.0, C, s)   # noqa: E731
            call()
            ms, clk = bench.timed(torch, st, call, 2, 0)
            got = C[rr][:, cc].cpu().numpy()
            e = errs(got, truth, absab)
            dg = np.abs(np.diag(got) - np.diag(truth)) / np.maximum(np.abs(np.diag(truth)), 1e-300)
            out[f"{name}/s{s}"] = {"tflops": round(2.0 * m * n * k / (ms * 1e-3) / 1e12, 2),
                                   "sm_mhz": clk.get("sm_mhz"), **e,
                                   "rel_on_cancelled_entries_max": float(np.max(dg))}
            want = oracle.dgemm("N", "N", 1.0, np.ascontiguousarray(A_h[rows[:8]]),
                                np.asfortranarray(Bv[:, cols[:8]]), 0.0, None, s)
            out[f"{name}/s{s}"]["bitexact_8x8"] = bool((got[:8, :8] == want).all())
        del B
    return out


def main():
    st = torch.cuda.current_stream()
    res = {"c2": c2_study(st), "c5_1gpu": c5_study(st)}
    with open(os.path.join(ROOT, "profiles", "r2_accuracy.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    print("| configs[1] family / op(B) / method / s | TF/s | rel | comp |")
    print("|---|---|---|---|")
    for k_, v in res["c2"].items():
        print(f"| {k_} | {v['tflops']} | {v['rel']:.2e} | {v['comp']:.2e} |")
    print()
    for k_, v in res["c5_1gpu"].items():
        print(k_, v if not isinstance(v, list) else [f"{x:.1e}" for x in v[:6]])


if __name__ == "__main__":
    main()
