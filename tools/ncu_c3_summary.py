"""Summarise tools/ncu_bench.sh outputs (gpurun_out/TAG_*) into profiles/ (tracked):
profiles/ncu_c3.json (per-s tensor-pipe %, DRAM bytes and duration of the C3 slice GEMM and of
the split kernels; read by bench.py into the roofline record) and profiles/TAG_ncu_c3.md.

usage: python tools/ncu_c3_summary.py TAG
"""
import csv
import io
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def rows(path):
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    return list(csv.DictReader(io.StringIO("".join(lines))))


def per_kernel(path):
    d = defaultdict(dict)
    for r in rows(path):
        d[(r["ID"], r["Kernel Name"])][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return d


def main(tag):
    n = 8192
    res = {"source": f"ncu --metrics ... --clock-control none -k regex:k_gemm_lv2 (tools/ncu_bench.sh, tag {tag}); "
                     "one C3 DGEMM 8192^3 call per s after 2 warm-up calls",
           "workload": "c3", "per_s": {}}
    md = [f"# C3 (DGEMM 8192^3, uniform) ncu summary, tag {tag}", "",
          "Per-launch values of one call (ncu replays; times are cold-cache and serialised, so only shares and "
          "ratios are comparable with bench.py).  Algorithmic GEMM bytes = slices of both operands "
          "(s x 2 x n^2) + C (8 n^2); split bytes = 2 x 8 n^2 read + 2 s n^2 written.", "",
          "| s | GEMM ms | tensor pipe active % | SM clock MHz | GEMM DRAM bytes (read+write) | x algorithmic | "
          "split kernels ms | split DRAM bytes | x algorithmic |", "|---|---|---|---|---|---|---|---|---|"]
    for s in range(3, 10):
        p = os.path.join(OUT, f"{tag}_c3_s{s}.csv")
        if not os.path.exists(p):
            continue
        (k, m), = per_kernel(p).items()
        dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        alg = s * 2 * n * n + 8 * n * n
        rec = {"tensor_pipe_pct": m["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"],
               "dram_bytes": int(dram), "algorithmic_bytes": alg, "gemm_ms": m["gpu__time_duration.sum"] / 1e6,
               "sm_hz": m["sm__cycles_elapsed.avg.per_second"], "kernel": k[1]}
        ps = os.path.join(OUT, f"{tag}_split_s{s}.csv")          # tools/ncu_split_cluster.sh
        if not os.path.exists(ps) or not per_kernel(ps):
            ps = os.path.join(OUT, f"{tag}_c3_split_s{s}.csv")    # tools/ncu_bench.sh
        ks = per_kernel(ps) if os.path.exists(ps) else {}
        if ks:
            rec["split_ms"] = sum(v["gpu__time_duration.sum"] for v in ks.values()) / 1e6
            rec["split_dram_bytes"] = int(sum(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in ks.values()))
            rec["split_algorithmic_bytes"] = 16 * n * n + 2 * s * n * n
            rec["split_kernels"] = sorted(kk[1] for kk in ks)
        res["per_s"][str(s)] = rec
        md.append(f"| {s} | {rec['gemm_ms']:.3f} | {rec['tensor_pipe_pct']:.1f} | {rec['sm_hz'] / 1e6:.0f} | "
                  f"{dram / 1e9:.2f} GB | {dram / alg:.2f} | {rec.get('split_ms', 0):.3f} | "
                  f"{rec.get('split_dram_bytes', 0) / 1e9:.2f} GB | "
                  f"{rec.get('split_dram_bytes', 0) / rec.get('split_algorithmic_bytes', 1):.2f} |")
    lp = os.path.join(OUT, f"{tag}_launches.csv")
    if os.path.exists(lp):
        tot = defaultdict(float)
        cnt = defaultdict(int)
        for r in rows(lp):
            if r["Metric Name"] == "gpu__time_duration.sum":
                name = r["Kernel Name"].split("(")[0]
                tot[name] += float(r["Metric Value"].replace(",", ""))
                cnt[name] += 1
        all_ns = sum(tot.values())
        md += ["", f"Launch list of `python bench.py --steps 2 --warmup 3 --no-extras` ({tag}_launches.csv):", "",
               "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for name, v in sorted(tot.items(), key=lambda x: -x[1]):
            md.append(f"| `{name}` | {cnt[name]} | {v / 1e6:.3f} | {v / all_ns:.3f} |")
        res["launch_shares"] = {name: round(v / all_ns, 4) for name, v in tot.items()}
    fp = os.path.join(OUT, f"{tag}_c3_s7_full_raw.csv")
    if os.path.exists(fp):
        with open(fp) as fh:
            r = list(csv.reader(fh))
        hdr, unit, val = r[0], r[1], r[2]
        keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
                "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "sm__cycles_elapsed.avg.per_second", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
        full = {k: f"{val[hdr.index(k)]} {unit[hdr.index(k)]}".strip() for k in keys if k in hdr}
        res["full_set_s7"] = full
        md += ["", "`ncu --set full` of the s=7 GEMM launch:", ""] + [f"- `{k}`: {v}" for k, v in full.items()]
    sp = os.path.join(OUT, f"{tag}_split_full_raw.csv")
    if os.path.exists(sp):   # tools/ncu_split_cluster.sh: --set full of the s=7 split launch
        with open(sp) as fh:
            r = list(csv.reader(fh))
        hdr, unit, val = r[0], r[1], r[2]
        keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__cluster_dim_x",
                "launch__occupancy_cluster_pct", "launch__registers_per_thread",
                "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second"]
        full = {k: f"{val[hdr.index(k)]} {unit[hdr.index(k)]}".strip() for k in keys if k in hdr}
        if "Kernel Name" in hdr:
            full["kernel"] = val[hdr.index("Kernel Name")]
        res["split_full_set_s7"] = full
        md += ["", "`ncu --set full` of the s=7 split launch (`k_split_cluster`, tools/ncu_split_cluster.sh):", ""] + \
              [f"- `{k}`: {v}" for k, v in full.items()]
    with open(os.path.join(PROF, "ncu_c3.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    with open(os.path.join(PROF, f"{tag}_ncu_c3.md"), "w") as fh:
        fh.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r2")
