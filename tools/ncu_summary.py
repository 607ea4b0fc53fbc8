"""Summarise ncu captures into profiles/ (tracked): launch shares + key metrics.

usage: python tools/ncu_summary.py TAG   (reads gpurun_out/*_TAG*, writes profiles/TAG_*)
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x",
    "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
]


def ncu_raw(rep):
    if rep.endswith(".csv"):   # raw page exported on the GPU box (the .ncu-rep stays there)
        text = open(rep).read()
    else:
        text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                              text=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
        for k in KEYS:
            for i, h in enumerate(hdr):
                if h == k:
                    d[k] = f"{vals[i]} {units[i]}".strip()
        out.append(d)
    return out


def launches(path):
    """Per-kernel total device time from the gpu__time_duration launch list."""
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    iu = hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[iu], 1.0)
        name = r[ik].split("(")[0]
        tot[name] += v * scale
        cnt[name] += 1
    return tot, cnt


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    md = [f"# ncu summary `{tag}`", ""]
    lpath = os.path.join(OUT, f"launches_{tag}.csv")
    if os.path.exists(lpath):
        tot, cnt = launches(lpath)
        s = sum(tot.values())
        md += ["## Launch list (ncu `gpu__time_duration.sum`, --clock-control none, cold/serialised)", "",
               "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            md.append(f"| `{k}` | {cnt[k]} | {v:.1f} | {v / s:.3f} |")
        md.append("")
        with open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as fh:
            fh.write(open(lpath).read())
    summary = {}
    for kind in ("gemm", "slice", "split"):
        rep = os.path.join(OUT, f"prof_{kind}_{tag}.ncu-rep")
        if not os.path.exists(rep):
            rep = os.path.join(OUT, f"prof_{kind}_{tag}_raw.csv")
        if not os.path.exists(rep):
            continue
        rows = ncu_raw(rep)
        summary[kind] = rows
        md += [f"## `ncu --set full` capture: {kind}", ""]
        for d in rows:
            md.append(f"### {d['kernel'][:110]}")
            md.append("")
            md.append("| metric | value |")
            md.append("|---|---|")
            for k in KEYS:
                if k in d:
                    md.append(f"| `{k}` | {d[k]} |")
            md.append("")
    with open(os.path.join(PROF, f"{tag}_ncu.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    # dominant-kernel DRAM traffic per launch, read by bench.py (roofline.traffic)
    for d in summary.get("gemm", [])[:1]:
        def num(x):
            v, u = x.split()[0], x.split()[-1]
            return float(v) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(u, 1.0)
        tr = num(d["dram__bytes_read.sum"]) + num(d["dram__bytes_write.sum"])
        with open(os.path.join(PROF, "gemm_traffic.json"), "w") as fh:
            json.dump({"tag": tag, "kernel": d["kernel"], "traffic_bytes_per_launch": tr,
                       "source": f"profiles/{tag}_summary.md (ncu --set full, 1 launch)",
                       "workload": "bench.py default (C2 x30, 4M, s=7)"}, fh, indent=1)
    with open(os.path.join(PROF, f"{tag}_summary.md"), "w") as fh:
        fh.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main(sys.argv[1])
