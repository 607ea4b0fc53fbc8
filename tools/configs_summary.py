"""gpurun_out/cfg_*.json (tools/configs_round.sh) -> profiles/TAG_configs.md/json."""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(tag):
    rows = []
    for f in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "cfg_*.json"))):
        try:
            d = json.load(open(f))
        except Exception:
            continue
        r = d.get("roofline", {})
        ph = d.get("phase_ms_per_step", {})
        rows.append({"file": os.path.basename(f), "workload": d.get("config", {}).get("workload", ""),
                     "s": d.get("config", {}).get("slices"), "value": d.get("value"),
                     "ms_per_step": d.get("ms_per_step"), "gemm_ms": r.get("kernel_ms_per_launch"),
                     "gemm_frac": r.get("frac"),
                     "split_ms": round(ph.get("k1_slice", 0.0) + ph.get("k1_exponent", 0.0), 5),
                     "clocks": d.get("clocks", {})})
    with open(os.path.join(ROOT, "profiles", f"{tag}_configs.json"), "w") as fh:
        json.dump(rows, fh, indent=1)
    with open(os.path.join(ROOT, "profiles", f"{tag}_configs.md"), "w") as fh:
        fh.write(f"# Secondary BASELINE configs on 1 B200 (round 1, tag {tag})\n\n")
        fh.write("Command: `bash tools/configs_round.sh` (bench.py --workload ...), CUDA-event timing, 3+ "
                 "warm-ups.\nFP64-eq = 2mnk (DGEMM) / 8mnk (ZGEMM) per second; GEMM frac = INT8 ops of the "
                 "slice GEMM / its event-timed duration / (measured bf16 burst x 2 = 3264.8 TOPS) -- frac > 1 "
                 "means the bf16-derived INT8 peak understates the real INT8 rate (nominal 4.5 POPS).\n\n")
        fh.write("| workload | s | FP64-eq TF/s | ms/step | GEMM ms | GEMM frac | split ms | SM MHz |\n")
        fh.write("|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            fh.write(f"| {r['workload']} | {r['s']} | {r['value']} | {r['ms_per_step']} | {r['gemm_ms']} | "
                     f"{r['gemm_frac']} | {r['split_ms']} | {r['clocks'].get('sm_mhz')} |\n")
    print(f"wrote profiles/{tag}_configs.md ({len(rows)} rows)")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "rX")
