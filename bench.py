#!/usr/bin/env python
"""bench.py -- FP64-equivalent TFLOP/s of the INT8 Ozaki-I DGEMM/ZGEMM path on B200.

Metric (BASELINE.json): "FP64-equiv TFLOP/s (ZGEMM/DGEMM) vs slice count; INT8
pipe util; max rel err".  Default workload = BASELINE configs[2], the config the
metric is quoted on: square DGEMM 8192 x 8192 x 8192 on one B200, uniform [-1,1)
inputs (synth.uniform), headline at s = 7 (the paper's 55-bit mode),
with the sweep s = 3..9 for the uniform and the spread Phi(1) families (FP64-eq
TFLOP/s, GEMM INT8 TOPS against the roofline with that pass's clocks, max relative
error vs the true FP64 product on 1024 sampled entries, both SURVEY c-13 definitions).
One step = one ozaki_dgemm call (split + slice GEMM with the fused FP64 epilogue).
Multi-GPU (--gpus N): the GEMM is sharded by column slabs of C with the all-gather of
C overlapped with the GEMM (paper_2603_29975_b200.dist) -- strong scaling.

Other workloads (--workload): c2x30 (30 x ZGEMM 512^3 KKR, 4M, the round-1 headline),
c1, c2, c4, c5 (BASELINE configs[0], [1], [3], [4]).  `--impl reference` times the
CPU oracle (oracle/) on a bounded sample of the same workload on the host cores (the
reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

BURST_FALLBACK_BF16 = 1590.0    # B200_PROFILING.md fallback (TFLOP/s) if MEASURED_PEAKS.json absent
INT8_OVER_BF16 = 4.5 / 2.25     # nominal dense ratio (B200_PROFILING.md / datasheet)
MAC_PER_CLK_SM = 8192           # measured kind::i8 M128 N128 K32 rate per SM
SMS = 148
METRIC = "FP64-equiv TFLOP/s (ZGEMM/DGEMM) vs slice count; INT8 pipe util; max rel err"

def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--slices", type=int, default=7)
    ap.add_argument("--method", default="4m", choices=["4m", "3m"])
    ap.add_argument("--batch", type=int, default=30)
    ap.add_argument("--n", type=int, default=None, help="matrix size (default: the workload's)")
    ap.add_argument("--gamma", type=float, default=3.0)
    ap.add_argument("--no-extras", action="store_true", help="skip sweep / e2e / extra workloads / cpu baseline")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-overlap", action="store_true",
                    help="headline without cross-call overlap (ozaki_set_overlap off)")
    ap.add_argument("--workload", default="c3", choices=["c3", "c2x30", "c1", "c2", "c4", "c5"],
                    help="c3 (default, the headline: BASELINE configs[2]) or another config")
    return ap.parse_args()

# The other BASELINE.json configs (parity cases / secondary measurements).
CONFIGS = {
    "c1": dict(kind="d", m=64, n=64, k=64, batch=1, fam="uniform", shard="replica",
               desc="configs[0]: DGEMM 64^3, uniform"),
    "c2": dict(kind="z", m=512, n=512, k=512, batch=1, fam="kkr", gamma=3.0, shard="replica",
               desc="configs[1] single block: ZGEMM 512^3 KKR (gamma=3)"),
    "c3": dict(kind="d", m=8192, n=8192, k=8192, batch=1, fam="uniform", shard="replica",
               desc="configs[2]: DGEMM 8192^3, uniform"),
    "c4": dict(kind="z", m=1024, n=1024, k=1024, batch=256, fam="kkr", gamma=1.0, shard="batch",
               desc="configs[3]: 256 x ZGEMM 1024^3 KKR (gamma=1), batch-sharded across ranks"),
    "c5": dict(kind="d", m=32768, n=32768, k=4096, batch=1, fam="spread", phi=4.0, shard="columns",
               desc="configs[4]: DGEMM 32768x32768x4096 spread(phi=4), column slabs + all-gather of C"),
}

def _rank_device(torch, local):
    """One process per GPU.  OZAKI_DIST_BACKEND=gloo lets several ranks share one device (a test
    hook for the multi-rank path on a 1-GPU box); with NCCL every rank owns its own GPU."""
    idx = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(idx)
    return torch.device("cuda", idx)

def _init_dist(dist, device):
    backend = os.environ.get("OZAKI_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=device)
    else:
        dist.init_process_group(backend)

def run_config(args):
    """Secondary workloads: one timed step = the whole GEMM (or this rank's shard of it)."""
    import torch
    import torch.distributed as dist
    import paper_2603_29975_b200 as oz
    from paper_2603_29975_b200 import dist as zd

    cfg = CONFIGS[args.workload]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    device = _rank_device(torch, local)
    if world > 1:
        _init_dist(dist, device)
    s = args.slices
    m, n, k, kind = cfg["m"], cfg["n"], cfg["k"], cfg["kind"]
    batch = args.batch if (cfg["shard"] == "batch" and args.batch != 30) else cfg["batch"]
    cplx = kind == "z"
    kw = {x: cfg[x] for x in ("gamma", "phi") if x in cfg}

    def gen(r, c, seed):
        return synth.make(cfg["fam"], r, c, seed, complex_=cplx, **kw)

    def colmajor_dev(X):
        return oz.colmajor(torch.from_numpy(np.asfortranarray(X)).to(device))

    if cfg["shard"] == "batch":
        b0, b1 = zd.batch_shard(batch, rank, world)
        nb = b1 - b0
        distinct = 8   # distinct blocks, tiled over the batch (identical GEMM work per entry)
        As = [colmajor_dev(gen(m, k, 10 + i)) for i in range(distinct)]
        Bs = [colmajor_dev(gen(k, n, 50 + i)) for i in range(distinct)]
        A = torch.stack([As[(b0 + i) % distinct] for i in range(nb)]).transpose(1, 2).contiguous().transpose(1, 2)
        B = torch.stack([Bs[(b0 + i) % distinct] for i in range(nb)]).transpose(1, 2).contiguous().transpose(1, 2)
        C = torch.zeros((nb, n, m), dtype=A.dtype, device=device).transpose(1, 2)
        fn = oz.zgemm_strided_batched if cplx else oz.dgemm_strided_batched
        step = lambda: fn("N", "N", 1.0, A, B, 0.0, C, s)   # noqa: E731
        units = batch
    else:
        A = colmajor_dev(gen(m, k, 1))
        B = colmajor_dev(gen(k, n, 2))
        C = torch.zeros((n, m), dtype=A.dtype, device=device).t()
        fn = oz.zgemm if cplx else oz.dgemm
        if cfg["shard"] == "columns":
            gemm = lambda a, b, c: fn("N", "N", 1.0, a, b, 0.0, c, s)   # noqa: E731
            step = lambda: zd.sharded_gemm_columns(gemm, A, B, C, rank, world)   # noqa: E731
            units = 1
        else:
            step = lambda: fn("N", "N", 1.0, A, B, 0.0, C, s)   # noqa: E731
            units = world   # replicas
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    st0 = oz.get_stats()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):      # timed pass 1 (headline): no per-launch events
        step()
    e1.record()
    torch.cuda.synchronize()
    clocks.stop()
    st1 = oz.get_stats()
    ms = zd.max_over_ranks(e0.elapsed_time(e1), device) / args.steps
    if world > 1:
        dist.barrier()
    oz.profile_enable(True)          # timed pass 2: per-launch events -> kernel times
    oz.profile_read()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    prof = oz.profile_read()
    oz.profile_enable(False)
    flop_unit = (8 if cplx else 2) * m * n * k
    value = flop_unit * units / (ms * 1e-3) / 1e12
    gemm = prof["k2_gemm"]
    gemm_ms = gemm["ms"] / max(1, gemm["launches"])
    pairs = s * (s + 1) // 2
    per_launch_units = (nb if cfg["shard"] == "batch" else 1)
    if cfg["shard"] == "columns":
        # per GEMM launch: this rank's owned columns are computed in one launch per non-empty
        # chunk block (dist.sharded_gemm_columns, 4 chunks) -- average columns per launch / n
        own = [b - a for a, b in zd.column_blocks(n, rank, world, 4)[1] if b > a] if world > 1 else [n]
        frac_cols = (sum(own) / max(1, len(own))) / n
    else:
        frac_cols = 1.0
    alg_ops = 2 * pairs * (4 if cplx else 1) * m * n * k * per_launch_units * frac_cols
    bf16_burst, _, peak_src = peaks()
    peak_int8 = bf16_burst * INT8_OVER_BF16
    achieved = alg_ops / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
    out = {
        "metric": "FP64-equiv TFLOP/s (ZGEMM/DGEMM) vs slice count; INT8 pipe util; max rel err",
        "value": round(value, 3), "unit": f"TFLOP/s (FP64-equivalent, {'8' if cplx else '2'}mnk)",
        "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "strong" if cfg["shard"] in ("batch", "columns") else "weak",
        "vs_baseline": None, "dtype": "f64 in/out; int8 tensor-core products; f64 epilogue",
        "data": f"synthetic (synth.{cfg['fam']}, seeded)",
        "config": {"workload": cfg["desc"], "slices": s, "m": m, "n": n, "k": k, "batch": batch,
                   "parallelism": f"{cfg['shard']} x{world}"},
        "roofline": {"bound": "tensor", "kernel": "slice GEMM (K2+K3)",
                     "achieved": round(achieved, 2) if achieved else None, "peak": round(peak_int8, 1),
                     "unit": "TOPS (INT8 dense)", "frac": round(achieved / peak_int8, 4) if achieved else None,
                     "peak_source": f"{peak_src} bf16 burst x 2", "kernel_ms_per_launch": round(gemm_ms, 5),
                     "traffic": None},
        "phase_ms_per_step": {k2: round(v["ms"] / args.steps, 5) for k2, v in prof.items()},
        "gpu_launches": int(st1["kernel_launches"] - st0["kernel_launches"]),
        "clocks": clocks.summary(),
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()

def traffic_from_profile(s, method, n, batch, gamma):
    """DRAM bytes/launch of the GEMM from the committed ncu capture (profiles/gemm_traffic.json),
    only for the default workload it was captured on; else None."""
    if (s, method, n, batch, gamma) != (7, "4m", 512, 30, 3.0):
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "gemm_traffic.json")) as fh:
            return float(json.load(fh)["traffic_bytes_per_launch"])
    except Exception:  # noqa: BLE001
        return None

def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    except Exception:  # noqa: BLE001
        return BURST_FALLBACK_BF16, 1400.0, "fallback"

# ---------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.005):
        self.index = index
        self.period = period_s
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001
            self.ok = False

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0,
                    "source": "nvml unavailable" if not self.ok else "no samples"}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and v != "gpu_idle"]
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples), "source": "nvml 5 ms"}

# ------------------------------------------------------------ workload
def make_inputs(batch, n, gamma, seed0):
    """Batch of KKR-like complex blocks (column-major per entry), numpy."""
    A = np.empty((batch, n, n), dtype=np.complex128, order="C")
    B = np.empty((batch, n, n), dtype=np.complex128, order="C")
    for i in range(batch):
        A[i] = synth.kkr(n, n, seed=seed0 + 2 * i, gamma=gamma)
        B[i] = synth.kkr(n, n, seed=seed0 + 2 * i + 1, gamma=gamma)
    return A, B

def to_dev_batched(torch, X, device):
    # (batch, n, n) numpy with Fortran entries -> column-major per entry on device
    t = torch.from_numpy(np.ascontiguousarray(np.transpose(X, (0, 2, 1))))  # row-major of X^T
    return t.to(device).transpose(1, 2)

def fp64_equiv_flops(batch, n, cplx=True):
    return batch * (8 if cplx else 2) * n ** 3

def int8_ops(batch, n, s, method):
    mult = 4 if method == "4m" else 3
    return 2 * mult * (s * (s + 1) // 2) * n ** 3 * batch

# ------------------------------------------------------------------ main
def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2603_29975_b200 as oz

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    device = _rank_device(torch, local)
    if world > 1:
        _init_dist(dist, device)

    n, batch, s = (args.n or 512), args.batch, args.slices
    fn = oz.zgemm_strided_batched if args.method == "4m" else oz.zgemm3m_strided_batched
    A_h, B_h = make_inputs(batch, n, args.gamma, seed0=1000 * (rank + 1))
    A = to_dev_batched(torch, A_h, device)
    B = to_dev_batched(torch, B_h, device)
    C = torch.zeros((batch, n, n), dtype=torch.complex128, device=device).transpose(1, 2)
    stream = torch.cuda.current_stream()

    def step():
        fn("N", "N", 1.0, A, B, 0.0, C, s)

    # cross-call overlap (ozaki_set_overlap): each step's split starts under the previous step's
    # GEMM (same results; the bench places nothing between the calls)
    oz.set_overlap(not args.no_overlap)
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # ---- timed pass 1 (the headline): no per-launch instrumentation -- a timing event between
    # two kernels forces a full drain and defeats the split -> GEMM programmatic launch overlap
    clocks = ClockSampler(local)
    st0 = oz.get_stats()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    clocks.stop()
    if world > 1:
        dist.barrier()
    st1 = oz.get_stats()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    flops_all = fp64_equiv_flops(batch, n) * world
    value = flops_all / (ms_step * 1e-3) / 1e12
    launches = int(st1["kernel_launches"] - st0["kernel_launches"])

    # ---- timed pass 2 (same K steps): per-launch CUDA events on the launch stream give each
    # kernel's device time -> the roofline's kernel duration and the phase split
    # the kernel's own duration: without cross-call overlap (in pass 1 the next step's split CTAs
    # share the GEMM's last wave, which lengthens the GEMM grid while shortening the step)
    oz.set_overlap(False)
    oz.profile_enable(True)
    oz.profile_read()
    torch.cuda.synchronize()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        step()
    p1.record(stream)
    torch.cuda.synchronize()
    prof = oz.profile_read()
    oz.profile_enable(False)
    oz.set_overlap(not args.no_overlap)
    ms_instrumented = p0.elapsed_time(p1) / args.steps

    bf16_burst, bf16_sus, peak_src = peaks()
    peak_int8 = bf16_burst * INT8_OVER_BF16
    gemm = prof["k2_gemm"]
    gemm_ms = gemm["ms"] / max(1, gemm["launches"])
    alg_ops = int8_ops(batch, n, s, args.method)   # per launch: one GEMM launch per step (4M; fused 3M)
    achieved = alg_ops / (gemm_ms * 1e-3) / 1e12
    step_phase_ms = {k: v["ms"] / args.steps for k, v in prof.items()}

    out = {
        "metric": "FP64-equiv TFLOP/s (ZGEMM/DGEMM) vs slice count; INT8 pipe util; max rel err",
        "value": round(value, 3),
        "unit": "TFLOP/s (FP64-equivalent, 8mnk per ZGEMM)",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64 in/out; int8 x int8 -> int32 tensor-core products; f64 epilogue",
        "data": "synthetic (synth.kkr: graded-channel KKR blocks, seeded)",
        "config": {
            "workload": (f"BASELINE configs[1]: ZGEMM {n}x{n}x{n} KKR blocks (gamma={args.gamma}), "
                         f"{args.method.upper()}, s={s} ({8 * s - 1}-bit mode), strided-batched "
                         f"over {batch} energy points per GPU"),
            "slices": s, "method": args.method, "m": n, "n": n, "k": n,
            "batch_per_gpu": batch, "global_batch": batch * world,
            "parallelism": f"batch-sharded x{world} (no collective)",
            "cross_call_overlap": not args.no_overlap,
            "l2": "inputs exceed L2 (%.0f MB per GPU > 126 MB)" % (batch * 3 * n * n * 16 / 1e6),
        },
        "roofline": {
            "bound": "tensor",
            "kernel": "k_gemm (K2+K3: tcgen05 kind::i8 slice GEMM + FP64 epilogue)",
            "achieved": round(achieved, 2),
            "peak": round(peak_int8, 1),
            "unit": "TOPS (INT8 dense)",
            "frac": round(achieved / peak_int8, 4),
            "peak_source": f"{peak_src} bf16 burst {bf16_burst} TF/s x nominal int8/bf16 ratio 2",
            "algorithmic_ops_per_launch": alg_ops,
            "traffic": traffic_from_profile(s, args.method, n, batch, args.gamma),
            "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, profiles/gemm_traffic.json)",
            "kernel_ms_per_launch": round(gemm_ms, 5),
            "kernel_share_of_step": round(gemm_ms * gemm["launches"] / args.steps / max(1e-9, ms_instrumented), 4),
            "timing": ("kernel time from per-launch CUDA events on the launch stream in a second timed "
                       "pass of the same K steps without cross-call overlap (%.4f ms/step with the "
                       "events; the headline pass has none)" % ms_instrumented),
        },
        "roofline_split": split_roofline(step_phase_ms.get("k1_slice", 0.0), batch, n, s, args.method),
        "paper_context": {
            "claim": "GEMMul8 (Ozaki-II) high-precision modes: averaged 1.7x speedup of the LSMS "
                     "scattering-matrix inversion vs native FP64 (2 SCF iterations)",
            "hardware": "NVIDIA GB200 NVL4, cuBLAS + SCILIB-Accel offload (PAPER.md:121)",
            "source": "PAPER.md:129", "use": "context only, not a target for this metric"},
        "phase_ms_per_step": {k: round(v, 5) for k, v in step_phase_ms.items()},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    # e2e through the public API with HOST buffers (pinned), H2D + compute + D2H per step
    if not args.no_extras:
        C0 = C[0].cpu().numpy()          # entry 0 of the timed result, checked in the cpu_baseline leg
        out["e2e"] = e2e_leg(torch, oz, fn, A_h, B_h, batch, n, s, device, args, world)
        out["sweep"], sweep_samples = sweep_leg(torch, oz, A, B, C, batch, n)
        out["ozaki2"], C0_oz2, oz2_samples = ozaki2_leg(torch, oz, A, B, C, batch, n)
        out["native_fp64"] = native_leg(torch, A, B, batch, n)
    if rank == 0 and not args.no_extras and not args.no_cpu:
        # the ONLY use of oracle/ in the GPU arm: the host-core baseline and the parity samples
        out["cpu_baseline"], out["accuracy"], out["ozaki2"]["bitexact_vs_oracle_N16_sample"] = \
            cpu_baseline_leg(A_h, B_h, C0, C0_oz2, s, args.method, n)
        out["error_vs_true_fp64"] = error_table(A_h, B_h, n, {**sweep_samples, **oz2_samples})
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()

def e2e_leg(torch, oz, fn, A_h, B_h, batch, n, s, device, args, world):
    """End to end through the public API with HOST (pinned) buffers: the library's
    offload path pipelines H2D copies, the emulated ZGEMM and D2H copies."""
    import torch.distributed as dist
    stream = torch.cuda.current_stream()
    Ap = torch.from_numpy(np.ascontiguousarray(np.transpose(A_h, (0, 2, 1)))).pin_memory()
    Bp = torch.from_numpy(np.ascontiguousarray(np.transpose(B_h, (0, 2, 1)))).pin_memory()
    Cp = torch.empty((batch, n, n), dtype=torch.complex128).pin_memory()

    def step():
        fn("N", "N", 1.0, Ap.transpose(1, 2), Bp.transpose(1, 2), 0.0, Cp.transpose(1, 2), s)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    steps = max(3, min(args.steps, 10))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    val = fp64_equiv_flops(batch, n) * world / (ms * 1e-3) / 1e12
    return {"value": round(val, 3), "unit": "TFLOP/s (FP64-equivalent)", "ms_per_step": round(ms, 3),
            "h2d_bytes_per_step": int(Ap.numel() * 16 + Bp.numel() * 16),
            "d2h_bytes_per_step": int(Cp.numel() * 16),
            "path": "ozaki_zgemm_strided_batched on pinned HOST tensors (library offload: chunked, "
                    "H2D / GEMM / D2H overlapped on 3 streams)"}

def accuracy_leg(A_h, B_h, C0, s, method):
    """Entry 0: parity vs the oracle and error vs the TRUE product on a sample (called from the
    cpu_baseline leg, the only place bench.py uses oracle/)."""
    import oracle
    n = A_h.shape[1]
    rows = np.unique(np.r_[0, 1, 127, 128, 255, n - 1, np.arange(3, n, 37)])
    cols = np.unique(np.r_[0, 63, 64, 127, n - 1, np.arange(5, n, 41)])
    A0 = np.asfortranarray(A_h[0])
    B0 = np.asfortranarray(B_h[0])
    got = C0[np.ix_(rows, cols)]
    want = oracle.zgemm("N", "N", 1.0, A0[rows], B0[:, cols], 0.0, None, s, method)
    truth = oracle.exact_zproduct(A0[rows], B0[:, cols])
    absab = np.abs(A0[rows]) @ np.abs(B0[:, cols])
    nz = truth != 0
    bitexact = bool((got.real == want.real).all() and (got.imag == want.imag).all())
    return {"sample": f"entry 0, {len(rows)}x{len(cols)} entries incl. tile edges",
            "bitexact_vs_oracle": bitexact,
            "max_rel_err_vs_true_fp64": float(np.max(np.abs(got - truth)[nz] / np.abs(truth[nz]))),
            "max_err_over_absAB": float(np.max(np.abs(got - truth) / absab))}

def ozaki2_parity(A_h, B_h, C0_oz2, n, nmod=16):
    """Entry 0 of the Ozaki-II N=16 run vs oracle/ozaki2.py on a sample (cpu_baseline leg)."""
    from oracle import ozaki2 as o2
    rows = np.unique(np.r_[0, 127, 128, 255, n - 1, np.arange(3, n, 61)])
    cols = np.unique(np.r_[0, 127, 128, n - 1, np.arange(5, n, 67)])
    A0 = np.asfortranarray(A_h[0])
    B0 = np.asfortranarray(B_h[0])
    got = C0_oz2[np.ix_(rows, cols)]
    want = o2.zgemm("N", "N", 1.0, A0[rows], B0[:, cols], 0.0, None, nmod)
    return bool((got.real == want.real).all() and (got.imag == want.imag).all())

def error_table(A_h, B_h, n, samples):
    """North star: "max relative error against true FP64 per slice count" (SURVEY c-13, both
    definitions) for every swept mode, on the entry-0 sample; truth = oracle's exact product."""
    import oracle
    rows, cols = err_sample_idx(n)
    A0 = np.asfortranarray(A_h[0])
    B0 = np.asfortranarray(B_h[0])
    truth = oracle.exact_zproduct(A0[rows], B0[:, cols])
    absab = np.abs(A0[rows]) @ np.abs(B0[:, cols])
    nz = truth != 0
    out = {"sample": f"entry 0, {len(rows)}x{len(cols)} entries incl. tile edges",
           "definitions": "rel = max |C-T|/|T| over T != 0; comp = max |C-T| / (|A||B|)"}
    for key, got in samples.items():
        out[key] = {"rel": float(np.max(np.abs(got - truth)[nz] / np.abs(truth[nz]))),
                    "comp": float(np.max(np.abs(got - truth) / absab))}
    return out

def cpu_baseline_leg(A_h, B_h, C0, C0_oz2, s, method, n):
    base = cpu_baseline(A_h, B_h, s, method, n)
    acc = accuracy_leg(A_h, B_h, C0, s, method)
    oz2 = ozaki2_parity(A_h, B_h, C0_oz2, n) if C0_oz2 is not None else "not run"
    return base, acc, oz2

def err_sample_idx(n):
    rows = np.unique(np.r_[0, 1, 127, 128, 255, n - 1, np.arange(3, n, 29)])
    cols = np.unique(np.r_[0, 63, 64, 127, n - 1, np.arange(5, n, 31)])
    return rows, cols

def sweep_leg(torch, oz, A, B, C, batch, n):
    """FP64-eq TFLOP/s vs s for 4M and 3M on the same inputs (short timing).  Returns (table,
    entry-0 samples per (method, s)) -- the samples' error vs the TRUE product is computed in the
    cpu_baseline leg (the only place bench.py touches oracle/)."""
    res = {}
    samples = {}
    rows, cols = err_sample_idx(n)
    for method, fn in (("4m", oz.zgemm_strided_batched), ("3m", oz.zgemm3m_strided_batched)):
        for s in (3, 4, 5, 6, 7, 8, 9):
            for _ in range(2):
                fn("N", "N", 1.0, A, B, 0.0, C, s)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            reps = 5
            e0.record()
            for _ in range(reps):
                fn("N", "N", 1.0, A, B, 0.0, C, s)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            res[f"{method}_s{s}"] = round(fp64_equiv_flops(batch, n) / (ms * 1e-3) / 1e12, 2)
            samples[f"{method}_s{s}"] = C[0].cpu().numpy()[np.ix_(rows, cols)]
    return res, samples

def split_roofline(split_ms, batch, n, s, method):
    """K1 (split) vs HBM: algorithmic bytes per step = FP64 inputs read once + the INT8 slices of
    the embedded operands written once (4M: A' = m x 2k, B' = 2n x 2k; 3M: three m x k and three
    k x n operands), over the K1 device time per step, against the measured copy bandwidth."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as fh:
            hbm = float(json.load(fh)["hbm_gbs"])
        src = "MEASURED_PEAKS.json hbm_gbs (copy read+write)"
    except Exception:
        hbm, src = 7700.0, "B200_PROFILING.md fallback"
    read = 2 * batch * n * n * 16
    write = s * batch * (2 * n * n + 4 * n * n) if method == "4m" else s * batch * 6 * n * n
    gbs = (read + write) / (split_ms * 1e-3) / 1e9 if split_ms > 0 else 0.0
    kname = "k_split_fast" if s <= 8 else "k_split_sm"
    return {"bound": "hbm", "kernel": f"{kname} (exponent scan + INT8 digits, both operands, one launch)",
            "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s", "frac": round(gbs / hbm, 4),
            "algorithmic_bytes_per_step": int(read + write), "peak_source": src}

def ozaki2_leg(torch, oz, A, B, C, batch, n):
    """NEXT-1: Ozaki-II (CRT) on the same inputs, FP64-eq TFLOP/s, phase split and the residue
    GEMM's INT8 TOPS per moduli count.  Returns (record, entry-0 result at N=16 for the parity
    sample checked in the cpu_baseline leg)."""
    res = {}
    oz2_samples = {}
    for nmod in (10, 12, 14, 16, 18):
        for _ in range(2):
            oz.ozaki2_zgemm_strided_batched("N", "N", 1.0, A, B, 0.0, C, nmod)
        torch.cuda.synchronize()
        oz.profile_enable(True)
        oz.profile_read()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            oz.ozaki2_zgemm_strided_batched("N", "N", 1.0, A, B, 0.0, C, nmod)
        e1.record()
        torch.cuda.synchronize()
        pr = oz.profile_read()
        oz.profile_enable(False)
        ms = e0.elapsed_time(e1) / reps
        gemm_ms = pr["k2_gemm"]["ms"] / reps
        ops = 2 * nmod * n * (2 * n) * (2 * n) * batch     # one m x 2k x 2n INT8 GEMM per modulus (4M)
        oz2_samples[f"ozaki2_N{nmod}"] = C[0].cpu().numpy()[np.ix_(*err_sample_idx(n))]
        res[f"N{nmod}"] = {"tflops": round(fp64_equiv_flops(batch, n) / (ms * 1e-3) / 1e12, 2),
                           "ms": round(ms, 4),
                           "phase_ms": {"split": round(pr["k1_slice"]["ms"] / reps, 4),
                                        "residue_gemm": round(gemm_ms, 4),
                                        "crt": round(pr["other"]["ms"] / reps, 4)},
                           "gemm_int8_tops": round(ops / (gemm_ms * 1e-3) / 1e12, 1)}
    out = {"unit": "TFLOP/s (FP64-equivalent)", "moduli": res,
           "path": "ozaki2_zgemm_strided_batched (split -> k_gemm_crt -> k_crt)"}
    oz.ozaki2_zgemm_strided_batched("N", "N", 1.0, A, B, 0.0, C, 16)
    torch.cuda.synchronize()
    return out, C[0].cpu().numpy(), oz2_samples

def native_leg(torch, A, B, batch, n):
    """Context only (PAPER.md:119 'native FP64 GEMM'): cuBLAS complex128 batched matmul on the same
    inputs, TFLOP/s (8mnk per ZGEMM)."""
    for _ in range(2):
        torch.bmm(A, B)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        torch.bmm(A, B)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return {"value": round(fp64_equiv_flops(batch, n) / (ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s",
            "path": "torch.bmm complex128 (cuBLAS native FP64), context only"}

def cpu_baseline(A_h, B_h, s, method, n, budget_s=10.0):
    """The oracle on the host cores: whole n^3 ZGEMM entries of the same batch,
    as many as fit in ~budget_s seconds (at least one)."""
    import oracle
    cores = oracle.num_threads()
    done = 0
    t0 = time.perf_counter()
    while done < A_h.shape[0]:
        oracle.zgemm("N", "N", 1.0, np.asfortranarray(A_h[done]), np.asfortranarray(B_h[done]), 0.0, None,
                     s, method)
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    flops = 8 * n ** 3 * done
    return {"value": round(flops / dt / 1e12, 6), "unit": "TFLOP/s (FP64-equivalent)", "cores": cores,
            "kind": "oracle",
            "sample": f"{done} full {n}^3 ZGEMM entries of the batch ({method}, s={s}), exact-integer oracle, "
                      f"time-bounded ~{budget_s:.0f} s",
            "seconds": round(dt, 3)}

# ------------------------------------------------------------ C3 headline (configs[2])
C3_N = 8192
C3_FAMILIES = {"U": ("uniform", {}), "Phi1": ("spread", {"phi": 1.0})}
SWEEP_S = (3, 4, 5, 6, 7, 8, 9)


def c3_inputs(n, fam):
    """Seeded host inputs of one C3 family (numpy, Fortran order): A (seed 1/3), B (seed 2/4)."""
    name, kw = C3_FAMILIES[fam]
    sa, sb = (1, 2) if fam == "U" else (3, 4)
    A = np.asfortranarray(synth.make(name, n, n, sa, **kw))
    B = np.asfortranarray(synth.make(name, n, n, sb, **kw))
    return A, B


def c3_sample_idx(n, count=32, seed=5):
    """32 rows x 32 columns = 1024 sampled entries: tile edges (127/128, 255/256 ...), the
    middle, the last row / column, and seeded random indices."""
    g = np.random.default_rng(seed)
    edges = [0, 1, 127, 128, 255, 256, n // 2 - 1, n // 2, n - 129, n - 128, n - 2, n - 1]
    out = []
    for off in (0, 1):
        idx = set(min(n - 1, e) for e in edges)
        while len(idx) < count:
            idx.add(int(g.integers(0, n)))
        out.append(np.array(sorted(idx))[:count])
    return out[0], out[1]


def sm_int8_peak_tops(mhz):
    """INT8 dense rate at a given SM clock from the measured per-SM MMA rate."""
    return 2 * MAC_PER_CLK_SM * SMS * mhz * 1e6 / 1e12 if mhz else None


def ncu_record(workload):
    """Tensor-pipe utilisation / DRAM bytes of the GEMM per s from the committed ncu capture of
    this workload (profiles/ncu_<workload>.json, written by tools/ncu_bench.sh), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", f"ncu_{workload}.json")) as fh:
            return json.load(fh)
    except Exception:  # noqa: BLE001
        return None


def timed(torch, stream, fn, reps, clocks_index=None):
    """ms per call of fn() over `reps` calls between two events on `stream` (+ clocks)."""
    clocks = ClockSampler(clocks_index) if clocks_index is not None else None
    torch.cuda.synchronize()
    if clocks:
        clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    if clocks:
        clocks.stop()
    return e0.elapsed_time(e1) / reps, (clocks.summary() if clocks else None)


def profiled(torch, oz, stream, fn, reps, clocks_index):
    """Second pass with per-launch events (phase profiler) and without cross-call overlap:
    (step ms of this pass, GEMM kernel ms per launch, phase ms per call, clocks of this pass)."""
    ov = oz.get_overlap()
    oz.set_overlap(False)
    oz.profile_enable(True)
    oz.profile_read()
    ms, clk = timed(torch, stream, fn, reps, clocks_index)
    prof = oz.profile_read()
    oz.profile_enable(False)
    oz.set_overlap(ov)
    g = prof["k2_gemm"]
    gemm_ms = g["ms"] / max(1, g["launches"])
    return ms, gemm_ms, {k: round(v["ms"] / reps, 5) for k, v in prof.items()}, clk


def c3_split_bytes(n, s):
    """K1 algorithmic bytes of one DGEMM n^3: both FP64 operands read once, s INT8 slices of
    each written once, the int32 exponents."""
    return 2 * 8 * n * n + 2 * s * n * n + 2 * 4 * n


def run_c3(args):
    import torch
    import torch.distributed as dist
    import paper_2603_29975_b200 as oz
    from paper_2603_29975_b200 import dist as zd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    device = _rank_device(torch, local)
    if world > 1:
        _init_dist(dist, device)
    n, s = args.n or C3_N, args.slices
    pairs = s * (s + 1) // 2
    stream = torch.cuda.current_stream()

    A_h, B_h = c3_inputs(n, "U")
    A = oz.colmajor(torch.from_numpy(A_h).to(device))
    B = oz.colmajor(torch.from_numpy(B_h).to(device))
    C = torch.zeros((n, n), dtype=torch.float64, device=device).t()

    def dgemm_dev(a, b, c, ss=s):
        oz.dgemm("N", "N", 1.0, a, b, 0.0, c, ss)

    def step(ss=s):
        if world == 1:
            dgemm_dev(A, B, C, ss)
        else:
            zd.sharded_gemm_columns(lambda a, b, c: dgemm_dev(a, b, c, ss), A, B, C, rank, world)

    oz.set_overlap(not args.no_overlap)
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # ---- timed pass 1 (headline): no per-launch instrumentation (PDL overlap intact)
    st0 = oz.get_stats()
    if world > 1:
        dist.barrier()
    ms_local, clocks = timed(torch, stream, step, args.steps, local)
    st1 = oz.get_stats()
    ms_step = zd.max_over_ranks(ms_local, device)
    value = 2.0 * n ** 3 / (ms_step * 1e-3) / 1e12
    launches = int(st1["kernel_launches"] - st0["kernel_launches"])

    # ---- timed pass 2: per-launch events give the GEMM kernel's own duration
    if world > 1:
        dist.barrier()
    ms_instr, gemm_ms, phase, clocks2 = profiled(torch, oz, stream, step, args.steps, local)
    bf16_burst, bf16_sus, peak_src = peaks()
    peak_int8 = bf16_burst * INT8_OVER_BF16
    if world > 1:
        own = [b - a for a, b in zd.column_blocks(n, rank, world, 4)[1] if b > a]
        frac_cols = (sum(own) / max(1, len(own))) / n
    else:
        frac_cols = 1.0
    alg_ops = 2 * pairs * n * n * n * frac_cols           # INT8 ops of one GEMM launch
    achieved = alg_ops / (gemm_ms * 1e-3) / 1e12
    at_clk = sm_int8_peak_tops(clocks2.get("sm_mhz")) if clocks2 else None
    ncu = ncu_record("c3")
    ncu_s = (ncu or {}).get("per_s", {}).get(str(s), {})
    split_ms = phase.get("k1_slice", 0.0) + phase.get("k1_exponent", 0.0)
    hbm = hbm_peak()
    out = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "TFLOP/s (FP64-equivalent, 2mnk per DGEMM)",
        "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f64 in/out; int8 x int8 -> int32 tensor-core products; f64 epilogue",
        "data": "synthetic (synth.uniform U[-1,1), seeded; sweep also synth.spread phi=1)",
        "config": {
            "workload": (f"BASELINE configs[2]: square DGEMM {n}x{n}x{n}, uniform inputs, s={s} "
                         f"({8 * s - 1}-bit mode), NN, alpha=1 beta=0"),
            "slices": s, "m": n, "n": n, "k": n, "global_batch": 1,
            "parallelism": (f"column slabs of C x{world} + chunked NCCL all-gather" if world > 1
                            else "1 GPU"),
            "cross_call_overlap": not args.no_overlap,
            "l2": "inputs exceed L2 (A, B, C %.0f MB each > 126 MB): no flush needed" % (8 * n * n / 1e6),
        },
        "roofline": {
            "bound": "tensor",
            "kernel": "k_gemm_lv2 (K2+K3: tcgen05 kind::i8 CTA-pair slice GEMM + fused FP64 epilogue)",
            "achieved": round(achieved, 2), "peak": round(peak_int8, 1),
            "unit": "TOPS (INT8 dense)", "frac": round(achieved / peak_int8, 4),
            "peak_source": f"{peak_src} bf16 burst {bf16_burst} TF/s x nominal int8/bf16 ratio 2",
            "traffic": ncu_s.get("dram_bytes"),
            "traffic_unit": "bytes per launch (ncu dram__bytes_read.sum + write.sum, profiles/ncu_c3.json)",
            "algorithmic_ops_per_launch": int(alg_ops),
            "kernel_ms_per_launch": round(gemm_ms, 5),
            "kernel_share_of_step": round(gemm_ms / max(1e-9, ms_instr), 4),
            "frac_at_pass_clock": round(achieved / at_clk, 4) if at_clk else None,
            "pass_clock_note": ("achieved / (148 SMs x 8192 MAC/clk x 2 x the SM clock sampled in the "
                                "kernel-time pass)"),
            "ncu_tensor_pipe_active_pct": ncu_s.get("tensor_pipe_pct"),
            "ncu_source": (ncu or {}).get("source"),
            "timing": ("kernel time from per-launch CUDA events on the launch stream in a second pass of "
                       "the same K steps without cross-call overlap (%.4f ms/step in that pass; the "
                       "headline pass has no events)" % ms_instr),
            "kernel_pass_clocks": clocks2,
        },
        "roofline_split": {
            "bound": "hbm", "kernel": "k_split_cluster (one HBM read per operand: clusters of up to 16 CTAs along K, partial row maxima exchanged through distributed shared memory, INT8 digits of both operands)",
            "achieved": round(c3_split_bytes(n, s) / (split_ms * 1e-3) / 1e9, 1) if split_ms else None,
            "peak": hbm[0], "unit": "GB/s",
            "frac": round(c3_split_bytes(n, s) / (split_ms * 1e-3) / 1e9 / hbm[0], 4) if split_ms else None,
            "algorithmic_bytes_per_step": c3_split_bytes(n, s), "peak_source": hbm[1],
            "ms_per_step": round(split_ms, 5),
            "traffic": ncu_s.get("split_dram_bytes"),
            "traffic_unit": "bytes per launch (ncu dram__bytes_read.sum + write.sum, profiles/ncu_c3.json)",
            "ncu_isolated": ({"ms": round(ncu_s["split_ms"], 5),
                              "frac": round(c3_split_bytes(n, s) / (ncu_s["split_ms"] * 1e-3) / 1e9 / hbm[0], 4),
                              "note": "the same launch timed alone under ncu (cold L2, no power-capped GEMM "
                                      "beside it); the bench pass above runs between the GEMMs of the step"}
                             if ncu_s.get("split_ms") else None)},
        "phase_ms_per_step": phase,
        "gpu_launches": launches,
        "clocks": clocks,
        "paper_context": {
            "claim": "GEMMul8 (Ozaki-II) high-precision modes: averaged 1.7x speedup of the LSMS "
                     "scattering-matrix inversion vs native FP64 (2 SCF iterations)",
            "hardware": "NVIDIA GB200 NVL4, cuBLAS + SCILIB-Accel offload (PAPER.md:121)",
            "source": "PAPER.md:129", "use": "context only, not a target for this metric"},
    }
    rows, cols = c3_sample_idx(n)
    samples = {}
    if not args.no_extras:
        out["e2e"] = c3_e2e_leg(torch, oz, A_h, B_h, n, s, device, rank, world, args)
    if not args.no_extras and world == 1:
        out["sweep"] = {}
        for fam in C3_FAMILIES:
            if fam == "U":
                Af, Bf, Ah_f, Bh_f = A, B, A_h, B_h
            else:
                Ah_f, Bh_f = c3_inputs(n, fam)
                Af = oz.colmajor(torch.from_numpy(Ah_f).to(device))
                Bf = oz.colmajor(torch.from_numpy(Bh_f).to(device))
            out["sweep"][fam] = {}
            for ss in SWEEP_S:
                call = lambda ss=ss: oz.dgemm("N", "N", 1.0, Af, Bf, 0.0, C, ss)   # noqa: E731
                for _ in range(2):
                    call()
                ms_u, clk_u = timed(torch, stream, call, 5, local)
                ms_p, g_ms, ph, clk_p = profiled(torch, oz, stream, call, 3, local)
                ops = 2 * (ss * (ss + 1) // 2) * n ** 3
                ach = ops / (g_ms * 1e-3) / 1e12
                pk_clk = sm_int8_peak_tops(clk_p.get("sm_mhz")) if clk_p else None
                out["sweep"][fam][f"s{ss}"] = {
                    "tflops": round(2.0 * n ** 3 / (ms_u * 1e-3) / 1e12, 2), "ms": round(ms_u, 4),
                    "clocks": {"sm_mhz": clk_u.get("sm_mhz"), "reasons": clk_u.get("reasons")},
                    "gemm_int8_tops": round(ach, 1), "gemm_frac_of_peak": round(ach / peak_int8, 4),
                    "gemm_frac_at_pass_clock": round(ach / pk_clk, 4) if pk_clk else None,
                    "gemm_ms": round(g_ms, 4), "instrumented_step_ms": round(ms_p, 4),
                    "kernel_le_step": bool(g_ms <= ms_p * 1.0001),
                    "instrumented_pass_clocks": {"sm_mhz": clk_p.get("sm_mhz"), "reasons": clk_p.get("reasons")},
                    "phase_ms": ph,
                    "ncu_tensor_pipe_active_pct": (ncu or {}).get("per_s", {}).get(str(ss), {}).get("tensor_pipe_pct")
                    if fam == "U" else None}
                samples[f"{fam}_s{ss}"] = C[torch.from_numpy(rows).to(device)][:, torch.from_numpy(cols).to(device)].cpu().numpy()
            if fam != "U":
                del Af, Bf
        out["ozaki2"] = c3_ozaki2_leg(torch, oz, A, B, C, n, stream, local, rows, cols, samples)
        out["native_fp64"] = native_gemm_leg(torch, A, B, n)
        out["general_alpha_beta"] = general_ab_leg(torch, oz, A, B, C, n, s, stream, local, device)
        out["extra_workloads"] = {"c2x30": c2x30_leg(torch, oz, device, stream, local, args),
                                  "c4": c4_leg(torch, oz, device, stream, local)}
    out["sweep_note"] = ("per s: FP64-eq TF/s from an uninstrumented pass (5 calls, clocks of that pass); "
                         "GEMM INT8 TOPS from per-launch events in a second pass (3 calls) with its own "
                         "clocks; the roofline fractions use the measured peak and the pass clock")
    if rank == 0 and world == 1 and not args.no_extras and not args.no_cpu:
        out["cpu_baseline"] = c3_cpu_baseline(A_h, B_h, s, n)
        out["accuracy"], out["error_vs_true_fp64"] = c3_accuracy(A_h, B_h, n, s, rows, cols, samples)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy read+write)"
    except Exception:  # noqa: BLE001
        return 7700.0, "B200_PROFILING.md fallback"


def c3_e2e_leg(torch, oz, A_h, B_h, n, s, device, rank, world, args):
    """End to end through the public API with pinned HOST buffers: ozaki_dgemm on host pointers
    (the library's offload path: row panels of A and column panels of B moved once each, block
    (i, j) of C computed and copied back as soon as its panels are in, H2D / GEMM / D2H on three
    streams) -- with N ranks each rank runs its column slab of C."""
    import torch.distributed as dist
    from paper_2603_29975_b200 import dist as zd
    j0, j1 = zd.column_slab(n, rank, world)
    Ap = torch.from_numpy(np.ascontiguousarray(A_h.T)).pin_memory().t()
    Bp = torch.from_numpy(np.ascontiguousarray(B_h[:, j0:j1].T)).pin_memory().t()
    Cp = torch.empty((j1 - j0, n), dtype=torch.float64).pin_memory().t()
    stream = torch.cuda.current_stream()

    def step():
        oz.dgemm("N", "N", 1.0, Ap, Bp, 0.0, Cp, s)

    step()
    torch.cuda.synchronize()
    reps = max(3, min(args.steps, 5))
    if world > 1:
        dist.barrier()
    ms, _ = timed(torch, stream, step, reps)
    ms = zd.max_over_ranks(ms, device)
    return {"value": round(2.0 * n ** 3 / (ms * 1e-3) / 1e12, 3), "unit": "TFLOP/s (FP64-equivalent)",
            "ms_per_step": round(ms, 3),
            "h2d_bytes_per_step": int((Ap.numel() + Bp.numel()) * 8 * world),
            "d2h_bytes_per_step": int(Cp.numel() * 8 * world),
            "path": "ozaki_dgemm on pinned HOST tensors (library 2-D block offload), "
                    + ("column slab per rank" if world > 1 else "one call per step")}


def c3_ozaki2_leg(torch, oz, A, B, C, n, stream, local, rows, cols, samples):
    res = {}
    dev = A.device
    for nmod in (12, 14, 16):
        call = lambda nmod=nmod: oz.ozaki2_dgemm("N", "N", 1.0, A, B, 0.0, C, nmod)   # noqa: E731
        for _ in range(2):
            call()
        ms_u, clk = timed(torch, stream, call, 5, local)
        ms_p, g_ms, ph, _ = profiled(torch, oz, stream, call, 3, local)
        ops = 2 * nmod * n ** 3
        res[f"N{nmod}"] = {"tflops": round(2.0 * n ** 3 / (ms_u * 1e-3) / 1e12, 2), "ms": round(ms_u, 4),
                           "sm_mhz": clk.get("sm_mhz"), "phase_ms": ph,
                           "residue_gemm_int8_tops": round(ops / (g_ms * 1e-3) / 1e12, 1)}
        samples[f"ozaki2_N{nmod}"] = C[torch.from_numpy(rows).to(dev)][:, torch.from_numpy(cols).to(dev)].cpu().numpy()
    return {"unit": "TFLOP/s (FP64-equivalent)", "moduli": res,
            "path": "ozaki2_dgemm (split -> k_gemm_crt -> k_crt), NEXT-1"}


def general_ab_leg(torch, oz, A, B, C, n, s, stream, local, device):
    """The LU trailing update's alpha = -1, beta = 1 (R7's general FMA epilogue, C read) against
    the alpha = 1, beta = 0 store, on C3 (s = 7) and on C2 x 30 (4M, s = 7)."""
    res = {}
    for name, ab in (("unit", (1.0, 0.0)), ("lu_update", (-1.0, 1.0))):
        call = lambda ab=ab: oz.dgemm("N", "N", ab[0], A, B, ab[1], C, s)   # noqa: E731
        for _ in range(2):
            call()
        ms, clk = timed(torch, stream, call, 5, local)
        res[f"c3_{name}"] = {"tflops": round(2.0 * n ** 3 / (ms * 1e-3) / 1e12, 2), "sm_mhz": clk.get("sm_mhz")}
    batch, nz = 30, 512
    A_h, B_h = make_inputs(batch, nz, 3.0, seed0=1000)
    Az, Bz = to_dev_batched(torch, A_h, device), to_dev_batched(torch, B_h, device)
    Cz = torch.zeros((batch, nz, nz), dtype=torch.complex128, device=device).transpose(1, 2)
    for name, ab in (("unit", (1.0, 0.0)), ("lu_update", (-1.0, 1.0))):
        call = lambda ab=ab: oz.zgemm_strided_batched("N", "N", ab[0], Az, Bz, ab[1], Cz, s)   # noqa: E731
        for _ in range(3):
            call()
        ms, clk = timed(torch, stream, call, 20, local)
        res[f"c2x30_{name}"] = {"tflops": round(fp64_equiv_flops(batch, nz) / (ms * 1e-3) / 1e12, 2),
                                "sm_mhz": clk.get("sm_mhz")}
    for w in ("c3", "c2x30"):
        res[f"{w}_ratio"] = round(res[f"{w}_lu_update"]["tflops"] / res[f"{w}_unit"]["tflops"], 4)
    return res


def native_gemm_leg(torch, A, B, n):
    """Context only (PAPER.md:119 'native FP64 GEMM'): cuBLAS FP64 matmul on the same inputs."""
    for _ in range(2):
        torch.matmul(A, B)
    ms, _ = timed(torch, torch.cuda.current_stream(), lambda: torch.matmul(A, B), 5)
    return {"value": round(2.0 * n ** 3 / (ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s",
            "path": "torch.matmul float64 (cuBLAS native FP64 DGEMM), context only"}


def c2x30_leg(torch, oz, device, stream, local, args):
    """Extra field: 30 x ZGEMM 512^3 KKR (gamma=3), 4M, s=7, one strided-batched call per step."""
    batch, n, s = 30, 512, 7
    A_h, B_h = make_inputs(batch, n, 3.0, seed0=1000)
    A = to_dev_batched(torch, A_h, device)
    B = to_dev_batched(torch, B_h, device)
    C = torch.zeros((batch, n, n), dtype=torch.complex128, device=device).transpose(1, 2)
    call = lambda: oz.zgemm_strided_batched("N", "N", 1.0, A, B, 0.0, C, s)   # noqa: E731
    for _ in range(3):
        call()
    ms, clk = timed(torch, stream, call, 20, local)
    ms_p, g_ms, ph, _ = profiled(torch, oz, stream, call, 10, local)
    ops = int8_ops(batch, n, s, "4m")
    return {"workload": "30 x ZGEMM 512^3 KKR (gamma=3), 4M, s=7 (configs[1] batched over 30 energy points)",
            "tflops": round(fp64_equiv_flops(batch, n) / (ms * 1e-3) / 1e12, 2), "ms": round(ms, 4),
            "sm_mhz": clk.get("sm_mhz"), "gemm_int8_tops": round(ops / (g_ms * 1e-3) / 1e12, 1),
            "phase_ms": ph}


def c4_leg(torch, oz, device, stream, local):
    """Extra field: configs[3] at its stated size, 256 x ZGEMM 1024^3 KKR (gamma=1), 4M, s=7,
    one strided-batched call (8 distinct blocks tiled over the batch)."""
    batch, n, s, distinct = 256, 1024, 7, 8
    As = [oz.colmajor(torch.from_numpy(np.asfortranarray(synth.kkr(n, n, seed=10 + i, gamma=1.0))).to(device))
          for i in range(distinct)]
    Bs = [oz.colmajor(torch.from_numpy(np.asfortranarray(synth.kkr(n, n, seed=50 + i, gamma=1.0))).to(device))
          for i in range(distinct)]
    A = torch.stack([As[i % distinct] for i in range(batch)]).transpose(1, 2).contiguous().transpose(1, 2)
    B = torch.stack([Bs[i % distinct] for i in range(batch)]).transpose(1, 2).contiguous().transpose(1, 2)
    del As, Bs
    C = torch.zeros((batch, n, n), dtype=torch.complex128, device=device).transpose(1, 2)
    call = lambda: oz.zgemm_strided_batched("N", "N", 1.0, A, B, 0.0, C, s)   # noqa: E731
    for _ in range(2):
        call()
    ms, clk = timed(torch, stream, call, 5, local)
    ms_p, g_ms, ph, _ = profiled(torch, oz, stream, call, 3, local)
    ops = int8_ops(batch, n, s, "4m")
    res = {"workload": "256 x ZGEMM 1024^3 KKR (gamma=1), 4M, s=7, one strided-batched call (configs[3], 1 GPU)",
           "tflops": round(fp64_equiv_flops(batch, n) / (ms * 1e-3) / 1e12, 2), "ms": round(ms, 4),
           "sm_mhz": clk.get("sm_mhz"), "gemm_int8_tops": round(ops / (g_ms * 1e-3) / 1e12, 1),
           "phase_ms": ph}
    del A, B, C
    torch.cuda.empty_cache()
    return res


def c3_cpu_baseline(A_h, B_h, s, n, rows=32):
    """The oracle, as it stands, on the host cores: a slab of `rows` full rows of C3 (all n
    columns, full k: the same per-row / per-column exponents as the whole problem)."""
    import oracle
    oracle.build()
    cores = oracle.num_threads()
    t0 = time.perf_counter()
    oracle.dgemm("N", "N", 1.0, A_h[:rows], B_h, 0.0, None, s)
    dt = time.perf_counter() - t0
    return {"value": round(2.0 * rows * n * n / dt / 1e12, 6), "unit": "TFLOP/s (FP64-equivalent)",
            "cores": cores, "kind": "oracle",
            "sample": f"C3 rows 0..{rows - 1} x all {n} columns (k = {n}, s = {s}) of the exact-integer oracle",
            "seconds": round(dt, 3),
            "per_entry_us": round(dt / (rows * n) * 1e6, 4),
            "extrapolated_full_s": round(dt * n / rows, 1),
            "extrapolated_note": "EXTRAPOLATED: full 8192^3 time = slab time x n / rows (not measured)"}


def c3_accuracy(A_h, B_h, n, s, rows, cols, samples):
    """Sampled parity of the headline result (and of every swept s) vs the oracle, and the
    north star's max relative error vs the TRUE FP64 product (SURVEY c-13, both definitions)
    on the 1024 sampled entries (truth = the oracle's exact long-accumulator product)."""
    import oracle
    from oracle import ozaki2 as o2
    acc = {"sample": f"{len(rows)} x {len(cols)} = {len(rows) * len(cols)} entries incl. tile edges",
           "bitexact_vs_oracle": {}}
    err = {"sample": acc["sample"],
           "definitions": "rel = max |C-T|/|T| over T != 0; comp = max |C-T| / (|A||B|)_ij; T = exact product"}
    for fam in C3_FAMILIES:
        Ah, Bh = (A_h, B_h) if fam == "U" else c3_inputs(n, fam)
        Ar, Bc = np.ascontiguousarray(Ah[rows]), np.asfortranarray(Bh[:, cols])
        truth = oracle.exact_product(Ar, Bc)
        absab = np.abs(Ar) @ np.abs(Bc)
        nz = truth != 0
        err[fam] = {}
        for ss in SWEEP_S:
            got = samples.get(f"{fam}_s{ss}")
            if got is None:
                continue
            want = oracle.dgemm("N", "N", 1.0, Ar, Bc, 0.0, None, ss)
            acc["bitexact_vs_oracle"][f"{fam}_s{ss}"] = bool((got == want).all())
            err[fam][f"s{ss}"] = {"rel": float(np.max(np.abs(got - truth)[nz] / np.abs(truth[nz]))),
                                  "comp": float(np.max(np.abs(got - truth) / absab))}
        if fam == "U":
            for key in [k for k in samples if k.startswith("ozaki2_N")]:
                got = samples[key]
                nmod = int(key.split("N")[-1])
                if nmod == 16:
                    want = o2.dgemm("N", "N", 1.0, Ar[:8], Bc[:, :8], 0.0, None, nmod)
                    acc["bitexact_vs_oracle"][f"ozaki2_N16 (8x8 sub-sample)"] = bool((got[:8, :8] == want).all())
                err[fam][key] = {"rel": float(np.max(np.abs(got - truth)[nz] / np.abs(truth[nz]))),
                                 "comp": float(np.max(np.abs(got - truth) / absab))}
        # native FP64 (ascending-k fma) on the same sample, for comparison
        nat = oracle.fp64_product(Ar, Bc) if hasattr(oracle, "fp64_product") else None
        if nat is not None:
            err[fam]["native_fp64_fma_loop"] = {"rel": float(np.max(np.abs(nat - truth)[nz] / np.abs(truth[nz]))),
                                                "comp": float(np.max(np.abs(nat - truth) / absab))}
    return acc, err


def run_reference(args):
    """Reference arm of this tier: the CPU oracle, as it stands, on the host cores, on the same
    workload as our arm; each step a bounded sample of it.  Under torchrun only rank 0 runs."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    oracle.build()
    cores = oracle.num_threads()
    s = args.slices
    if args.workload == "c3":
        n = args.n or C3_N
        A_h, B_h = c3_inputs(n, "U")
        rows = 8                   # bounded sample per step: an 8-row slab of C (all n columns)
        Ar = np.ascontiguousarray(A_h[:rows])
        work = lambda: oracle.dgemm("N", "N", 1.0, Ar, B_h, 0.0, None, s)   # noqa: E731
        flops = 2.0 * rows * n * n
        unit = "TFLOP/s (FP64-equivalent, 2mnk per DGEMM)"
        sample = (f"rows 0..{rows - 1} x all {n} columns of C3 per step (full k = {n}; the oracle "
                  f"splits all of B each step)")
        workload = (f"BASELINE configs[2]: square DGEMM {n}x{n}x{n}, uniform inputs, s={s} "
                    f"({8 * s - 1}-bit mode), NN, alpha=1 beta=0")
        cfg = {"workload": workload, "slices": s, "m": n, "n": n, "k": n, "global_batch": 1,
               "parallelism": "host cores (oracle)"}
    else:
        n = args.n or 512
        A_h, B_h = make_inputs(1, n, args.gamma, seed0=1000)
        A0 = np.asfortranarray(A_h[0])
        B0 = np.asfortranarray(B_h[0])
        rows = max(8, n // 16)     # bounded sample per step: a 32-row slab of one block
        work = lambda: oracle.zgemm("N", "N", 1.0, A0[:rows], B0, 0.0, None, s, args.method)   # noqa: E731
        flops = 8.0 * rows * n * n
        unit = "TFLOP/s (FP64-equivalent, 8mnk per ZGEMM)"
        sample = f"{rows} rows of one {n}^3 ZGEMM per step"
        cfg = {"workload": (f"BASELINE configs[1]: ZGEMM {n}^3 KKR block (gamma={args.gamma}), "
                            f"{args.method.upper()}, s={s}; each step a {rows}x{n} row slab"),
               "slices": s, "method": args.method}
    for _ in range(max(0, min(args.warmup, 1))):
        work()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        work()
    dt = (time.perf_counter() - t0) / args.steps
    val = flops / dt / 1e12
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(val, 6), "unit": unit,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64 / exact int64 (CPU oracle)",
        "data": "synthetic (seeded, same generator as our arm)",
        "config": cfg,
        "cpu_baseline": {"value": round(val, 6), "unit": unit, "cores": cores, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(val, 6), "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(args):
    """`python bench.py --gpus N` without a launcher: start N ranks with torch.distributed.run
    on 127.0.0.1 (one process per GPU) and pass rank 0's JSON line through."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")      # communicator / NVLS lines on stderr
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args)
        return
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.workload == "c3":
        run_c3(args)
    elif args.workload == "c2x30":
        run_ours(args)
    else:
        run_config(args)

if __name__ == "__main__":
    main()
