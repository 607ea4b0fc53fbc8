"""Small-GEMM latency on one B200 (SURVEY §8(a) a7, configs[0] / configs[1] single block):
per-call device time of back-to-back eager calls (CUDA events), the host time to enqueue one
call (Python binding + library), and the device time when the same calls are replayed from a
CUDA graph (no host in the loop).  Prints one JSON line per case.

usage: python tools/small_gemm_latency.py [--splitk auto|1]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2603_29975_b200 as oz  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--splitk", default="auto")
ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()
if a.splitk != "auto":
    os.environ["OZAKI_SPLITK"] = a.splitk


def dev(x):
    return oz.colmajor(torch.from_numpy(np.asfortranarray(x)).cuda())


cases = []
for s in (4, 7):
    A, B = dev(synth.uniform(64, 64, 1)), dev(synth.uniform(64, 64, 2))
    C = dev(np.zeros((64, 64)))
    cases.append((f"c1 DGEMM 64^3 s={s}", 2 * 64 ** 3, lambda A=A, B=B, C=C, s=s: oz.dgemm("N", "N", 1.0, A, B, 0.0, C, s)))
for s in (4, 7):
    A = dev(synth.kkr(512, 512, seed=1000, gamma=3.0))
    B = dev(synth.kkr(512, 512, seed=1001, gamma=3.0))
    C = dev(np.zeros((512, 512), complex))
    cases.append((f"c2 ZGEMM 512^3 4M s={s}", 8 * 512 ** 3, lambda A=A, B=B, C=C, s=s: oz.zgemm("N", "N", 1.0, A, B, 0.0, C, s)))
for n in (1024, 2048):
    A, B = dev(synth.uniform(n, n, 3)), dev(synth.uniform(n, n, 4))
    C = dev(np.zeros((n, n)))
    cases.append((f"DGEMM {n}^3 s=7", 2 * n ** 3, lambda A=A, B=B, C=C: oz.dgemm("N", "N", 1.0, A, B, 0.0, C, 7)))

# raw C-ABI calls (arguments marshalled once): the library's own host time per call
import ctypes  # noqa: E402
L = oz.lib()
L.ozaki_set_stream(ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
Ar = dev(synth.kkr(512, 512, seed=1000, gamma=3.0))
Br = dev(synth.kkr(512, 512, seed=1001, gamma=3.0))
Cr = dev(np.zeros((512, 512), complex))
one, zero = (ctypes.c_double * 2)(1.0, 0.0), (ctypes.c_double * 2)(0.0, 0.0)
raw_args = (b"N", b"N", 512, 512, 512, one, Ar.data_ptr(), 512, Br.data_ptr(), 512, zero, Cr.data_ptr(), 512, 7)
a64, b64, c64 = dev(synth.uniform(64, 64, 1)), dev(synth.uniform(64, 64, 2)), dev(np.zeros((64, 64)))
raw64 = (b"N", b"N", 64, 64, 64, 1.0, a64.data_ptr(), 64, b64.data_ptr(), 64, 0.0, c64.data_ptr(), 64, 7)
for nm, f, args in (("raw ozaki_zgemm 512^3 s=7", L.ozaki_zgemm, raw_args), ("raw ozaki_dgemm 64^3 s=7", L.ozaki_dgemm, raw64)):
    for _ in range(5):
        f(*args)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.reps):
        f(*args)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(json.dumps({"case": nm, "splitk": a.splitk, "host_us_per_call": round((t1 - t0) / a.reps * 1e6, 2),
                      "wall_us_per_call_incl_drain": round((t2 - t0) / a.reps * 1e6, 2)}), flush=True)

st = torch.cuda.current_stream()
for name, flops, fn in cases:
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    # eager: device time of back-to-back calls and host enqueue time
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    for _ in range(a.reps):
        fn()
    e1.record(st)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    eager_ms = e0.elapsed_time(e1) / a.reps
    host_us = (t1 - t0) / a.reps * 1e6
    # CUDA graph: capture reps calls, replay
    g = torch.cuda.CUDAGraph()
    s2 = torch.cuda.Stream()
    s2.wait_stream(st)
    with torch.cuda.stream(s2):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s2):
            for _ in range(a.reps):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0.record(st)
    g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    graph_ms = e0.elapsed_time(e1) / a.reps
    print(json.dumps({"case": name, "splitk": a.splitk, "eager_us_per_call": round(eager_ms * 1e3, 2),
                      "host_enqueue_us_per_call": round(host_us, 2), "graph_us_per_call": round(graph_ms * 1e3, 2),
                      "eager_tflops": round(flops / (eager_ms * 1e-3) / 1e12, 3),
                      "graph_tflops": round(flops / (graph_ms * 1e-3) / 1e12, 3)}), flush=True)
