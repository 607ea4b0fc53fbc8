"""A/B of small-problem device time (CUDA graph replay) between library builds: configs[1]
single ZGEMM 512^3 s=7 (split-K) and configs[0] DGEMM 64^3.  usage: ab_small.py <lib>"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_29975_b200 as oz  # noqa: E402

oz.LIB_PATH = os.path.join(ROOT, "paper_2603_29975_b200", sys.argv[1])
import synth  # noqa: E402


def dev(x):
    return oz.colmajor(torch.from_numpy(np.asfortranarray(x)).cuda())


def graph_us(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s2):
            for _ in range(reps):
                fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


A, B = dev(synth.kkr(512, 512, seed=1000, gamma=3.0)), dev(synth.kkr(512, 512, seed=1001, gamma=3.0))
C = dev(np.zeros((512, 512), complex))
res = {"lib": sys.argv[1]}
for sk in ("auto", "1"):
    if sk == "1":
        os.environ["OZAKI_SPLITK"] = "1"
    res[f"c2_s7_splitk_{sk}"] = round(graph_us(lambda: oz.zgemm("N", "N", 1.0, A, B, 0.0, C, 7)), 2)
    os.environ.pop("OZAKI_SPLITK", None)
a, b, c = dev(synth.uniform(64, 64, 1)), dev(synth.uniform(64, 64, 2)), dev(np.zeros((64, 64)))
res["c1_s7"] = round(graph_us(lambda: oz.dgemm("N", "N", 1.0, a, b, 0.0, c, 7)), 2)
print(json.dumps(res), flush=True)
