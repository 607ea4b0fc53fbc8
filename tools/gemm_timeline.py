"""Timeline of CTA 0 of the pair GEMM (globaltimer ns, relative to kernel entry) for small
problems: where the fixed per-launch time goes.  The timeline is compiled only with
-DOZK_TIMELINE: this tool builds paper_2603_29975_b200/libozaki_timeline.so (once, ~3 min) and
loads it instead of the production library.  usage: python tools/gemm_timeline.py"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2603_29975_b200 as oz  # noqa: E402
from paper_2603_29975_b200 import _build  # noqa: E402

TL_LIB = os.path.join(_build.PKG, "libozaki_timeline.so")
if not os.path.exists(TL_LIB):
    import subprocess
    cmd = [_build.nvcc(), *_build.NVCC_FLAGS, "-DOZK_TIMELINE", "-I", os.path.join(ROOT, "include"), "-I",
           _build.CSRC, os.path.join(_build.CSRC, "ozaki.cu"), "-o", TL_LIB]
    subprocess.run(cmd, check=True, capture_output=True)
oz.LIB_PATH = TL_LIB

EV = ["entry", "prologue", "depwait", "tma0_issued", "full0", "mma_pass0_done", "mma_end", "epi_pass0",
      "epi_last_pass", "epi_store_done", "exit", "epi_drained", "epi_probe_loads", "mma_slots_pass1", "epi_release_slot0", "mma_full_pass1", "entry_latest_cta", "exit_latest_cta", "mma_end_latest"]


def dev(x):
    return oz.colmajor(torch.from_numpy(np.asfortranarray(x)).cuda())


def timeline(name, fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    L = oz.lib()
    buf = (ctypes.c_uint64 * 64)()
    L.ozaki_debug_timing(1, buf, 64)
    fn()
    torch.cuda.synchronize()
    L.ozaki_debug_timing(0, buf, 64)
    t = [int(buf[32 + i]) for i in range(len(EV))]
    t0 = t[0]
    print(json.dumps({"case": name, **{e: (round((v - t0) / 1e3, 2) if v else None) for e, v in zip(EV, t)}}))


A, B, C = dev(synth.uniform(64, 64, 1)), dev(synth.uniform(64, 64, 2)), dev(np.zeros((64, 64)))
timeline("DGEMM 64^3 s=7", lambda: oz.dgemm("N", "N", 1.0, A, B, 0.0, C, 7))
A, B = dev(synth.kkr(512, 512, seed=1, gamma=3.0)), dev(synth.kkr(512, 512, seed=2, gamma=3.0))
C = dev(np.zeros((512, 512), complex))
for sk in ("1", "4"):
    os.environ["OZAKI_SPLITK"] = sk
    timeline(f"ZGEMM 512^3 4M s=7 splitk={sk}", lambda: oz.zgemm("N", "N", 1.0, A, B, 0.0, C, 7))
os.environ.pop("OZAKI_SPLITK")
n = 2048
A, B, C = dev(synth.uniform(n, n, 1)), dev(synth.uniform(n, n, 2)), dev(np.zeros((n, n)))
timeline(f"DGEMM {n}^3 s=7", lambda: oz.dgemm("N", "N", 1.0, A, B, 0.0, C, 7))
import bench  # noqa: E402
A_h, B_h = bench.make_inputs(30, 512, 3.0, 1000)
Az, Bz = bench.to_dev_batched(torch, A_h, "cuda"), bench.to_dev_batched(torch, B_h, "cuda")
Cz = torch.zeros((30, 512, 512), dtype=torch.complex128, device="cuda").transpose(1, 2)
timeline("C2x30 ZGEMM 512^3 4M s=7", lambda: oz.zgemm_strided_batched("N", "N", 1.0, Az, Bz, 0.0, Cz, 7))
