"""G(z) inversion (n = 4096, emulated TRSM) over the block size nb: native vs Ozaki-I s = 4 / 7,
the inversion alone timed (residual after), plus a per-stage breakdown of one s = 7 inversion
(CUDA events around the panel LU, the U12 solve, the trailing update, the two blocked TRSMs)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2603_29975_b200 import workload as W  # noqa: E402

n = 4096
H, ev = synth.hamiltonian(n, seed=12)
Hd = torch.from_numpy(np.ascontiguousarray(H)).cuda()
M = complex(-0.2 + 0.05j) * torch.eye(n, dtype=torch.complex128, device="cuda") - Hd
out = {}
for nb in (256, 512, 1024):
    for gm in (W.gemm_native(), W.gemm_ozaki1(4), W.gemm_ozaki1(7)):
        W.blocked_lu_invert(M, nb, gm, emulated_trsm=True, check=False)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(2):
            Minv, _ = W.blocked_lu_invert(M, nb, gm, emulated_trsm=True, check=False)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / 2 * 1e3
        out[f"nb{nb}_{gm.label}"] = {"ms": round(ms, 2), "resid": W.residual(M, Minv)}
        print(nb, gm.label, out[f"nb{nb}_{gm.label}"], flush=True)
print(json.dumps(out))
