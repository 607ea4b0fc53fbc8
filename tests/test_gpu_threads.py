"""Re-entrancy across threads and streams (include/ozaki.h "Threads"): several host
threads call the library at once, each on its own CUDA stream, from a FRESH process so the
first calls race on the per-device shared-memory opt-in and the lazily built tables; every
result must equal the oracle bit for bit."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SNIPPET = r"""
import sys, threading
sys.path.insert(0, %r)
import numpy as np, torch
import oracle, synth
import paper_2603_29975_b200 as oz
oracle.build()
torch.cuda.init()
dev = lambda x: oz.colmajor(torch.from_numpy(np.asfortranarray(x)).cuda())
jobs = []
for t in range(6):
    m, n, k = 150 + 40 * t, 130 + 30 * t, 200 + 64 * t
    s = 3 + t
    kind = ("d", "z", "z3", "o2", "d", "z")[t]
    cplx = kind != "d" and kind != "o2"
    A = synth.uniform(m, k, 10 + t, complex_=cplx)
    B = synth.spread(k, n, 20 + t, phi=1.0, complex_=cplx)
    jobs.append((kind, s, A, B))
out = [None] * len(jobs)
err = []
barrier = threading.Barrier(len(jobs))

def work(i):
    try:
        kind, s, A, B = jobs[i]
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            Ad, Bd = dev(A), dev(B)
            C = dev(np.zeros((A.shape[0], B.shape[1]), A.dtype))
            barrier.wait()
            for _ in range(5):
                if kind == "d": oz.dgemm("N", "N", 1.0, Ad, Bd, 0.0, C, s)
                elif kind == "z": oz.zgemm("N", "N", 1.0, Ad, Bd, 0.0, C, s)
                elif kind == "z3": oz.zgemm3m("N", "N", 1.0, Ad, Bd, 0.0, C, s)
                else: oz.ozaki2_dgemm("N", "N", 1.0, Ad, Bd, 0.0, C, 8 + s)
            st.synchronize()
            out[i] = C.cpu().numpy()
    except Exception as e:  # noqa: BLE001
        err.append(repr(e))

th = [threading.Thread(target=work, args=(i,)) for i in range(len(jobs))]
[t.start() for t in th]
[t.join() for t in th]
assert not err, err
from oracle import ozaki2 as o2
bad = 0
for (kind, s, A, B), got in zip(jobs, out):
    if kind == "d": want = oracle.dgemm("N", "N", 1.0, A, B, 0.0, None, s)
    elif kind == "z": want = oracle.zgemm("N", "N", 1.0, A, B, 0.0, None, s)
    elif kind == "z3": want = oracle.zgemm("N", "N", 1.0, A, B, 0.0, None, s, "3m")
    else: want = o2.dgemm("N", "N", 1.0, A[:20], B, 0.0, None, 8 + s); got = got[:20]
    bad += int(not (got == want).all())
print("BAD", bad)
"""


def test_threads_fresh_process_bitexact():
    r = subprocess.run([sys.executable, "-c", _SNIPPET % ROOT], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "BAD 0" in r.stdout, r.stdout + r.stderr[-2000:]
