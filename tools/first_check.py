"""Quick GPU sanity check: one small DGEMM through the C ABI vs the oracle."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2603_29975_b200 as oz

def dev(x):
    return oz.colmajor(torch.from_numpy(np.asfortranarray(x)).cuda())

print(oz.version(), torch.cuda.get_device_name(), flush=True)
for s in (1, 4, 8, 9):
    A = synth.uniform(64, 64, 1); B = synth.uniform(64, 64, 2)
    S = oz.debug_level_sums("N", "N", dev(A), dev(B), s).cpu().numpy()
    torch.cuda.synchronize()
    DA, _, _ = oracle.split_rows(np.ascontiguousarray(A), s)
    DB, _, _ = oracle.split_rows(np.ascontiguousarray(B.T), s)
    So = oracle.level_sums(DA, DB, s)
    print("s", s, "level sums match:", bool((S == So).all()), "max diff", int(np.abs(S - So).max()), flush=True)
    C = dev(np.zeros((64, 64)))
    oz.dgemm("N", "N", 1.0, dev(A), dev(B), 0.0, C, s)
    want = oracle.dgemm("N", "N", 1.0, A, B, 0.0, None, s)
    got = C.cpu().numpy()
    print("   dgemm bitexact:", bool((got == want).all()), "maxdiff", float(np.abs(got - want).max()), flush=True)
