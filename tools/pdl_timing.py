import os, sys, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, bench
import paper_2603_29975_b200 as oz
batch, n = 30, 512
A_h, B_h = bench.make_inputs(batch, n, 3.0, 1000)
dv = torch.device("cuda", 0)
A = bench.to_dev_batched(torch, A_h, dv); B = bench.to_dev_batched(torch, B_h, dv)
C = torch.zeros((batch, n, n), dtype=torch.complex128, device=dv).transpose(1, 2)
f = lambda: oz.zgemm_strided_batched("N", "N", 1.0, A, B, 0.0, C, 7)
for _ in range(5): f()
torch.cuda.synchronize()
res = []
for rep in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): f()
    e1.record(); torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / 50)
print(json.dumps({"pdl": os.environ.get("OZAKI_NO_PDL") is None, "ms": res}))
