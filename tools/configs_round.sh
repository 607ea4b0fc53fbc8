#!/bin/bash
# secondary BASELINE configs + C3 slice sweep (1 GPU); outputs gpurun_out/cfg_*.json
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
timeout 120 python bench.py --workload c1 --steps 50 --warmup 5 > gpurun_out/cfg_c1.json 2> gpurun_out/cfg_c1.err
timeout 120 python bench.py --workload c2 --steps 50 --warmup 5 > gpurun_out/cfg_c2.json 2> gpurun_out/cfg_c2.err
for s in 3 4 5 6 7 8 9; do
  timeout 300 python bench.py --workload c3 --slices $s --steps 5 --warmup 3 > gpurun_out/cfg_c3_s$s.json 2> gpurun_out/cfg_c3_s$s.err
done
timeout 600 python bench.py --workload c4 --batch 32 --steps 3 --warmup 3 > gpurun_out/cfg_c4.json 2> gpurun_out/cfg_c4.err
timeout 600 python bench.py --workload c5 --steps 3 --warmup 3 > gpurun_out/cfg_c5.json 2> gpurun_out/cfg_c5.err
