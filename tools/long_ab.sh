# A/B of the long-row split forms on C3 / C5 / C4 (OZAKI_SPLIT_LONG=0: single kernel, 1: exps + per-window).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for L in 0 1; do
  for w in c3 c5; do
    OZAKI_SPLIT_LONG=$L timeout 300 python bench.py --workload $w --steps 5 --warmup 3 ${BENCH_ARGS} > gpurun_out/l.json 2>gpurun_out/l.err
    python -c "import json;d=json.load(open('gpurun_out/l.json'));print('$L $w',d['value'],d['ms_per_step'],d.get('phase_ms_per_step'))" || tail -3 gpurun_out/l.err
  done
  OZAKI_SPLIT_LONG=$L timeout 300 python bench.py --workload c4 --batch 32 --steps 3 --warmup 3 > gpurun_out/l.json 2>gpurun_out/l.err
  python -c "import json;d=json.load(open('gpurun_out/l.json'));print('$L c4',d['value'],d['ms_per_step'],d.get('phase_ms_per_step'))" || tail -3 gpurun_out/l.err
done
