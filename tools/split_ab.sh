# A/B timing of the K1 variants on the bench workload (and C3 DGEMM split via bench --workload c3 if given).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in "OZAKI_SPLIT_ROWS=4" "OZAKI_SPLIT_ROWS=8" "OZAKI_SPLIT=generic"; do
  env $v timeout 300 python bench.py --no-extras --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v',d['value'],d['ms_per_step'],d['roofline_split']['achieved'],d.get('phase_ms_per_step'))" || tail -5 gpurun_out/ab.err
done
