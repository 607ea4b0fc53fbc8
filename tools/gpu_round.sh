#!/bin/bash
# One gpurun call: smoke, bench, launch list, ncu full captures.  Outputs in gpurun_out/.
set -x
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-extras ${BENCH_ARGS} > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 3 -c 1 -f -o gpurun_out/prof_gemm_$TAG \
    python bench.py --steps 1 --warmup 3 --no-extras ${BENCH_ARGS} > gpurun_out/ncu_gemm_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_split -s 3 -c 1 -f -o gpurun_out/prof_split_$TAG \
    python bench.py --steps 1 --warmup 3 --no-extras ${BENCH_ARGS} > gpurun_out/ncu_slice_$TAG.log 2>&1
for k in gemm split; do   # export the raw pages here; the reports are too big to bring back
  [ -f gpurun_out/prof_${k}_$TAG.ncu-rep ] || continue
  ncu -i gpurun_out/prof_${k}_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_${k}_${TAG}_raw.csv 2>&1
  ncu -i gpurun_out/prof_${k}_$TAG.ncu-rep --page details --csv > gpurun_out/prof_${k}_${TAG}_details.csv 2>&1
  rm -f gpurun_out/prof_${k}_$TAG.ncu-rep
done
fi
ls -la gpurun_out
