# ncu --set full capture of the split kernel on the bench workload + source/raw/details pages.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-split}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_split -s 3 -c 1 -f -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-extras ${BENCH_ARGS} > gpurun_out/ncu_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_src.csv 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>&1
