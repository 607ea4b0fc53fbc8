cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_split -s 3 -c 1 -f -o gpurun_out/prof_split_r1z python bench.py --steps 1 --warmup 3 --no-extras > gpurun_out/ncu_split_r1z.log 2>&1
ncu -i gpurun_out/prof_split_r1z.ncu-rep --page source --csv --print-source sass > gpurun_out/split_src_r1z.csv 2>&1
ncu -i gpurun_out/prof_split_r1z.ncu-rep --page raw --csv > gpurun_out/split_raw_r1z.csv 2>&1
ncu -i gpurun_out/prof_split_r1z.ncu-rep --page details --csv > gpurun_out/split_details_r1z.csv 2>&1
ls -la gpurun_out
