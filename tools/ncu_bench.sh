#!/bin/bash
# GPU-box script: launch list of the default bench command + per-s ncu metrics of the C3 slice
# GEMM + one full-set capture at s=7.  Outputs under gpurun_out/ (summarised by
# tools/ncu_c3_summary.py into profiles/).
set -u
TAG=${1:-r2}
O=gpurun_out
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-extras > $O/${TAG}_launches_bench.log 2>&1
for s in 3 4 5 6 7 8 9; do
  ncu --metrics $M --clock-control none -k regex:k_gemm_lv2 -s 2 -c 1 --csv \
      --log-file $O/${TAG}_c3_s${s}.csv python tools/ncu_c3.py --s $s > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:k_split -s 2 -c 1 --csv --log-file $O/${TAG}_c3_split_s${s}.csv python tools/ncu_c3.py --s $s > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:k_gemm_lv2 -s 2 -c 1 \
    -o $O/${TAG}_c3_s7_full -f python tools/ncu_c3.py --s 7 > $O/${TAG}_full.log 2>&1
ncu -i $O/${TAG}_c3_s7_full.ncu-rep --page raw --csv > $O/${TAG}_c3_s7_full_raw.csv 2>/dev/null
rm -f $O/${TAG}_c3_s7_full.ncu-rep
echo ncu_done
