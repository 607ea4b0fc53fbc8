#!/bin/bash
# GPU-box script: ncu of the single-read cluster split (k_split_cluster) on C3 at s = 3 and 7:
# duration + DRAM bytes per launch, and one --set full capture at s = 7 (raw / details / source
# pages exported as CSV; the report itself is too big to bring back).
set -u
TAG=${1:-r2s3}
O=gpurun_out
for s in 3 7; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
      --clock-control none -k regex:k_split_cluster -s 2 -c 1 --csv --log-file $O/${TAG}_split_s${s}.csv \
      python tools/ncu_c3.py --s $s > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:k_split_cluster -s 2 -c 1 \
    -o $O/${TAG}_split_full -f python tools/ncu_c3.py --s 7 > $O/${TAG}_split_full.log 2>&1
for p in raw details; do
  ncu -i $O/${TAG}_split_full.ncu-rep --page $p --csv > $O/${TAG}_split_full_$p.csv 2>/dev/null
done
rm -f $O/${TAG}_split_full.ncu-rep
echo ncu_split_done
