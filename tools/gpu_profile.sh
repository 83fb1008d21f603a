#!/bin/bash
# ncu evidence: launch list of a short bench run, one full capture of the TC kernel and
# of the cuBLAS comparator, and the cold-ring DRAM traffic ranges (roofline.traffic).
mkdir -p gpurun_out
TAG=${TAG:-prof}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
  --no-e2e --no-block --no-configs --gather none > gpurun_out/${TAG}_launches_bench.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kv_proj_tc -s 2 -c 1 \
  -o gpurun_out/${TAG}_full python tools/prof_kernel.py --reps 4 --dense > gpurun_out/${TAG}_full.log 2>&1
echo "full rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:"gemm|Kernel|sm100|cutlass|nvjet" -s 2 -c 1 \
  -o gpurun_out/${TAG}_dense python tools/prof_kernel.py --reps 4 --dense > gpurun_out/${TAG}_dense.log 2>&1
echo "dense rc=$?"
for impl in bd dense; do
  timeout 600 ncu --replay-mode app-range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --csv --log-file gpurun_out/${TAG}_traffic_${impl}.csv python tools/traffic_range.py --impl $impl --launches 40 \
    > gpurun_out/${TAG}_traffic_${impl}.log 2>&1
  echo "traffic $impl rc=$?"
done
tail -3 gpurun_out/${TAG}_full.log
