#!/bin/bash
# breakdown: evict-first vs cached start loads, windows
mkdir -p gpurun_out
for env in "DDSIM_BD_STREAM=1" "X=1" "DDSIM_BD_WINDOWS=2" "DDSIM_BD_WINDOWS=10"; do
  echo "$env: $(env $env timeout 600 python tools/bench_breakdown.py 2>&1 | tail -1)"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:breakdown_kernel -c 1 --csv python tools/bench_breakdown.py > gpurun_out/bd_ncu.csv 2>&1
grep -E "breakdown_kernel" gpurun_out/bd_ncu.csv | awk -F'","' '{print $(NF-2), $NF}' | head
