#!/bin/bash
# lean breakdown merge vs the previous kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_breakdown_gpu.py tests/test_whatif_batch_gpu.py -q -x 2>&1 | tail -2
for env in "X=1" "DDSIM_BD_LB_SCALAR=1" "DDSIM_BD_WINDOWS=14"; do
  echo "$env: $(env $env timeout 600 python tools/bench_breakdown.py 2>&1 | tail -1)"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"breakdown|bd_" -c 4 --csv python tools/bench_breakdown.py > gpurun_out/bd_ncu2.csv 2>&1
grep -E "breakdown|bd_" gpurun_out/bd_ncu2.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-150
