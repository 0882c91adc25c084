#!/bin/bash
# lanes kernel + separate lane-busy pass vs in-kernel lane busy (DDSIM_DYN_LB) on configs 2/3
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sweeps_gpu.py tests/test_sim_gpu.py tests/test_fullsize_gpu.py tests/test_whatif_batch_gpu.py tests/test_breakdown_gpu.py -q -x 2>&1 | tail -1
for cfg in "X=1" "DDSIM_DYN_LB=1"; do
  env $cfg timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lanes" --csv --log-file gpurun_out/u.csv python tools/bench_configs.py --only 2,3 --out gpurun_out/u.json > gpurun_out/u.log 2>&1
  echo "$cfg:"; grep -E 'lanes' gpurun_out/u.csv | awk -F'","' '{print "   "substr($5,1,30)" "$NF}' | tr -d '"'
  env $cfg timeout 600 python tools/bench_configs.py --only 2,3 --out gpurun_out/u2.json > gpurun_out/u2.log 2>&1; grep -o '"device_s": [0-9.e-]*' gpurun_out/u2.log
done
