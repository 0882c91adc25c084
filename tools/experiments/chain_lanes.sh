#!/bin/bash
# permutable chains on the lanes path: parity (sweeps, full-size config 3, what-if batch) + config 3 timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sweeps_gpu.py tests/test_fullsize_gpu.py tests/test_whatif_batch_gpu.py tests/test_sim_gpu.py tests/test_breakdown_gpu.py -q -x -rf 2>&1 | tail -4
for cfg in "DDSIM_NO_EXPAND=1" "X=1"; do
  env $cfg timeout 600 python tools/bench_configs.py --only 3 --out gpurun_out/c3.json > gpurun_out/c3.log 2>&1
  echo "$cfg config3: $(grep -o '"device_s": [0-9.e-]*' gpurun_out/c3.log) $(tail -c 400 gpurun_out/c3.log | grep -i error)"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python tools/bench_configs.py --only 3 --out gpurun_out/c3n.json > gpurun_out/c3n.log 2>&1
grep -E "lanes|maxplus|expand" gpurun_out/c3_launches.csv | awk -F'","' '{print $5, $NF}' | sort | uniq -c | sort -rn | head -8
