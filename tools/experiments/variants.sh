#!/bin/bash
# Compare kernel variants on the config-4 bench (device arm only).
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_sim_gpu.py -q -x -k "dense" 2>&1 | tail -1
for cfg in "DDSIM_LANES_V=1" "DDSIM_LANES_V=2" "DDSIM_LANES_V=1 DDSIM_JIT_UNROLL=2" "DDSIM_LANES_V=1 DDSIM_NO_JIT=1" "DDSIM_LANES_V=2 DDSIM_JIT_UNROLL=4"; do
  env $cfg timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/v.log 2>&1
  echo "$cfg: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/v.log) $(grep -o '"frac": [0-9.]*' gpurun_out/v.log) $(grep -o '"kernel": "[^"]*"' gpurun_out/v.log)"
done
