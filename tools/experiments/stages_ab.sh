#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2 3; do
  for st in 4 5 6; do
    DDSIM_LANES_STAGES=$st timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/v.log 2>&1
    echo "stages=$st rep$rep: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/v.log)"
  done
done
