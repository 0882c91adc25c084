#!/bin/bash
# A/B lanes-kernel bodies on the config-4 bench: bash tools/ab.sh body1.cuh body2.cuh ...
for b in "$@"; do
  for rep in 1 2 3; do
    DDSIM_LANES_BODY=$PWD/$b timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/ab.log 2>&1
    echo "$b rep$rep: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab.log) $(grep -o '"kernel": "[^"]*"' gpurun_out/ab.log)"
  done
done
