#!/bin/bash
# alternate the current lanes body and a saved one on the config-4 bench (device arm)
mkdir -p gpurun_out
for rep in 1 2 3; do
  for b in "" "$1"; do
    if [ -n "$b" ]; then export DDSIM_LANES_BODY=$PWD/$b; else unset DDSIM_LANES_BODY; fi
    timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/ab.log 2>&1
    echo "${b:-current} rep$rep: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab.log) $(grep -o '"pattern_copy_gbs": [0-9.]*' gpurun_out/ab.log)"
  done
done
