#!/bin/bash
# lanes kernel CTA size on config 4: 112 (2 CTAs/SM, default) vs 224 (1 CTA/SM) vs 64 / 80
mkdir -p gpurun_out
for rep in 1 2; do
  for bd in "" 224 64 80; do
    if [ -n "$bd" ]; then export DDSIM_LANES_BD=$bd; else unset DDSIM_LANES_BD; fi
    timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/v.log 2>&1
    echo "BD=${bd:-112} rep$rep: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/v.log) $(tail -c 300 gpurun_out/v.log | grep -io error | head -1)"
  done
done
