#!/bin/bash
# config-4 variants re-measured once the first-launch pool penalty is gone (interleaved repeats)
mkdir -p gpurun_out
for rep in 1 2 3; do
for cfg in ${AB_CFGS:-"X=1" "DDSIM_JIT_UNROLL=2" "DDSIM_JIT_UNROLL=4"}; do
  env $cfg timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/v.log 2>&1
  echo "$cfg: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/v.log)"
done; done
