#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/v.log 2>&1
echo "config4: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/v.log) $(grep -o '"achieved": [0-9.]*' gpurun_out/v.log) $(grep -o '"pattern_copy_gbs": [0-9.]*' gpurun_out/v.log)"
done
