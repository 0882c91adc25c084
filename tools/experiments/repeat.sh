#!/bin/bash
# Repeat the config-4 bench to measure run-to-run variance (with clocks).
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv
for rep in 1 2 3 4; do
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/rep.log 2>&1
  echo "rep$rep: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/rep.log) $(grep -o '"clocks": {[^}]*}' gpurun_out/rep.log)"
done
nvidia-smi --query-compute-apps=pid,used_memory --format=csv
