#!/bin/bash
for gb in 1 4 16 100; do
  DDSIM_CHUNK_GB=$gb timeout 600 python bench.py --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/e2e.log 2>&1
  echo "chunk ${gb}GB: $(grep -o '"e2e": {[^}]*}' gpurun_out/e2e.log)"
done
