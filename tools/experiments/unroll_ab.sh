#!/bin/bash
# config 2 (dyn lanes handler, latency-bound): kernel time vs record-loop unrolling
mkdir -p gpurun_out
for u in "" 2 4 16; do
  if [ -n "$u" ]; then export DDSIM_JIT_UNROLL=$u; else unset DDSIM_JIT_UNROLL; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lanes --csv --log-file gpurun_out/u.csv python tools/bench_configs.py --only 2,3 --out gpurun_out/u.json > gpurun_out/u.log 2>&1
  echo "unroll=${u:-1}: $(grep lanes gpurun_out/u.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
