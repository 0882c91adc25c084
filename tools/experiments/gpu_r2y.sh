#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/dropin_latency.py 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lanes|maxplus|listsched|probe|seg" -c 16 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log | cut -c1-120
for c in 2 3; do timeout 600 python bench.py --impl reference --config $c --steps 2 --warmup 1 2>&1 | tail -1 | cut -c1-300; done
