#!/bin/bash
# config 3 / config 1 launch lists and full ncu of the segment kernels at config 3
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_launches.csv python bench.py --config 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ddsim_seg -s 6 -c 4 -o gpurun_out/prof_c3_seg python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c3_ncu.log 2>&1; echo rc=$?; tail -1 gpurun_out/c3_ncu.log
