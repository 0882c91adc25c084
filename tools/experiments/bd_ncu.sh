#!/bin/bash
# expansion suites + breakdown merge kernel: timing and one full ncu capture with source
mkdir -p gpurun_out
bash tools/experiments/exp32.sh
timeout 600 python tools/bench_breakdown.py 2>&1 | tail -3
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:breakdown_lean -c 1 -o gpurun_out/prof_bd_lean python tools/bench_breakdown.py > gpurun_out/bd_ncu.log 2>&1; echo ncu rc=$?; tail -2 gpurun_out/bd_ncu.log
