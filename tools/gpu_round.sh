#!/bin/bash
# One GPU session: parity tests, bench, ncu launch list + full capture.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1
tail -3 gpurun_out/tests.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:maxplus_dense -s 1 -c 1 -o gpurun_out/prof_dense python bench.py --scenarios 8192 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
