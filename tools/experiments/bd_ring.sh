#!/bin/bash
# ring vs lean breakdown merge: tests, timings at 65,536 x 100k
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_breakdown_gpu.py -x -q > gpurun_out/bdring_tests.log 2>&1; tail -1 gpurun_out/bdring_tests.log
for r in 1 2 3; do echo ring=$r; DDSIM_BD_RING=$r timeout 600 python tools/bench_breakdown.py 2>&1 | tail -1 | cut -c1-200; done
echo lean; DDSIM_BD_LEAN=1 timeout 600 python tools/bench_breakdown.py 2>&1 | tail -1 | cut -c1-200
