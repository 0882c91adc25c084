#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_seg_gpu.py tests/test_fullsize_gpu.py tests/test_scale_vectors_gpu.py tests/test_sim_gpu.py tests/test_sweeps_gpu.py -x -q > gpurun_out/expsm_tests.log 2>&1; tail -1 gpurun_out/expsm_tests.log
for c in 2 1; do timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-170; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2x_launches.csv python bench.py --config 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
