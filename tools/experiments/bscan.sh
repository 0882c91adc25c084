#!/bin/bash
# block scan + small-S expansion: seg suites, config 1 timing
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_seg_gpu.py tests/test_fullsize_gpu.py tests/test_scale_vectors_gpu.py tests/test_sim_gpu.py -x -q > gpurun_out/bscan_tests.log 2>&1; tail -1 gpurun_out/bscan_tests.log
grep -E "Error|assert" gpurun_out/bscan_tests.log | head -5
for c in 1 2; do timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-150; done
