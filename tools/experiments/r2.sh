#!/bin/bash
# two-scenario replay: seg suites, A/B vs one scenario per thread (DDSIM_SEG_R1)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_seg_gpu.py tests/test_fullsize_gpu.py tests/test_sweeps_gpu.py tests/test_whatif_batch_gpu.py tests/test_sim_gpu.py tests/test_breakdown_gpu.py tests/test_scale_vectors_gpu.py -x -q > gpurun_out/r2_tests.log 2>&1; tail -1 gpurun_out/r2_tests.log
grep -E "^E  |Error" gpurun_out/r2_tests.log | head -8
timeout 300 python tools/seg_probe.py config3 2>&1 | grep '"seg"'
timeout 300 python tools/seg_probe.py config3 DDSIM_SEG_R1=1 2>&1 | grep '"seg"'
for m in 160 240; do timeout 300 python tools/seg_probe.py config3 DDSIM_SEG_MIN_LEN=$m 2>&1 | grep '"seg"'; done
timeout 300 python tools/seg_probe.py config4 2048 8192 16384 2>&1 | grep '"seg"'
timeout 300 python tools/seg_probe.py config4 2048 8192 16384 DDSIM_SEG_R1=1 2>&1 | grep '"seg"'
