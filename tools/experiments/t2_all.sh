#!/bin/bash
# two-scenario transfer for derived durations / chains / carries: suites, A/B vs one scenario per thread
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_seg_gpu.py tests/test_fullsize_gpu.py tests/test_sweeps_gpu.py tests/test_whatif_batch_gpu.py tests/test_sim_gpu.py tests/test_breakdown_gpu.py -x -q > gpurun_out/t2_tests.log 2>&1; tail -1 gpurun_out/t2_tests.log
grep -E "Error|error" gpurun_out/t2_tests.log | head -5
for w in config3 config2; do timeout 300 python tools/seg_probe.py $w 2>&1 | grep '"seg"'; timeout 300 python tools/seg_probe.py $w DDSIM_SEG_T1=1 2>&1 | grep '"seg"'; done
timeout 300 python tools/seg_probe.py config4 8192 2>&1 | grep '"seg"'
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3t2_launches.csv python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
