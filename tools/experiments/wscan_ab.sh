#!/bin/bash
# warp-parallel segment scan vs the sequential one (DDSIM_SEG_SEQSCAN), plus the seg suites
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_seg_gpu.py tests/test_fullsize_gpu.py tests/test_sim_gpu.py tests/test_scale_vectors_gpu.py -x -q > gpurun_out/wscan_tests.log 2>&1; tail -2 gpurun_out/wscan_tests.log
for w in config2 config3; do timeout 600 python tools/seg_probe.py $w 2>&1 | tail -4; done
timeout 600 python tools/seg_probe.py config4 2048 8192 2>&1 | grep -v "^$" | tail -8
timeout 300 python bench.py --config 1 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200
timeout 300 python bench.py --config 2 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/wscan_c2_launches.csv python bench.py --config 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
