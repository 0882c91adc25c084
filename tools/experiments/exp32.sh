#!/bin/bash
# int32 duration expansion + retuned segment length: suites, config 2/3 timings, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_seg_gpu.py tests/test_fullsize_gpu.py tests/test_sim_gpu.py tests/test_scale_vectors_gpu.py tests/test_sweeps_gpu.py tests/test_whatif_batch_gpu.py -x -q > gpurun_out/exp32_tests.log 2>&1; tail -2 gpurun_out/exp32_tests.log
timeout 300 python tools/seg_probe.py config2 2>&1 | tail -4
timeout 300 python tools/seg_probe.py config2 DDSIM_EXPAND64=1 2>&1 | grep '"seg"'
for m in 128 160 256; do timeout 300 python tools/seg_probe.py config2 DDSIM_SEG_MIN_LEN=$m 2>&1 | grep '"seg"'; done
for c in 1 2 3; do timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-150; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp32_c2_launches.csv python bench.py --config 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
