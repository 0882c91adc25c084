#!/bin/bash
# chain members loaded one ahead: chain suites, config 3 timing and launch split
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_seg_gpu.py tests/test_fullsize_gpu.py tests/test_sweeps_gpu.py tests/test_breakdown_gpu.py tests/test_whatif_batch_gpu.py tests/test_sim_gpu.py -x -q > gpurun_out/chainpf_tests.log 2>&1; tail -2 gpurun_out/chainpf_tests.log
timeout 300 python tools/seg_probe.py config3 2>&1 | tail -4
timeout 300 python bench.py --config 3 --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3pf_launches.csv python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
