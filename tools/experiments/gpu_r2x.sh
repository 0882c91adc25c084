#!/bin/bash
# round-2 headline profiles + memcheck over the new kernels
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log | cut -c1-200
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lanes -s 1 -c 1 -o gpurun_out/prof_hot_r02 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_seg_gpu.py tests/test_breakdown_gpu.py tests/test_scale_vectors_gpu.py -q -x -k "not fullsize" > gpurun_out/memcheck_a.log 2>&1; echo "memcheck a rc=$?"; tail -3 gpurun_out/memcheck_a.log
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_columnar_gpu.py tests/test_whatif_batch_gpu.py -q -x -k "not million" > gpurun_out/memcheck_b.log 2>&1; echo "memcheck b rc=$?"; tail -3 gpurun_out/memcheck_b.log
