#!/bin/bash
# memcheck + racecheck over the segment-path suites (block scan smem, two-scenario replay / transfer)
mkdir -p gpurun_out
T="tests/test_seg_gpu.py::test_seg_scan_kernels_many_segments tests/test_seg_gpu.py::test_seg_chain_carries_vs_single_pass_and_oracle tests/test_seg_gpu.py::test_seg_slot_graph_vs_oracle_and_single_pass"
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest $T -x -q -p no:cacheprovider > gpurun_out/san_mem.log 2>&1
echo "memcheck rc=$? $(grep -E 'passed|failed' gpurun_out/san_mem.log | tail -1) $(grep -c 'Invalid\|ERROR SUMMARY: [1-9]' gpurun_out/san_mem.log)"
timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest "tests/test_seg_gpu.py::test_seg_scan_kernels_many_segments" -x -q -p no:cacheprovider > gpurun_out/san_race.log 2>&1
echo "racecheck rc=$? $(grep -E 'passed|failed' gpurun_out/san_race.log | tail -1) $(grep -c 'Hazard\|ERROR SUMMARY: [1-9]' gpurun_out/san_race.log)"
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_breakdown_gpu.py tests/test_sweeps_gpu.py -x -q -p no:cacheprovider > gpurun_out/san_mem2.log 2>&1
echo "memcheck2 rc=$? $(grep -E 'passed|failed' gpurun_out/san_mem2.log | tail -1) $(grep -c 'Invalid\|ERROR SUMMARY: [1-9]' gpurun_out/san_mem2.log)"
