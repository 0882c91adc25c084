#!/bin/bash
# GPU tests, then compute-sanitizer memcheck / racecheck over the small-graph GPU tests.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/tests.log 2>&1; tail -2 gpurun_out/tests.log
for t in test_sim_gpu test_sweeps_gpu test_breakdown_gpu test_ingest_gpu test_transform_gpu; do
  timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/$t.py -m gpu -x -q -p no:cacheprovider > gpurun_out/memcheck_$t.log 2>&1
  echo "memcheck $t rc=$? $(grep -E 'passed|failed' gpurun_out/memcheck_$t.log | tail -1) $(grep -c 'Invalid\|ERROR SUMMARY: [1-9]' gpurun_out/memcheck_$t.log)"
done
