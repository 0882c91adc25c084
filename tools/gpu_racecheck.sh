#!/bin/bash
# racecheck over the small-graph GPU suites (shared-memory hazards), then the full GPU suite
mkdir -p gpurun_out
for t in test_sim_gpu test_sweeps_gpu test_breakdown_gpu test_ingest_gpu test_transform_gpu; do
  timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 400 python -m pytest tests/$t.py -m gpu -x -q -p no:cacheprovider > gpurun_out/racecheck_$t.log 2>&1
  echo "racecheck $t rc=$? $(grep -E 'passed|failed' gpurun_out/racecheck_$t.log | tail -1) | $(tail -1 gpurun_out/racecheck_$t.log) | kernels: $(grep -o 'access at [a-zA-Z_:<>0-9]*' gpurun_out/racecheck_$t.log | sort | uniq -c | tr '\n' ' ')"
done
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/tests.log 2>&1; tail -2 gpurun_out/tests.log
