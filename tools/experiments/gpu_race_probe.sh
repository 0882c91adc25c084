#!/bin/bash
# probe variants (traffic-pattern SOL) + racecheck / synccheck on the small-graph kernels
mkdir -p gpurun_out
timeout 600 python tools/probe_variants.py > gpurun_out/probe_variants.log 2>&1; cat gpurun_out/probe_variants.log | tail -8
for tool in racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -m pytest tests/test_sim_gpu.py tests/test_sweeps_gpu.py -m gpu -x -q -p no:cacheprovider > gpurun_out/${tool}.log 2>&1
  echo "$tool rc=$? $(grep -E 'passed|failed' gpurun_out/${tool}.log | tail -1) $(tail -1 gpurun_out/${tool}.log)"
done
