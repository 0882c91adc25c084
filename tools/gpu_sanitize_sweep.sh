#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the breakdown sweep tests
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  sel="sweep_jittered or (keywords and sweep and not depth1)"
  [ $tool = memcheck ] && sel="sweep"
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python -m pytest tests/test_breakdown_gpu.py -x -q -p no:cacheprovider -k "$sel" > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'passed|failed' gpurun_out/san_$tool.log | tail -1) $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_$tool.log | sort | uniq -c | tr '\n' ';')"
done | tee gpurun_out/san_summary.txt
