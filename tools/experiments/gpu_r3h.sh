#!/bin/bash
timeout 900 python -m pytest tests/test_breakdown_gpu.py tests/test_whatif_batch_gpu.py -q -x 2>&1 | tail -1
for env in "X=1" "DDSIM_BD_LEAN=1" "DDSIM_BD_WINDOWS=20" "DDSIM_BD_WINDOWS=5"; do
  echo "$env: $(env $env timeout 600 python tools/bench_breakdown.py 2>&1 | tail -1 | cut -c1-260)"
done
