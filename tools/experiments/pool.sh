#!/bin/bash
# scratch pool + JIT source on miss: full GPU suite, host overhead, configs 1-4
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pool_tests.log 2>&1; tail -1 gpurun_out/pool_tests.log
grep -E "^FAILED|Error" gpurun_out/pool_tests.log | head -5
python tools/experiments/c1_host.py 2>&1 | head -2
for c in 1 2 3; do timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-170; done
timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-170
