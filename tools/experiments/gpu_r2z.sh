#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sim_gpu.py tests/test_fullsize_gpu.py -q -x 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(l['ms_per_step'], l['roofline']['frac'], l['roofline']['pattern_frac'])"; done
