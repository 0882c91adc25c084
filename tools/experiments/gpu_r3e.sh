#!/bin/bash
for c in 1 2 3; do timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print($c, round(l['ms_per_step'],4), '%.3g' % l['e2e']['value'])"; done
timeout 900 python -m pytest tests/test_seg_gpu.py tests/test_fullsize_gpu.py -q -x 2>&1 | tail -1
