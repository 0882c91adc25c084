#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/seg_probe.py config3 2>&1 | tail -3
timeout 600 python tools/seg_probe.py config2 2>&1 | tail -3
timeout 1700 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for c in 1 2 3; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_o_c$c.jsonl 2>&1; python -c "
import json; l=json.loads(open('gpurun_out/bench_o_c$c.jsonl').read().strip().splitlines()[-1]); print($c, l['ms_per_step'], l['roofline']['frac'], l['roofline'].get('path'), l['e2e']['value'])"; done
