#!/bin/bash
mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_w_c4.jsonl 2> gpurun_out/bench_w_c4.err; python -c "
import json; l=json.loads(open('gpurun_out/bench_w_c4.jsonl').read().strip().splitlines()[-1]); print(l['value'], l['ms_per_step'], l['roofline']['frac'], l['e2e'], l['e2e_with_starts']['value'], l['cpu_baseline']['value'])"
for c in 2 3; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_w_c$c.jsonl 2>&1; python -c "
import json; l=json.loads(open('gpurun_out/bench_w_c$c.jsonl').read().strip().splitlines()[-1]); print($c, l['ms_per_step'], l['roofline']['frac'], l['clocks'])"; done
