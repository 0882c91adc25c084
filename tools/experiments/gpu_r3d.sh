#!/bin/bash
# config 1 (2 scenarios): segment length floor
for e in X=1 DDSIM_SEG_MIN_LEN=160 DDSIM_SEG_MIN_LEN=96 DDSIM_SEG_MIN_LEN=48; do
  env $e timeout 300 python bench.py --config 1 --no-cpu-baseline --steps 20 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$e', round(l['ms_per_step'],4), '%.3g' % l['e2e']['value'])"
done
