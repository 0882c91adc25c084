#!/bin/bash
# lazy kernel programs: full GPU suite + config 5 stage timing
mkdir -p gpurun_out
timeout 1700 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
DDSIM_INGEST_TIMING=1 timeout 900 python bench.py --config 5 --no-cpu-baseline --steps 3 --warmup 1 > gpurun_out/c5_lazy.jsonl 2> gpurun_out/c5_lazy.err
grep -E "compile_graph|FrozenGraph|ks_ingest\]|ingest_arrays|rep " gpurun_out/c5_lazy.err | tail -40
python -c "
import json; l=json.loads(open('gpurun_out/c5_lazy.jsonl').read().strip().splitlines()[-1]); print(l['ms_per_step'], l['config'], l['e2e']['value'])"
