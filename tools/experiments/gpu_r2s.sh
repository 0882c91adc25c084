#!/bin/bash
# device freeze of ingested traces
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_columnar_gpu.py tests/test_ingest_gpu.py -q -x 2>&1 | tail -3
DDSIM_INGEST_TIMING=1 timeout 1200 python bench.py --config 5 --no-cpu-baseline --steps 3 --warmup 1 > gpurun_out/c5_dev.jsonl 2> gpurun_out/c5_dev.err
grep -E "compile_graph|FrozenGraph|ks_ingest\]|ingest_arrays" gpurun_out/c5_dev.err | tail -24
tail -5 gpurun_out/c5_dev.err | grep -iE "error|Trace" 
python -c "
import json; l=json.loads(open('gpurun_out/c5_dev.jsonl').read().strip().splitlines()[-1]); print(l['ms_per_step'], l['config'], l['e2e']['value'], l['parity_checked'])"
