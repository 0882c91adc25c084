#!/bin/bash
# GPU tests + the secondary-config measurements (configs 1, 2, 3, 5) + ingest stage profile.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/tests.log 2>&1; tail -3 gpurun_out/tests.log
timeout 1200 python tools/bench_configs.py --out gpurun_out/configs.json > gpurun_out/configs.log 2>&1; tail -c 2500 gpurun_out/configs.log
DDSIM_TRACE_TIMING= timeout 600 python tools/profile_ingest.py > gpurun_out/prof_ingest.log 2>&1; grep -E "rep|compile_graph|ks_ingest\]" gpurun_out/prof_ingest.log | tail -40
